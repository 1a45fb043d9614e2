cd $GRAFT_REPO_ROOT
O=gpurun_out
T=sm1
timeout 900 python -m pytest tests/test_semimarkov_gpu.py -x -q --timeout=300 > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
