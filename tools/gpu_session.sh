cd $GRAFT_REPO_ROOT
O=gpurun_out
T=k1
timeout 900 python -m pytest tests/test_kbest_gpu.py -x -q --timeout=300 > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
