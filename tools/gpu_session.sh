cd $GRAFT_REPO_ROOT
O=gpurun_out
T=w1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_semimarkov_gpu.py -x -q --timeout=600 -k "wide or semimarkov" > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
