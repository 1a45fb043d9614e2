cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_semimarkov_gpu.py -x -q --timeout=900 > $O/smv_tests.log 2>&1; echo "rc=$?" >> $O/smv_tests.log
