cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_dist_gpu.py -x -q --timeout=900 > $O/exp_tests.log 2>&1; echo "rc=$?" >> $O/exp_tests.log
