cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python -m pytest tests/test_dist_gpu.py -x -q --timeout=600 > $O/det_tests.log 2>&1; echo "rc=$?" >> $O/det_tests.log
