cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_dist_gpu.py -x -q --timeout=900 -k "wide or entropy" > $O/wide_tests.log 2>&1; echo "rc=$?" >> $O/wide_tests.log
