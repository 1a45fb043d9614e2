cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q --timeout=900 -k "wide" > $O/wide_tests.log 2>&1; echo "rc=$?" >> $O/wide_tests.log
timeout 300 python tools/wide_time.py prod > $O/wide_prod.log 2>&1
