cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_scan_gpu.py tests/test_segments_gpu.py -x -q --timeout=120 --timeout_method=thread > $O/s17_scan_tests.log 2>&1
