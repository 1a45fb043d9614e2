cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
  timeout 900 python -m pytest tests/test_tiny_gpu.py tests/test_parity_gpu.py tests/test_scan_gpu.py tests/test_cfg5_full_gpu.py tests/test_dist_gpu.py -q -p no:cacheprovider -p no:randomly 2>&1 | tail -1
done
