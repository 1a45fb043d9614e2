cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tiny_gpu.py tests/test_parity_gpu.py tests/test_dist_gpu.py -q -x -p no:cacheprovider > gpurun_out/tiny_tests.log 2>&1; tail -3 gpurun_out/tiny_tests.log
timeout 300 python bench.py --steps 2000 --warmup 50 --reps 3 --side "" --no-cpu-baseline --e2e-steps 20 > gpurun_out/tiny_bench.json 2> gpurun_out/tiny_bench.err
timeout 300 python bench.py --steps 20 --warmup 3 --reps 3 --side "" --no-cpu-baseline --e2e-steps 20 > gpurun_out/tiny_bench20.json 2>> gpurun_out/tiny_bench.err
