cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 60 ./tools/phase_cscan > gpurun_out/phase_cscan.txt 2>&1
timeout 900 python -m pytest tests/test_tiny_gpu.py -q -x -p no:cacheprovider > gpurun_out/cscan_tests.log 2>&1; tail -15 gpurun_out/cscan_tests.log
timeout 300 python bench.py --steps 2000 --warmup 50 --reps 3 --side "" --no-cpu-baseline --e2e-steps 20 > gpurun_out/cscan_bench.json 2> gpurun_out/cscan_bench.err
tail -3 gpurun_out/cscan_bench.err
