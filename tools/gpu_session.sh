cd $GRAFT_REPO_ROOT
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/s1_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout=300 --timeout_method=thread > $O/s1_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/s1_gpu_tests.log
timeout 300 python bench.py > $O/s1_bench.json 2> $O/s1_bench.err
timeout 600 python tools/bench_configs.py --configs 2,3,4,5 --iters 5 > $O/s1_configs.jsonl 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/s1_smoke.log 2>&1
