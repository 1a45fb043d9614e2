cd $GRAFT_REPO_ROOT
O=gpurun_out
T=fin
timeout 1500 python -m pytest tests -m gpu -q --timeout=600 > $O/${T}_gpu_tests.log 2>&1; echo "rc=$?" >> $O/${T}_gpu_tests.log
timeout 300 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1
timeout 600 python tools/bench_configs.py --configs 2,3,4,5 --iters 5 > $O/${T}_configs.jsonl 2>&1
timeout 600 python tools/bench_ops.py > $O/${T}_ops.jsonl 2>&1
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > $O/${T}_ref.json 2>&1
bash tools/profile_all.sh r1d > $O/${T}_prof.log 2>&1
