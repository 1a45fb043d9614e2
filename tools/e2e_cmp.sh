cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do
python bench.py --steps 2000 --warmup 50 --reps 3 --side "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench e2e us/call', 800/d['e2e']['value']*1e6, 'warm', d['e2e']['warmup_calls'])"
python tools/e2e_only.py
python bench.py --steps 20 --warmup 3 --reps 0 --side "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench(20 steps) e2e us/call', 800/d['e2e']['value']*1e6, 'warm', d['e2e']['warmup_calls'])"
done
