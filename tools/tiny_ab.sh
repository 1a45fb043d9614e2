# A/B of bench cfg2 between library builds (TS_B200_LIB), alternating processes.
cd $GRAFT_REPO_ROOT
for r in 1 2; do for lib in "$@"; do
  echo -n "$lib: "; TS_B200_LIB=$PWD/paper_2002_00876_b200/$lib python bench.py --steps 2000 --warmup 50 --reps 3 --side "" --no-cpu-baseline --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3, 4), d['timing'] if 'timing' in d else '')"
done; done
