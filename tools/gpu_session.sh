cd $GRAFT_REPO_ROOT
O=gpurun_out
T=o2
timeout 60 ./tools/phase_tiny_ovl 32 25 20 > $O/${T}_phase2.txt 2>&1
timeout 600 python -m pytest tests/test_tiny_gpu.py -x -q --timeout=120 > $O/${T}_tiny.log 2>&1; echo "rc=$?" >> $O/${T}_tiny.log
for m in 1 2 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 1000 --tiny-mode $m --e2e-steps 20 >> $O/${T}_bench.jsonl 2>> $O/${T}_bench.err; done
