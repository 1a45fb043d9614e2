cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 60 ./tools/phase_tiny 32 25 20 > $O/g4_phase.txt 2>&1
timeout 600 python -m pytest tests/test_tiny_gpu.py tests/test_parity_gpu.py -x -q --timeout=600 > $O/g4_tests.log 2>&1; echo "rc=$?" >> $O/g4_tests.log
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --e2e-steps 20 >> $O/g4_bench.jsonl 2>> $O/g4_bench.err; done
