cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q --timeout=900 -k "wide" > $O/wide_tests.log 2>&1; echo "rc=$?" >> $O/wide_tests.log
timeout 600 python tools/bench_ops.py --iters 5 > $O/ops3.jsonl 2> $O/ops3.err
