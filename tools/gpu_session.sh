cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_kbest_gpu.py tests/test_dist_gpu.py -x -q --timeout=900 > $O/kb_tests.log 2>&1; echo "rc=$?" >> $O/kb_tests.log
timeout 600 python tools/bench_ops.py --iters 5 > $O/ops10.jsonl 2> $O/ops10.err
