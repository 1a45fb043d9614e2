cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout=1200 -k "viterbi or Viterbi or segment or max or kbest or tie" > $O/vit_tests.log 2>&1; echo "rc=$?" >> $O/vit_tests.log
timeout 600 python tools/bench_ops.py --iters 5 > $O/ops7.jsonl 2> $O/ops7.err
