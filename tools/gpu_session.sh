cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_semimarkov_gpu.py tests/test_parity_gpu.py -k "semimarkov or wide" -x -q --timeout=900 > $O/sm_tests.log 2>&1; echo "rc=$?" >> $O/sm_tests.log
timeout 600 python tools/bench_ops.py --iters 5 > $O/ops5.jsonl 2> $O/ops5.err
