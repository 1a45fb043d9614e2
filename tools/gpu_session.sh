cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python tools/bench_ops.py > $O/ops3.jsonl 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_kbest_gpu.py tests/test_semimarkov_gpu.py -x -q --timeout=600 > $O/ops3_tests.log 2>&1; echo "rc=$?" >> $O/ops3_tests.log
