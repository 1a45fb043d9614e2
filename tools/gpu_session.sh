cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python tools/bench_ops.py > $O/ops2.jsonl 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_vit2_gpu.py tests/test_kbest_gpu.py -x -q --timeout=600 > $O/ops2_tests.log 2>&1; echo "rc=$?" >> $O/ops2_tests.log
