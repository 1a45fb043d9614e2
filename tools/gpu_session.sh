cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_scan_gpu.py -x -q -k "tensor_core" > $O/s13_tc_tests.log 2>&1
timeout 300 python tools/bench_configs.py --configs 5 --iters 3 --tc 3 > $O/s13_cfg5.jsonl 2>&1
timeout 300 python tools/bench_configs.py --configs 5 --iters 3 --tc 1 >> $O/s13_cfg5.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/s13_launches_cfg5.csv \
     python tools/run_once.py --op marg --B 4 --N 65536 --C 128 --reps 1 > /dev/null 2>&1
