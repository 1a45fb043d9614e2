cd $GRAFT_REPO_ROOT
O=gpurun_out
T=tc3
timeout 900 python -m pytest tests/test_scan_gpu.py tests/test_segments_gpu.py tests/test_parity_gpu.py -x -q --timeout=300 > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 300 python tools/bench_configs.py --configs 5 --iters 3 > $O/${T}_cfg5.jsonl 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:summary|tree|fwd2|bwd2' -c 40 --csv --log-file $O/${T}_launches_cfg5.csv python tools/bench_configs.py --configs 5 --iters 1 > /dev/null 2>&1
