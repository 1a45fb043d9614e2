cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_scan_gpu.py tests/test_segments_gpu.py -x -q --timeout=600 > $O/tu_tests.log 2>&1; echo "rc=$?" >> $O/tu_tests.log
timeout 300 python tools/bench_configs.py --configs 5 --iters 3 > $O/tu_cfg5.jsonl 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:tree' -c 20 --csv --log-file $O/tu_launches.csv python tools/bench_configs.py --configs 5 --iters 1 > /dev/null 2>&1
