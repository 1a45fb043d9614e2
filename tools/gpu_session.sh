cd $GRAFT_REPO_ROOT
O=gpurun_out
T=tc6
timeout 60 ./tools/phase_tc 64 1 > $O/${T}_phase.txt 2>&1
timeout 60 ./tools/phase_tc 1024 148 >> $O/${T}_phase.txt 2>&1
timeout 300 python tools/bench_configs.py --configs 5 --iters 3 > $O/${T}_cfg5.jsonl 2>&1
timeout 900 python -m pytest tests/test_scan_gpu.py tests/test_segments_gpu.py -x -q --timeout=600 > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
