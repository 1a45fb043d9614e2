cd $GRAFT_REPO_ROOT
O=gpurun_out
T=san2
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 9 python tools/sanitize_all.py > $O/${T}_racecheck.log 2>&1; echo "rc=$?" >> $O/${T}_racecheck.log
timeout 600 python -m pytest tests/test_tiny_gpu.py -x -q --timeout=120 > $O/${T}_tiny.log 2>&1; echo "rc=$?" >> $O/${T}_tiny.log
