cd $GRAFT_REPO_ROOT
O=gpurun_out
T=f2
timeout 1500 python -m pytest tests -m gpu -q --timeout=600 > $O/${T}_gpu_tests.log 2>&1; echo "rc=$?" >> $O/${T}_gpu_tests.log
timeout 300 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 9 python tools/sanitize_all.py > $O/${T}_racecheck.log 2>&1; echo "rc=$?" >> $O/${T}_racecheck.log
