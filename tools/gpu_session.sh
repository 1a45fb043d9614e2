cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout=1500 -p no:cacheprovider > $O/fin6_tests.log 2>&1; echo "rc=$?" >> $O/fin6_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke OK')" > $O/fin6_smoke.log 2>&1; echo "rc=$?" >> $O/fin6_smoke.log
timeout 1200 compute-sanitizer --tool racecheck python tools/sanitize_all.py > $O/fin6_racecheck.log 2>&1; echo "rc=$?" >> $O/fin6_racecheck.log
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_all.py > $O/fin6_memcheck.log 2>&1; echo "rc=$?" >> $O/fin6_memcheck.log
timeout 300 python bench.py > $O/fin6_bench.json 2>$O/fin6_bench.err
