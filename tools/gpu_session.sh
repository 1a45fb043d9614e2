cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout=1500 -p no:cacheprovider > $O/fin7_tests.log 2>&1; echo "rc=$?" >> $O/fin7_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke OK')" > $O/fin7_smoke.log 2>&1; echo "rc=$?" >> $O/fin7_smoke.log
timeout 300 python bench.py > $O/fin7_bench.json 2>$O/fin7_bench.err
timeout 300 python bench.py --impl reference > $O/fin7_ref.json 2>>$O/fin7_bench.err
