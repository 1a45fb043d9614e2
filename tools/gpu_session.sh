cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout=1500 -p no:cacheprovider > $O/fin4_tests.log 2>&1; echo "rc=$?" >> $O/fin4_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke OK')" > $O/fin4_smoke.log 2>&1; echo "rc=$?" >> $O/fin4_smoke.log
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_all.py > $O/fin4_memcheck.log 2>&1; echo "rc=$?" >> $O/fin4_memcheck.log
for i in 1 2; do timeout 300 python bench.py > $O/fin4_bench_$i.json 2>>$O/fin4_bench.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r1e_ops_launches.csv python tools/bench_ops.py --iters 1 > /dev/null 2>&1
timeout 600 python tools/bench_ops.py --iters 5 > $O/r1e_ops.jsonl 2> $O/ops8.err
