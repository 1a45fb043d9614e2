cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout=1500 -p no:cacheprovider > $O/fin3_tests.log 2>&1; echo "rc=$?" >> $O/fin3_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke OK')" > $O/fin3_smoke.log 2>&1; echo "rc=$?" >> $O/fin3_smoke.log
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_all.py > $O/fin3_memcheck.log 2>&1; echo "rc=$?" >> $O/fin3_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck python tools/sanitize_all.py > $O/fin3_racecheck.log 2>&1; echo "rc=$?" >> $O/fin3_racecheck.log
for i in 1 2; do timeout 300 python bench.py > $O/fin3_bench_$i.json 2>>$O/fin3_bench.err; done
timeout 300 python bench.py --impl reference > $O/fin3_ref.json 2>>$O/fin3_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:fb_wide_ring" -c 1 -f -o $O/r1e_full_wide_ring python tools/run_once.py --op marg --B 64 --N 1024 --C 256 --reps 1 > $O/r1e_full_wide.log 2>&1
ncu -i $O/r1e_full_wide_ring.ncu-rep --page raw --csv > $O/r1e_full_wide_ring_raw.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:fb_wide_marg" -c 1 -f -o $O/r1e_full_wide_marg python tools/run_once.py --op marg --B 64 --N 1024 --C 256 --reps 1 > $O/r1e_full_wide2.log 2>&1
ncu -i $O/r1e_full_wide_marg.ncu-rep --page raw --csv > $O/r1e_full_wide_marg_raw.csv 2>/dev/null
rm -f $O/*.ncu-rep
