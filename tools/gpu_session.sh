cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q --timeout=900 -k "host" > $O/host_tests.log 2>&1; echo "rc=$?" >> $O/host_tests.log
for i in 1 2 3; do timeout 300 python bench.py > $O/host_bench_$i.json 2>>$O/host_bench.err; done
