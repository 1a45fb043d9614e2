cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 120 python tools/e2e_ab.py paper_2002_00876_b200/libts_b200.so >> $O/e2eab3.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > $O/e2eab3_bench.json 2>/dev/null
timeout 120 python tools/e2e_ab.py paper_2002_00876_b200/libts_b200.so >> $O/e2eab3.txt 2>&1
