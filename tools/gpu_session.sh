cd $GRAFT_REPO_ROOT
O=gpurun_out
L=paper_2002_00876_b200
cp $L/libts_b200.so /tmp/keep.so
for d in 0 4 6 8; do cp $L/libts_b200_k_w$d.so $L/libts_b200.so; timeout 300 python tools/wide_time.py w$d >> $O/wide_l2.log 2>&1; done
cp /tmp/keep.so $L/libts_b200.so
