# A/B of the e2e (host-buffer) leg between library builds: alternating processes.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2 3; do
  for lib in libts_b200_k0.so libts_b200.so; do
    echo "== $lib run $r"
    TS_B200_LIB=$PWD/paper_2002_00876_b200/$lib timeout 200 python tools/e2e_only.py
  done
done
