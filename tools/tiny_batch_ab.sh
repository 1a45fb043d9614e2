cd $GRAFT_REPO_ROOT
for lib in libts_b200_k0.so libts_b200.so; do echo "== $lib"; TS_B200_LIB=$PWD/paper_2002_00876_b200/$lib python tools/tiny_batch_probe.py; done
bash tools/tiny_ab.sh libts_b200_k0.so libts_b200.so
