cd $GRAFT_REPO_ROOT
./tools/phase_tc 256 148 | tail -1; ./tools/phase_tc_ps 256 148 | tail -1; ./tools/phase_tc_ps 256 148 | sed -n 2,8p
for lib in libts_b200.so libts_b200_ps.so; do echo "== $lib"; TS_B200_LIB=$PWD/paper_2002_00876_b200/$lib python tools/cfg5_chunk_sweep.py 2>&1 | head -1; done
TS_B200_LIB=$PWD/paper_2002_00876_b200/libts_b200_ps.so timeout 1200 python -m pytest tests/test_scan_gpu.py tests/test_cfg5_full_gpu.py tests/test_semi_scan_gpu.py tests/test_segments_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -3
