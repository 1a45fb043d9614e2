#!/bin/bash
# Profiling recipe (B200_PROFILING.md) for the bench workload; run under gpurun.
# 1) launch list of the timed kernels (cold-cache, serialised: compare SHARES, not absolutes)
# 2) one --set full capture of the dominant kernel
set -x
CFG=${1:-2}
OUT=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'fb_|sweep|viterbi|backtrack|indicator|summary|tree' \
    -c 60 --csv --log-file $OUT/launches_cfg$CFG.csv \
    python bench.py --config $CFG --steps 20 --warmup 5 --mode eager --no-cpu-baseline --e2e-steps 3 > $OUT/launches_cfg$CFG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"${2:-fb_small}" -s 10 -c 1 -f \
    -o $OUT/prof_cfg$CFG python bench.py --config $CFG --steps 20 --warmup 5 --mode eager --no-cpu-baseline --e2e-steps 3 > $OUT/prof_cfg$CFG.log 2>&1
ls -la $OUT
