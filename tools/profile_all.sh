#!/bin/bash
# Profiling recipe (B200_PROFILING.md) for every BASELINE config; run under gpurun (1 GPU).
# Launch lists (gpu__time_duration, cold + serialised: compare shares) and one --set full
# capture of each config's dominant kernel(s).
cd $GRAFT_REPO_ROOT
O=gpurun_out
TAG=${1:-r1}
K='regex:fb_|sweep|fwd2|bwd2|meet|vit|backtrack|indicator|summary|tree|segment'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 60 --csv \
    --log-file $O/${TAG}_launches_cfg2.csv \
    python bench.py --config 2 --steps 20 --warmup 5 --mode eager --no-cpu-baseline --e2e-steps 3 > $O/${TAG}_l2.log 2>&1
for c in 3 4 5; do
  ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 80 --csv \
      --log-file $O/${TAG}_launches_cfg$c.csv \
      python tools/bench_configs.py --configs $c --iters 2 > $O/${TAG}_l$c.log 2>&1
done
full() {  # cfg script-args kernel-regex name skip
  ncu --set full --clock-control none --import-source on -k "regex:$3" -s ${5:-0} -c 1 -f \
      -o $O/${TAG}_full_$4 $2 > $O/${TAG}_full_$4.log 2>&1
  ncu -i $O/${TAG}_full_$4.ncu-rep --page raw --csv > $O/${TAG}_full_$4_raw.csv 2>/dev/null
  ncu -i $O/${TAG}_full_$4.ncu-rep --page details --csv > $O/${TAG}_full_$4_details.csv 2>/dev/null
}
full 2 "python bench.py --config 2 --steps 20 --warmup 5 --mode eager --no-cpu-baseline --e2e-steps 3" fb_tiny cfg2_fb_tiny 10
full 3 "python tools/bench_configs.py --configs 3 --iters 2" meet64 cfg3_meet64 1
full 4 "python tools/bench_configs.py --configs 4 --iters 2" vit2 cfg4_vit2 1
for k in summary_tc fwd2 bwd2 tree_up; do
  full 5 "python tools/bench_configs.py --configs 5 --iters 2" $k cfg5_$k 1
done
rm -f $O/*.ncu-rep.tmp
ls -la $O
