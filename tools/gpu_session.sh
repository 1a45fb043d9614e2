#!/bin/bash
# One gpurun session: GPU tests, smoke, bench (both arms), launch list + one ncu --set full
# capture of the headline kernel.  Usage: tools/gpu_session.sh <tag>
cd $GRAFT_REPO_ROOT
T=${1:-r2}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${T}_gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --timeout=1500 -p no:cacheprovider > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "rc=$?" >> $O/${T}_smoke.log
timeout 600 python bench.py > $O/${T}_bench.json 2>$O/${T}_bench.err
timeout 300 python bench.py --impl reference > $O/${T}_ref.json 2>>$O/${T}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fb_|meet|summary|tree|fwd|bwd|vit|backtrack|segment" -c 60 --csv \
  --log-file $O/${T}_launches_cfg2.csv python bench.py --steps 20 --warmup 3 --reps 0 --side "" \
  --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fb_tiny -s 10 -c 1 \
  -o $O/${T}_full_fb_tiny -f python bench.py --steps 20 --warmup 3 --reps 0 --side "" \
  --no-cpu-baseline --e2e-steps 1 > $O/${T}_ncu_full.log 2>&1
echo done
