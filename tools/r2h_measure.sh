# Round-2 final measurement session (one gpurun call): bench line (both arms), side ops,
# cfg5 Viterbi plans, launch list + one ncu --set full capture of the headline kernel.
cd $GRAFT_REPO_ROOT; O=gpurun_out; T=${1:-r2h}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${T}_gpu.txt 2>&1
timeout 600 python bench.py > $O/${T}_bench.json 2>$O/${T}_bench.err
timeout 300 python bench.py --impl reference > $O/${T}_ref.json 2>>$O/${T}_bench.err
timeout 600 python tools/bench_ops.py > $O/${T}_ops.jsonl 2>$O/${T}_ops.err
timeout 900 python tools/cfg5_viterbi_time.py > $O/${T}_cfg5_viterbi.jsonl 2>$O/${T}_cfg5v.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fb_|meet|summary|tree|fwd|bwd|vit|backtrack|segment" -c 60 --csv \
  --log-file $O/${T}_launches_cfg2.csv python bench.py --steps 20 --warmup 3 --reps 0 --side "" \
  --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fb_tiny -s 10 -c 1 \
  -o $O/${T}_full_fb_tiny -f python bench.py --steps 20 --warmup 3 --reps 0 --side "" \
  --no-cpu-baseline --e2e-steps 1 > $O/${T}_ncu_full.log 2>&1
echo done
