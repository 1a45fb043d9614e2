cd $GRAFT_REPO_ROOT
O=gpurun_out
./tools/mufu_peak > $O/mufu.jsonl 2>&1
nvidia-smi --query-gpu=clocks.sm --format=csv >> $O/mufu.jsonl 2>&1
