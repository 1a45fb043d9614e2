cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python bench.py --config 5 --time-shard --steps 5 --warmup 3 > $O/ts1.json 2> $O/ts1.err
