cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_dist_gpu.py -x -q --timeout=900 > $O/samp_tests.log 2>&1; echo "rc=$?" >> $O/samp_tests.log
timeout 600 python tools/bench_ops.py --iters 5 > $O/ops9.jsonl 2> $O/ops9.err
timeout 600 compute-sanitizer --tool racecheck python -c "
import numpy as np, torch, paper_2002_00876_b200 as tsb, tsgen
pot = torch.from_numpy(tsgen.potentials(3, 30, 20, seed=1)).cuda()
tsb.sample(pot, torch.rand((11, 3, 30), device='cuda')); torch.cuda.synchronize(); print('ok')" > $O/samp_race.log 2>&1
