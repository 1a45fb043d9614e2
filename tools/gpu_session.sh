cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_semimarkov_gpu.py -x -q --timeout=900 > $O/sm_tests.log 2>&1; echo "rc=$?" >> $O/sm_tests.log
timeout 600 python -c "
import numpy as np, torch, paper_2002_00876_b200 as tsb
sm = torch.from_numpy(np.random.default_rng(0).standard_normal((32, 24, 4, 20, 20)).astype(np.float32)).cuda()
def t(f):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/20
print('marg', t(lambda: tsb.semimarkov(sm)))
print('nomarg', t(lambda: tsb.semimarkov(sm, want_marg=False)))
print('vit', t(lambda: tsb.semimarkov_viterbi(sm)))
" > $O/sm_time.log 2>&1
