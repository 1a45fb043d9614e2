"""Single-GPU time-chunked Viterbi (vchunk.cu; SURVEY §8(a) a7's chunked variant, the Max
semiring of Table 2 P:200 on the §6(a) scan P:307-311; C <= 158, two staged C x C tiles per
CTA; wider labels keep the serial sweep): plan invariance — the path and score
are bit-identical to the fp64 oracle (and to the serial kernels) for every chunk length,
L in {1, 7, 64, E}, including L = 1 (every edge its own chunk: the pure Fig. 4 leaves) —
with frequent exact ties (coarse dyadic inputs), variable lengths and flagged sequences.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2002_00876_b200 as tsb
import tsgen

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _reset():
    yield
    tsb.set_plan_chunk(0)


def run(pot_np, lengths_np, dev, L):
    tsb.set_plan_chunk(L)
    pot = torch.from_numpy(np.ascontiguousarray(pot_np)).to(dev)
    lengths = (torch.from_numpy(lengths_np.astype(np.int32)).to(dev)
               if lengths_np is not None else None)
    path, score, flags = tsb.viterbi(pot, lengths)
    kern = tsb.last_kernel()
    return path.cpu().numpy(), score.cpu().numpy(), flags.cpu().numpy().astype(np.uint32), kern


def check(pot_np, lengths_np, dev, Ls):
    p_ref, s_ref, f_ref = oracle.chain_viterbi(pot_np, lengths_np, threads=8)
    E = pot_np.shape[1]
    for L in Ls:
        path, score, flags, kern = run(pot_np, lengths_np, dev, L)
        C = pot_np.shape[-1]
        if 1 <= L < E and E >= 2 and C <= 128:  # two staged tiles fit in SMEM
            want = "vch_summary_mm_kernel" if C in (32, 64, 128) else "vch_summary_kernel"
            assert kern == want, (L, kern)
        np.testing.assert_array_equal(flags, f_ref, err_msg=f"L={L}")
        np.testing.assert_array_equal(path, p_ref, err_msg=f"L={L}")
        ok = f_ref == 0
        assert (score[ok] == s_ref[ok].astype(np.float32)).all(), L


@pytest.mark.parametrize("B,N,C", [(3, 65, 20), (2, 200, 37), (2, 129, 128), (1, 40, 256), (4, 9, 3)])
def test_plan_invariance_dyadic(dev, B, N, C):
    pot = tsgen.potentials(B, N, C, seed=1000 + N + C, s=tsgen.quantum(N - 1))
    check(pot, None, dev, [1, 7, 64, N - 1])


@pytest.mark.parametrize("C", [4, 20, 128])
def test_plan_invariance_ties(dev, C):
    """Coarse integer potentials: many exactly tied paths; the smallest-index rule (reading
    R5) must survive the chunk boundaries."""
    rng = np.random.default_rng(C)
    pot = (rng.integers(-2, 3, size=(3, 50, C, C)) * 0.5).astype(np.float32)
    check(pot, None, dev, [1, 3, 7, 49])


def test_lengths_and_flags(dev):
    B, N, C = 8, 41, 12
    pot = tsgen.potentials(B, N, C, seed=5, s=tsgen.quantum(N - 1))
    lengths = np.array([1, 2, 17, 41, 41, 30, 0, 41], dtype=np.int32)
    pot[3] = -np.inf                  # EMPTY
    pot[4, 11, 2, 5] = np.nan         # NONFINITE
    pot[5, 40 - 1, 0, 0] = np.nan     # beyond its length: ignored
    check(pot, lengths, dev, [1, 5, 16, 40])


def test_max_semiring_logz_and_indicator(dev):
    """ts_logpartition(TS_MAX) (summaries + combine only) and ts_marginals(TS_MAX) (the
    one-hot indicator of the chunked path) equal the serial plan's."""
    pot_np = tsgen.potentials(3, 100, 24, seed=9, s=tsgen.quantum(99))
    pot = torch.from_numpy(pot_np).to(dev)
    tsb.set_plan_chunk(0)
    lz0, f0 = tsb.logpartition(pot, semiring="max")
    m0, l0, g0 = tsb.marginals(pot, semiring="max")
    tsb.set_plan_chunk(9)
    lz1, f1 = tsb.logpartition(pot, semiring="max")
    assert tsb.last_kernel() == "vch_summary_kernel"
    m1, l1, g1 = tsb.marginals(pot, semiring="max")
    assert torch.equal(lz0, lz1) and torch.equal(f0, f1)
    assert torch.equal(m0, m1) and torch.equal(l0, l1) and torch.equal(g0, g1)


@pytest.mark.parametrize("C", [32, 64, 128])
def test_mm_summaries_equal_row_chains(dev, C):
    """The register-blocked max-plus summaries (FADD2 + 3-input max over strided 8x8 blocks)
    and the row-chain summaries give the identical path and score (and both the oracle's),
    with ragged lengths, a -inf sequence and NaN potentials."""
    B, N = 3, 150
    pot = tsgen.potentials(B, N, C, seed=77 + C, s=tsgen.quantum(N - 1))
    lengths = np.array([150, 97, 150], dtype=np.int32)
    pot[2, 40, 3, 5] = np.nan
    try:
        for mm in (True, False):
            tsb.set_vchunk_mm(mm)
            if mm:
                check(pot, lengths, dev, [1, 13, 64])
            out = run(pot, lengths, dev, 13)
            assert out[3] == ("vch_summary_mm_kernel" if mm else "vch_summary_kernel")
            if mm:
                ref = out
            else:
                for a, b in zip(ref[:3], out[:3]):
                    np.testing.assert_array_equal(a, b)
    finally:
        tsb.set_vchunk_mm(True)


@pytest.mark.parametrize("B,N,C", [(1, 4097, 64), (2, 2049, 128), (6, 1500, 32)])
def test_auto_plan_chunks_long_chains(dev, B, N, C):
    """With the knob at auto (0), few long chains with C in {32, 64, 128} take the chunked
    scan (abi.cu vit_chunk's calibrated rule) and stay bit-identical to the oracle."""
    pot = tsgen.potentials(B, N, C, seed=31 + N, s=tsgen.quantum(N - 1))
    p_ref, s_ref, f_ref = oracle.chain_viterbi(pot, None, threads=8)
    path, score, flags, kern = run(pot, None, dev, 0)
    assert kern == "vch_summary_mm_kernel", kern
    np.testing.assert_array_equal(flags, f_ref)
    np.testing.assert_array_equal(path, p_ref)
    assert (score == s_ref.astype(np.float32)).all()
