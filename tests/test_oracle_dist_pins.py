"""Pins for the oracle's distribution properties (entropy,
expectation of an additive feature, density / log_prob, forward-filtering backward-sampling; §3, Table 2
P:202-206) against things other than the oracle itself: brute-force enumeration of
every labelling (P:149 footnote), closed forms of the definitions, and exact sampling
frequencies.  A plausible bug (sign of the expectation term, conditioning on the wrong
neighbour, an off-by-one position, a transposed tile) fails at least one test here.
"""
import math

import numpy as np
import pytest

import oracle
import tsgen
from oracle import brute

CASES = [(1, 5, 3), (3, 2, 2), (2, 3, 4), (2, 6, 3), (1, 4, 6), (1, 1, 5)]


@pytest.mark.parametrize("B,N,C", CASES)
def test_entropy_matches_enumeration(B, N, C):
    pot = tsgen.potentials(B, N, C, seed=2000 + 7 * N + C, s=8)
    H, logz, flags = oracle.chain_entropy(pot)
    assert (flags == 0).all()
    for b in range(B):
        assert abs(H[b] - brute.entropy(pot[b], N)) <= 1e-10 * max(1.0, abs(H[b]))


def test_entropy_masked_and_lengths():
    B, N, C = 4, 6, 3
    pot = tsgen.tagging_potentials(B, N, C, seed=5, mask_frac=0.3)
    lengths = np.array([6, 3, 1, 5], dtype=np.int32)
    H, _, flags = oracle.chain_entropy(pot, lengths)
    for b in range(B):
        n = int(lengths[b])
        assert abs(H[b] - brute.entropy(pot[b], n)) <= 1e-10 * max(1.0, abs(H[b]))
    assert H[2] == pytest.approx(math.log(C), abs=1e-12)  # len 1: uniform over C labels


def test_entropy_closed_forms():
    # l = 0: p uniform over C^n labelings -> H = n ln C
    for (N, C) in [(25, 20), (200, 7)]:
        H, _, _ = oracle.chain_entropy(np.zeros((1, N - 1, C, C), np.float32))
        assert H[0] == pytest.approx(N * math.log(C), rel=1e-12)
    # separable l[t,i,j] = phi_t[j]: z_0 uniform, z_{t+1} ~ softmax(phi_t) independently
    rng = np.random.default_rng(3)
    N, C = 50, 9
    phi = rng.standard_normal((N - 1, C)).astype(np.float32)
    pot = np.broadcast_to(phi[:, None, :], (N - 1, C, C)).astype(np.float32)[None]
    H, _, _ = oracle.chain_entropy(pot)
    ref = math.log(C)
    for t in range(N - 1):
        p = np.exp(phi[t].astype(np.float64) - phi[t].max())
        p /= p.sum()
        ref -= float(np.sum(p * np.log(p)))
    assert H[0] == pytest.approx(ref, rel=1e-12)


def test_entropy_flags():
    pot = tsgen.potentials(3, 5, 3, seed=1)
    pot[0] = -np.inf
    pot[1, 2, 0, 0] = np.nan
    H, _, flags = oracle.chain_entropy(pot)
    assert math.isnan(H[0]) and math.isnan(H[1]) and not math.isnan(H[2])
    assert flags[0] == oracle.F_EMPTY and flags[1] == oracle.F_NONFINITE


@pytest.mark.parametrize("B,N,C", CASES)
def test_expectation_matches_enumeration(B, N, C):
    """Table 2 'Exp.': E_p[Σ_t r_t(z_t, z_{t+1})] against Σ_z p(z) f(z)."""
    pot = tsgen.potentials(B, N, C, seed=2500 + 7 * N + C, s=8)
    r = np.random.default_rng(N * C).standard_normal(pot.shape).astype(np.float32)
    ev, _, flags = oracle.chain_expectation(pot, r)
    assert (flags == 0).all()
    for b in range(B):
        assert abs(ev[b] - brute.expectation(pot[b], r[b], N)) <= 1e-10 * max(1.0, abs(ev[b]))


def test_expectation_masked_lengths_and_garbage_at_masks():
    B, N, C = 4, 6, 3
    pot = tsgen.tagging_potentials(B, N, C, seed=9, mask_frac=0.3)
    lengths = np.array([6, 4, 1, 5], dtype=np.int32)
    r = np.random.default_rng(1).standard_normal(pot.shape).astype(np.float32)
    r2 = r.copy()
    r2[np.isneginf(pot)] = np.nan            # r at masked parts (mu = 0) never matters
    r2[1, 3:] = np.inf                       # nor beyond the sequence
    ev, _, _ = oracle.chain_expectation(pot, r, lengths)
    ev2, _, _ = oracle.chain_expectation(pot, r2, lengths)
    for b in range(B):
        n = int(lengths[b])
        assert abs(ev[b] - brute.expectation(pot[b], r[b], n)) <= 1e-10 * max(1.0, abs(ev[b]))
    assert np.array_equal(ev, ev2)
    assert ev[2] == 0.0                      # len 1: no edges


def test_expectation_closed_forms():
    # r = 1: every labelling has len-1 edges
    pot = tsgen.potentials(2, 30, 7, seed=4)
    ev, _, _ = oracle.chain_expectation(pot, np.ones_like(pot), np.array([30, 11], np.int32))
    assert ev[0] == pytest.approx(29.0, rel=1e-12) and ev[1] == pytest.approx(10.0, rel=1e-12)
    # separable l[t,i,j] = phi_t[j], r[t,i,j] = psi_t[j]: z_{t+1} ~ softmax(phi_t) -> Σ_t <p_t, psi_t>
    rng = np.random.default_rng(8)
    N, C = 40, 6
    phi = rng.standard_normal((N - 1, C)).astype(np.float32)
    psi = rng.standard_normal((N - 1, C)).astype(np.float32)
    pot = np.broadcast_to(phi[:, None, :], (N - 1, C, C)).astype(np.float32)[None]
    r = np.broadcast_to(psi[:, None, :], (N - 1, C, C)).astype(np.float32)[None]
    ev, _, _ = oracle.chain_expectation(pot, r)
    ref = 0.0
    for t in range(N - 1):
        p = np.exp(phi[t].astype(np.float64) - phi[t].max())
        ref += float(np.sum(p / p.sum() * psi[t]))
    assert ev[0] == pytest.approx(ref, rel=1e-12)
    # an indicator feature picks out one marginal: E[z_p] = p(z_p = 1) (Table 2)
    pot = tsgen.potentials(1, 5, 3, seed=6, s=8)
    r = np.zeros_like(pot)
    r[0, 2, 1, 0] = 1.0
    ev, _, _ = oracle.chain_expectation(pot, r)
    Z, p = brute.probabilities(pot[0], 5)
    assert ev[0] == pytest.approx(float(p[(Z[:, 2] == 1) & (Z[:, 3] == 0)].sum()), abs=1e-12)


@pytest.mark.parametrize("B,N,C", CASES)
def test_log_prob_matches_enumeration_and_normalises(B, N, C):
    pot = tsgen.potentials(B, N, C, seed=3000 + N + C, s=8)
    for b in range(B):
        Z, p = brute.probabilities(pot[b], N)
        z = np.broadcast_to(np.zeros((1, N), np.int32), (B, N)).copy()
        lp_all = []
        for zz in Z:
            z[b] = zz
            lp_all.append(oracle.chain_log_prob(pot, z)[b])
        lp_all = np.array(lp_all)
        np.testing.assert_allclose(lp_all, np.log(p), rtol=0, atol=1e-10)
        assert math.fsum(np.exp(lp_all).tolist()) == pytest.approx(1.0, abs=1e-12)


def test_score_paper_two_edge_example_and_bad_labels():
    # Score of z = (c1, c2, c3) is l_{1,c1,c2} + l_{2,c2,c3}
    pot = tsgen.potentials(1, 3, 4, seed=9, s=8)
    z = np.array([[3, 1, 2]], np.int32)
    assert oracle.chain_score(pot, z)[0] == float(pot[0, 0, 3, 1]) + float(pot[0, 1, 1, 2])
    z_bad = np.array([[3, 4, 2]], np.int32)
    assert math.isnan(oracle.chain_score(pot, z_bad)[0])
    # positions beyond len are ignored
    z_tail = np.array([[3, 1, -7]], np.int32)
    assert oracle.chain_score(pot, z_tail, np.array([2], np.int32))[0] == float(pot[0, 0, 3, 1])


def test_forward_alpha_gives_logz():
    pot = tsgen.potentials(2, 30, 5, seed=4)
    logz, _, _ = oracle.chain_marginals(pot)
    for b in range(2):
        al = oracle.forward_alpha(pot[b], 30)
        m = al[-1].max()
        assert m + math.log(np.exp(al[-1] - m).sum()) == pytest.approx(logz[b], rel=1e-13)


def test_ffbs_frequencies_match_enumeration():
    """Exact sampling: empirical frequencies of 60k draws vs p(z) by enumeration (TV < 0.02,
    SURVEY §8(f) f2) for a 3-position, 3-label chain (27 labelings)."""
    N, C, K = 3, 3, 60000
    pot = tsgen.potentials(1, N, C, seed=11, s=6)
    rng = np.random.default_rng(12)
    u = rng.random((K, 1, N))
    z = oracle.ffbs_sample(pot, u)[:, 0, :]
    Z, p = brute.probabilities(pot[0], N)
    code = (z * np.array([1, C, C * C])).sum(axis=1)
    freq = np.bincount(code, minlength=C ** N) / K
    codes_enum = (Z * np.array([1, C, C * C])).sum(axis=1)
    tv = 0.5 * np.abs(freq[codes_enum] - p).sum()
    assert tv < 0.02, tv


def test_ffbs_inverse_cdf_and_conditioning():
    """Deterministic structure: u -> 0 picks the first label with nonzero probability,
    u -> 1 the last; a chain whose edges force z_{t} = z_{t+1} (identity-like potentials)
    yields constant paths; masked labels are never drawn."""
    C, N = 4, 6
    pot = np.full((1, N - 1, C, C), -np.inf, np.float32)
    for t in range(N - 1):
        np.fill_diagonal(pot[0, t], 0.0)  # only z_t = z_{t+1} allowed
    u = np.random.default_rng(1).random((200, 1, N))
    z = oracle.ffbs_sample(pot, u)[:, 0, :]
    assert (z == z[:, :1]).all()
    lo = oracle.ffbs_sample(pot, np.zeros((1, 1, N)))[0, 0]
    hi = oracle.ffbs_sample(pot, np.full((1, 1, N), 1 - 1e-12))[0, 0]
    assert (lo == 0).all() and (hi == C - 1).all()
    # lengths: -1 beyond len; len 1 -> z_0 uniform over C
    pot2 = tsgen.potentials(2, N, C, seed=3)
    z2 = oracle.ffbs_sample(pot2, np.full((1, 2, N), 0.6), np.array([N, 1], np.int32))
    assert (z2[0, 1, 1:] == -1).all() and z2[0, 1, 0] == 2  # floor(0.6 * 4)


# ---------------------------------------------------------------- f3: K-Max (k-best)

@pytest.mark.parametrize("B,N,C,K", [(2, 4, 3, 5), (1, 5, 3, 243), (2, 3, 4, 7), (1, 1, 4, 6),
                                     (2, 6, 2, 10)])
def test_kbest_matches_enumeration(B, N, C, K):
    # coarse dyadic values: many exact ties, so the tie order is exercised
    pot = (np.random.default_rng(N * C + K).integers(-2, 3, size=(B, N - 1, C, C)) * 0.5
           ).astype(np.float32)
    paths, scores, flags = oracle.chain_kbest(pot, K)
    for b in range(B):
        Zr, sr = brute.kbest(pot[b], N, K)
        m = len(sr)
        np.testing.assert_array_equal(paths[b, :m], Zr)
        np.testing.assert_array_equal(scores[b, :m], sr)
        assert (scores[b, m:] == -np.inf).all() and (paths[b, m:] == -1).all()


def test_kbest_k1_is_viterbi_and_zero_potentials():
    pot = tsgen.potentials(3, 30, 6, seed=2, s=8)
    paths, scores, _ = oracle.chain_kbest(pot, 1)
    p_ref, s_ref, _ = oracle.chain_viterbi(pot)
    np.testing.assert_array_equal(paths[:, 0], p_ref)
    np.testing.assert_array_equal(scores[:, 0], s_ref)
    # l = 0: every labelling scores 0; the order is reverse-lexicographic (z_{n-1} most
    # significant), so the q-th labelling is q written in base C with z_0 the lowest digit
    N, C, K = 4, 3, 10
    paths, scores, _ = oracle.chain_kbest(np.zeros((1, N - 1, C, C), np.float32), K)
    assert (scores == 0).all()
    q = np.arange(K)
    ref = np.stack([(q // C ** p) % C for p in range(N)], axis=1)
    np.testing.assert_array_equal(paths[0], ref)


def test_kbest_lengths_and_flags():
    pot = tsgen.potentials(4, 6, 3, seed=5, s=8)
    pot[2] = -np.inf
    pot[3, 1, 0, 0] = np.nan
    lengths = np.array([6, 2, 6, 6], np.int32)
    paths, scores, flags = oracle.chain_kbest(pot, 4, lengths)
    Zr, sr = brute.kbest(pot[1], 2, 4)
    np.testing.assert_array_equal(paths[1, :, :2], Zr)
    assert (paths[1, :, 2:] == -1).all()
    assert (scores[2] == -np.inf).all() and (paths[2] == -1).all()
    assert np.isnan(scores[3]).all() and (paths[3] == -1).all()
    assert flags[2] == oracle.F_EMPTY and flags[3] == oracle.F_NONFINITE


# ---------------------------------------------------------------- f4: semi-Markov (R17)

@pytest.mark.parametrize("N,K,C", [(5, 2, 2), (4, 3, 3), (6, 3, 2), (3, 1, 3), (5, 4, 2), (1, 2, 3)])
def test_semimarkov_matches_enumeration(N, K, C):
    rng = np.random.default_rng(N * 100 + K * 10 + C)
    pot = (rng.integers(-64, 65, size=(2, max(N - 1, 0), K, C, C)) / 32.0).astype(np.float32)
    logz, marg, flags = oracle.semimarkov_marginals(pot)
    assert (flags == 0).all()
    for b in range(2):
        A, mu = brute.semimarkov(pot[b], N)
        assert abs(logz[b] - A) <= 1e-12 * max(1.0, abs(A))
        np.testing.assert_allclose(marg[b], mu, rtol=0, atol=1e-12)


def test_semimarkov_k1_is_the_linear_chain():
    pot = tsgen.potentials(3, 20, 5, seed=8)
    lz, mg, _ = oracle.chain_marginals(pot)
    lz2, mg2, _ = oracle.semimarkov_marginals(pot[:, :, None, :, :])
    np.testing.assert_allclose(lz2, lz, rtol=1e-13)
    np.testing.assert_allclose(mg2[:, :, 0], mg, atol=1e-13)


def test_semimarkov_count_compositions_and_coverage():
    # C = 1, l = 0: A = log(#compositions of E into parts <= K) (E=4, K=2 -> 5)
    for (E, K, cnt) in [(4, 2, 5), (3, 3, 4), (10, 3, 274)]:
        lz, _, _ = oracle.semimarkov_marginals(np.zeros((1, E, K, 1, 1), np.float32))
        assert lz[0] == pytest.approx(math.log(cnt), rel=1e-13)
    # every step is covered by exactly one segment: Σ mu * k = E_b
    pot = (np.random.default_rng(4).standard_normal((2, 12, 4, 3, 3))).astype(np.float32)
    lengths = np.array([13, 7], np.int32)
    _, mu, _ = oracle.semimarkov_marginals(pot, lengths)
    ks = np.arange(1, 5)[None, None, :, None, None]
    for b in range(2):
        assert float((mu[b] * ks[0]).sum()) == pytest.approx(lengths[b] - 1, rel=1e-12)


def test_semimarkov_finite_differences_and_flags():
    pot = (np.random.default_rng(5).standard_normal((1, 6, 3, 2, 2))).astype(np.float64)
    _, mu, _ = oracle.semimarkov_marginals(pot)
    h = 2.0 ** -13
    rng = np.random.default_rng(6)
    for _ in range(8):
        q = tuple(rng.integers(0, s) for s in pot.shape)
        if q[1] + q[2] + 1 > 6:
            continue
        pp, pm = pot.copy(), pot.copy()
        pp[q] += h
        pm[q] -= h
        fd = (oracle.semimarkov_marginals(pp, want_marg=False)[0][0] -
              oracle.semimarkov_marginals(pm, want_marg=False)[0][0]) / (2 * h)
        assert fd == pytest.approx(mu[q], abs=1e-7)
    bad = (np.random.default_rng(7).standard_normal((3, 5, 2, 2, 2))).astype(np.float32)
    bad[0] = -np.inf
    bad[1, 1, 0, 1, 1] = np.nan
    lz, mg, fl = oracle.semimarkov_marginals(bad)
    assert fl[0] == oracle.F_EMPTY and lz[0] == -np.inf and (mg[0] == 0).all()
    assert fl[1] == oracle.F_NONFINITE and math.isnan(lz[1])
    assert fl[2] == 0


@pytest.mark.parametrize("N,K,C,s", [(5, 3, 2, 1), (6, 2, 3, 1), (4, 4, 3, 0), (7, 3, 2, 2),
                                     (1, 2, 3, 1), (2, 1, 3, 1)])
def test_semimarkov_viterbi_matches_enumeration(N, K, C, s):
    """Semi-Markov Viterbi (R17/R18) against the canonical enumerated argmax; coarse dyadic
    values (2^-s grid) so ties are frequent and the tie rule is exercised."""
    rng = np.random.default_rng(100 * N + 10 * K + C + s)
    B = 6
    pot = (rng.integers(-3, 4, size=(B, N - 1, K, C, C)) * 2.0 ** -s).astype(np.float32)
    pot[1, ..., 0, :] = -np.inf if N > 1 else 0.0      # masked transitions out of label 0
    seg, score, flags = oracle.semimarkov_viterbi(pot)
    for b in range(B):
        ref_seg, ref = brute.semimarkov_argmax(pot[b], N)
        assert score[b] == ref and np.array_equal(seg[b], ref_seg), (b, seg[b], ref_seg)


def test_semimarkov_viterbi_k1_is_chain_viterbi_and_flags():
    pot = tsgen.potentials(4, 12, 5, seed=3, s=8)
    lengths = np.array([12, 7, 1, 12], np.int32)
    seg, score, flags = oracle.semimarkov_viterbi(pot[:, :, None], lengths)
    path, sc, fl = oracle.chain_viterbi(pot, lengths)
    assert np.array_equal(seg, path) and np.array_equal(score, sc) and (flags == fl).all()
    bad = tsgen.potentials(4, 6, 3, seed=1)[:, :, None].repeat(2, axis=2)
    bad[0] = -np.inf
    bad[1, 2, 0, 0, 0] = np.nan
    seg, score, flags = oracle.semimarkov_viterbi(bad, np.array([6, 6, 0, 6], np.int32))
    assert list(flags[:3]) == [oracle.F_EMPTY, oracle.F_NONFINITE, oracle.F_BADLEN]
    assert score[0] == -np.inf and math.isnan(score[1]) and math.isnan(score[2])
    assert (seg[:3] == -1).all() and flags[3] == 0
