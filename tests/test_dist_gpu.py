"""GPU parity of the distribution properties (§3
P:113-123, Table 2): entropy, expectation, log_prob / score and FFBS sampling through the C ABI, against the
fp64 oracle (oracle.chain_entropy / chain_log_prob / ffbs_sample, pinned in
tests/test_oracle_dist_pins.py).

Gates (readings R13-R15):
  entropy   |dH| <= 1e-5 * max(1, |A|)   (H = A - E_p[Score]; both terms are O(|A|))
  log_prob  |d log p| <= 1e-5 * max(1, |A|)
  sampling  exact paths equal the oracle's for the same uniforms except where the oracle's
            own inverse-CDF decision is within 1e-4 (relative) of a boundary; empirical
            frequencies match enumeration (TV < 0.02).
"""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_2002_00876_b200 as tsb
import tsgen
from _util import check_logz
from oracle import brute

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _dev(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def _check_rel(gpu, ref, A):
    gpu = np.asarray(gpu, np.float64)
    for b in range(len(ref)):
        if math.isnan(ref[b]):
            assert math.isnan(gpu[b]), (b, gpu[b])
        else:
            assert abs(gpu[b] - ref[b]) <= TOL * max(1.0, abs(A[b])), (b, gpu[b], ref[b])


SHAPES = [(1, 5, 3), (32, 25, 20), (5, 25, 7), (3, 130, 64), (2, 41, 128), (2, 300, 20),
          (2, 80, 100)]


@pytest.mark.parametrize("B,N,C", SHAPES)
def test_entropy_parity(dev, B, N, C):
    pot = tsgen.potentials(B, N, C, seed=4000 + N + C)
    H_ref, lz_ref, fl_ref = oracle.chain_entropy(pot, threads=8)
    H, marg, lz, fl = tsb.entropy(_dev(pot, dev))
    check_logz(lz.cpu().numpy(), lz_ref)
    assert (fl.cpu().numpy().astype(np.uint32) == fl_ref).all()
    _check_rel(H.cpu().numpy(), H_ref, lz_ref)


def test_entropy_lengths_flags_masks(dev):
    for (B, N, C) in [(8, 25, 20), (6, 60, 64), (5, 12, 3)]:
        pot = tsgen.tagging_potentials(B, N, C, seed=C, mask_frac=0.2)
        lengths = tsgen.random_lengths(B, N, C)
        lengths[0], lengths[1] = 1, N
        pot[2] = -np.inf
        lengths[2] = N
        pot[3, 0, 0, 0] = np.nan
        lengths[3] = N
        lengths[4] = 0
        H_ref, lz_ref, fl_ref = oracle.chain_entropy(pot, lengths, threads=8)
        H, _, lz, fl = tsb.entropy(_dev(pot, dev), _dev(lengths, dev))
        assert (fl.cpu().numpy().astype(np.uint32) == fl_ref).all()
        _check_rel(H.cpu().numpy(), H_ref, np.nan_to_num(lz_ref, nan=1.0, neginf=1.0))


def test_entropy_closed_form_uniform(dev):
    N, C = 25, 20
    H, _, _, _ = tsb.entropy(torch.zeros((4, N - 1, C, C), device=dev))
    assert np.allclose(H.cpu().numpy(), N * math.log(C), rtol=1e-6)


@pytest.mark.parametrize("B,N,C", SHAPES)
def test_expectation_parity(dev, B, N, C):
    """Table 2 'Exp.': Σ mu·r against oracle.chain_expectation (pinned by
    enumeration); gate |dE| <= 1e-5 * max(1, Σ|mu·r|-scale) with the scale = len - 1."""
    pot = tsgen.potentials(B, N, C, seed=4500 + N + C)
    r = np.random.default_rng(N + 3 * C).standard_normal(pot.shape).astype(np.float32)
    ref, lz_ref, fl_ref = oracle.chain_expectation(pot, r, threads=8)
    ev, marg, lz, fl = tsb.expectation(_dev(pot, dev), _dev(r, dev))
    check_logz(lz.cpu().numpy(), lz_ref)
    assert (fl.cpu().numpy().astype(np.uint32) == fl_ref).all()
    _check_rel(ev.cpu().numpy(), ref, np.full(B, float(N - 1)))


def test_expectation_lengths_flags_closed_form(dev):
    B, N, C = 6, 40, 20
    pot = tsgen.tagging_potentials(B, N, C, seed=12, mask_frac=0.2)
    lengths = tsgen.random_lengths(B, N, C)
    lengths[0], lengths[1] = 1, N
    pot[2] = -np.inf
    lengths[2] = N
    lengths[3] = 0
    ones = np.ones_like(pot)
    ref, _, fl_ref = oracle.chain_expectation(pot, ones, lengths, threads=8)
    ev, _, _, fl = tsb.expectation(_dev(pot, dev), _dev(ones, dev), _dev(lengths, dev))
    assert (fl.cpu().numpy().astype(np.uint32) == fl_ref).all()
    ev = ev.cpu().numpy()
    _check_rel(ev, ref, np.full(B, float(N)))
    for b in (0, 1, 4, 5):   # r = 1 counts the edges: len - 1
        assert abs(ev[b] - (lengths[b] - 1)) <= 1e-5 * max(1, lengths[b]), (b, ev[b])
    # r = l: E_p[Score] = A - H
    pot = tsgen.potentials(4, 25, 20, seed=2)
    H, _, lz, _ = tsb.entropy(_dev(pot, dev))
    es, _, _, _ = tsb.expectation(_dev(pot, dev), _dev(pot, dev))
    assert float((es.double() - (lz.double() - H.double())).abs().max()) <= 1e-5 * float(lz.abs().max())


@pytest.mark.parametrize("B,N,C", SHAPES)
def test_log_prob_parity(dev, B, N, C):
    pot = tsgen.potentials(B, N, C, seed=5000 + N + C)
    rng = np.random.default_rng(N + C)
    z = rng.integers(0, C, size=(B, N)).astype(np.int32)
    ref = oracle.chain_log_prob(pot, z, threads=8)
    lz_ref, _, _ = oracle.chain_marginals(pot, want_marg=False, threads=8)
    out = tsb.log_prob(_dev(pot, dev), _dev(z, dev))
    _check_rel(out.cpu().numpy(), ref, lz_ref)
    # the Viterbi path: Score(z*) = A* exactly (dyadic inputs)
    path, score, _ = tsb.viterbi(_dev(pot, dev))
    sc = tsb.score(_dev(pot, dev), path)
    assert torch.equal(sc, score)


def test_log_prob_bad_labels_and_lengths(dev):
    B, N, C = 4, 10, 5
    pot = tsgen.potentials(B, N, C, seed=3)
    z = np.zeros((B, N), np.int32)
    z[0, 3] = C           # bad label on a used position -> NaN
    z[1, 8] = -1          # beyond len -> ignored
    lengths = np.array([N, 6, 1, N], np.int32)
    ref = oracle.chain_log_prob(pot, z, lengths)
    out = tsb.log_prob(_dev(pot, dev), _dev(z, dev), _dev(lengths, dev)).cpu().numpy()
    assert math.isnan(out[0]) and math.isnan(ref[0])
    for b in (1, 2, 3):
        assert abs(out[b] - ref[b]) <= TOL * max(1.0, abs(ref[b])), (b, out[b], ref[b])


def test_sampling_frequencies_match_enumeration(dev):
    N, C, K = 3, 3, 200000
    pot = tsgen.potentials(2, N, C, seed=11, s=6)
    u = torch.rand((K, 2, N), generator=torch.Generator().manual_seed(5)).to(dev)
    z, _, _ = tsb.sample(_dev(pot, dev), u)
    z = z.cpu().numpy()
    for b in range(2):
        Z, p = brute.probabilities(pot[b], N)
        code = (z[:, b, :] * np.array([1, C, C * C])).sum(axis=1)
        freq = np.bincount(code, minlength=C ** N) / K
        codes_enum = (Z * np.array([1, C, C * C])).sum(axis=1)
        tv = 0.5 * np.abs(freq[codes_enum] - p).sum()
        assert tv < 0.02, tv


def _oracle_margin(pot_seq, n, zpath, u, t):
    """Relative distance of u*total to the nearest CDF boundary of the oracle's draw at t."""
    al = oracle.forward_alpha(np.asarray(pot_seq, np.float64), n)
    lw = al[n - 1] if t == n - 1 else al[t] + np.asarray(pot_seq, np.float64)[t, :, zpath[t + 1]]
    p = np.exp(lw - lw.max())
    c = np.cumsum(p)
    return float(np.min(np.abs(c - u * c[-1])) / c[-1])


@pytest.mark.parametrize("B,N,C", [(3, 40, 20), (2, 60, 64), (2, 30, 128), (4, 25, 7),
                                   (2, 30, 200), (2, 20, 256), (2, 15, 131)])
def test_sampling_matches_oracle_paths(dev, B, N, C):
    K = 8
    pot = tsgen.potentials(B, N, C, seed=6000 + N + C)
    u = np.random.default_rng(N * C).random((K, B, N)).astype(np.float32)
    ref = oracle.ffbs_sample(pot, u.astype(np.float64))
    z, lz, fl = tsb.sample(_dev(pot, dev), _dev(u, dev))
    z = z.cpu().numpy()
    lz_ref, _, _ = oracle.chain_marginals(pot, want_marg=False)
    check_logz(lz.cpu().numpy(), lz_ref)
    same = 0
    for k in range(K):
        for b in range(B):
            if np.array_equal(z[k, b], ref[k, b]):
                same += 1
                continue
            t = max(i for i in range(N) if z[k, b, i] != ref[k, b, i])  # first from the end
            m = _oracle_margin(pot[b], N, ref[k, b], float(u[k, b, t]), t)
            assert m < 1e-4, (k, b, t, m)
    assert same >= 0.9 * K * B, same


def test_sampling_wide_labels_lengths_flags(dev):
    """128 < C <= 256 (forward filtering through the wide-label recursion): lengths, len 1,
    EMPTY and BADLEN rows behave as for narrow labels."""
    B, N, C = 5, 12, 160
    pot = tsgen.potentials(B, N, C, seed=18)
    lengths = np.array([N, 1, 5, 0, N], np.int32)
    pot[4] = -np.inf
    u = np.random.default_rng(3).random((3, B, N)).astype(np.float32)
    z, lz, fl = tsb.sample(_dev(pot, dev), _dev(u, dev), _dev(lengths, dev))
    z = z.cpu().numpy()
    ref = oracle.ffbs_sample(pot, u.astype(np.float64), lengths)
    assert (z[:, 3] == -1).all() and (z[:, 4] == -1).all()
    assert (z[:, 2, 5:] == -1).all() and (z[:, 1, 1:] == -1).all()
    np.testing.assert_array_equal(z[:, 1, 0], ref[:, 1, 0])
    assert (fl.cpu().numpy()[[3, 4]] != 0).all()
    lz_ref, _, _ = oracle.chain_marginals(pot, lengths, want_marg=False)
    check_logz(lz.cpu().numpy()[[0, 1, 2]], lz_ref[[0, 1, 2]])


def test_sampling_lengths_flags(dev):
    B, N, C = 5, 12, 6
    pot = tsgen.potentials(B, N, C, seed=8)
    lengths = np.array([N, 1, 5, 0, N], np.int32)
    pot[4] = -np.inf
    u = np.random.default_rng(2).random((3, B, N)).astype(np.float32)
    z, _, fl = tsb.sample(_dev(pot, dev), _dev(u, dev), _dev(lengths, dev))
    z = z.cpu().numpy()
    ref = oracle.ffbs_sample(pot, u.astype(np.float64), lengths)
    assert (z[:, 3] == -1).all() and (z[:, 4] == -1).all()
    assert (z[:, 2, 5:] == -1).all() and (z[:, 1, 1:] == -1).all()
    np.testing.assert_array_equal(z[:, 1, 0], ref[:, 1, 0])  # len 1: uniform draw
    assert (fl.cpu().numpy()[[3, 4]] != 0).all()


def test_new_ops_deterministic_bitwise(dev):
    """Identical inputs give bit-identical outputs for every §8(f) entry point."""
    pot = torch.from_numpy(tsgen.potentials(6, 40, 20, seed=13)).to(dev)
    u = torch.rand((3, 6, 40), generator=torch.Generator().manual_seed(1)).to(dev)
    z = torch.randint(0, 20, (6, 40), generator=torch.Generator().manual_seed(2)).to(torch.int32).to(dev)
    sm = torch.from_numpy(np.random.default_rng(3).standard_normal((3, 19, 4, 12, 12)).astype(
        np.float32)).to(dev)
    runs = []
    for _ in range(2):
        H, _, _, _ = tsb.entropy(pot)
        ex, _, _, _ = tsb.expectation(pot, pot * 0.5 + 1.0)
        lp = tsb.log_prob(pot, z)
        zz, _, _ = tsb.sample(pot, u)
        kp, ks, _ = tsb.kbest(pot, 5)
        mg, lz, _ = tsb.semimarkov(sm)
        sg, ss, _ = tsb.semimarkov_viterbi(sm)
        runs.append([x.clone() for x in (H, ex, lp, zz, kp, ks, mg, lz, sg, ss)])
    for a, b in zip(*runs):
        assert torch.equal(a, b)
