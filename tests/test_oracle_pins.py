"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself.

Each pin cites what fixes the expected value: brute-force enumeration (P:149
footnote), closed forms of the definition, the paper's worked
chain, finite differences of A, the §6(c)
product's reduction to a real matmul, the Fig. 4 tree,
and the golden fixtures under tests/golden/.  A plausible oracle bug (dropped
term, wrong index order, transposed tile, wrong tie rule, off-by-one length)
fails at least one test here.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import tsgen
from oracle import brute

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def dyadic(shape, seed, s=6, lo=-4.0, hi=4.0):
    rng = np.random.default_rng(seed)
    k = rng.integers(int(lo * (1 << s)), int(hi * (1 << s)) + 1, size=shape)
    return (k.astype(np.float32) / np.float32(1 << s)).astype(np.float32)


# ---------------------------------------------------------------- brute force pins

CASES = [(1, 5, 3), (3, 2, 2), (2, 3, 4), (2, 6, 3), (1, 4, 6), (2, 8, 2), (1, 1, 5)]


@pytest.mark.parametrize("B,N,C", CASES)
def test_logz_marginals_match_enumeration(B, N, C):
    pot = tsgen.potentials(B, N, C, seed=1000 + N * 10 + C)
    logz, marg, flags = oracle.chain_marginals(pot)
    assert (flags == 0).all()
    for b in range(B):
        A = brute.log_partition(pot[b], N)
        assert abs(logz[b] - A) <= 1e-12 * max(1.0, abs(A))
        mu = brute.marginals(pot[b], N)
        np.testing.assert_allclose(marg[b], mu, rtol=0, atol=1e-12)


def test_cfg1_against_enumeration_of_243_labelings():
    cfg = tsgen.CONFIGS[1]
    pot = tsgen.config_potentials(cfg)
    assert brute.count(cfg.N, cfg.C) == 243  # 3^5 (BASELINE.json configs[0])
    logz, marg, _ = oracle.chain_marginals(pot)
    assert abs(logz[0] - brute.log_partition(pot[0], cfg.N)) < 1e-12 * abs(logz[0])
    np.testing.assert_allclose(marg[0], brute.marginals(pot[0], cfg.N), atol=1e-12, rtol=0)


@pytest.mark.parametrize("seed", range(40))
def test_viterbi_matches_enumeration_with_ties(seed):
    # coarse integer potentials in {-1,0,1}: ties are frequent, so the tie rule matters
    rng = np.random.default_rng(seed)
    N, C = int(rng.integers(2, 7)), int(rng.integers(2, 5))
    pot = rng.integers(-1, 2, size=(1, N - 1, C, C)).astype(np.float32)
    path, score, flags = oracle.chain_viterbi(pot)
    z, best = brute.argmax(pot[0], N)
    assert flags[0] == 0
    assert score[0] == best
    np.testing.assert_array_equal(path[0], z)
    # the returned path is optimal and is the reverse-lexicographic minimum of the optimal set
    opt = brute.optimal_set(pot[0], N)
    assert any((o == path[0]).all() for o in opt)


@pytest.mark.parametrize("seed", range(12))
def test_variable_lengths_match_truncated_enumeration(seed):
    B, N, C = 4, 6, 3
    pot = tsgen.potentials(B, N, C, seed=77 + seed)
    lengths = tsgen.random_lengths(B, N, seed)
    logz, marg, flags = oracle.chain_marginals(pot, lengths)
    path, score, vflags = oracle.chain_viterbi(pot, lengths)
    for b in range(B):
        n = int(lengths[b])
        assert abs(logz[b] - brute.log_partition(pot[b], n)) <= 1e-12 * max(1, abs(logz[b]))
        mu = brute.marginals(pot[b], n)
        np.testing.assert_allclose(marg[b, : n - 1], mu, atol=1e-12, rtol=0)
        assert (marg[b, n - 1:] == 0).all()  # reading R10: padded edges give 0
        z, best = brute.argmax(pot[b], n)
        assert score[b] == best
        np.testing.assert_array_equal(path[b, :n], z)
        assert (path[b, n:] == -1).all()


# ---------------------------------------------------------------- closed forms

def test_zero_potentials_closed_form():
    # l == 0: every labelling scores 0, A = n ln C, mu = 1/C^2, z* = 0...0
    B, N, C = 2, 40, 7
    pot = np.zeros((B, N - 1, C, C), dtype=np.float32)
    logz, marg, _ = oracle.chain_marginals(pot)
    np.testing.assert_allclose(logz, N * math.log(C), rtol=1e-14)
    np.testing.assert_allclose(marg, 1.0 / C ** 2, rtol=1e-12)
    path, score, _ = oracle.chain_viterbi(pot)
    assert (path == 0).all() and (score == 0).all()


def test_separable_closed_form():
    # l[t,i,j] = phi_t[j]  =>  A = ln C + sum_t LSE(phi_t);  mu_t = p_t (outer) softmax(phi_t)
    # with p_0 uniform, p_t = softmax(phi_{t-1});  z*_0 = 0, z*_{t+1} = min argmax phi_t.
    N, C = 200, 16
    phi = dyadic((N - 1, C), seed=5)
    pot = np.broadcast_to(phi[:, None, :], (N - 1, C, C))[None].astype(np.float32)
    logz, marg, _ = oracle.chain_marginals(pot)
    ph = phi.astype(np.float64)
    lse = np.log(np.exp(ph - ph.max(1, keepdims=True)).sum(1)) + ph.max(1)
    A = math.log(C) + lse.sum()
    assert abs(logz[0] - A) <= 1e-12 * abs(A)
    sm = np.exp(ph - lse[:, None])
    p = np.vstack([np.full((1, C), 1.0 / C), sm[:-1]])
    np.testing.assert_allclose(marg[0], p[:, :, None] * sm[:, None, :], atol=1e-12, rtol=1e-10)
    path, score, _ = oracle.chain_viterbi(pot)
    assert path[0, 0] == 0
    np.testing.assert_array_equal(path[0, 1:], np.argmax(ph, axis=1))  # argmax = first index
    assert score[0] == ph.max(1).sum()


def test_worked_example_single_edge():
    # single edge, l = [[1,0],[0,0]]: mu(0,0) = e/(e+3), A = ln(e+3)
    pot = np.array([[[[1, 0], [0, 0]]]], dtype=np.float32)
    logz, marg, _ = oracle.chain_marginals(pot)
    e = math.e
    assert abs(logz[0] - math.log(e + 3)) < 1e-15
    assert abs(marg[0, 0, 0, 0] - e / (e + 3)) < 1e-15
    assert abs(marg[0, 0, 1, 1] - 1 / (e + 3)) < 1e-15


def test_paper_two_edge_chain_factorisation():
    # T=2 edges, A = LSE_{c3,c2}[ l_{2,c2,c3} + LSE_{c1} l_{1,c1,c2} ]
    C = 5
    pot = dyadic((1, 2, C, C), seed=9)
    l1, l2 = pot[0, 0].astype(np.float64), pot[0, 1].astype(np.float64)
    inner = np.log(np.exp(l1).sum(axis=0))  # LSE over c1 -> vector over c2
    A = np.log(np.exp(l2 + inner[:, None]).sum())
    logz, _, _ = oracle.chain_marginals(pot)
    assert abs(logz[0] - A) < 1e-12 * abs(A)


# ---------------------------------------------------------------- golden fixtures

def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def test_golden_ln8():
    g = _golden("chain_T2_C2_zeros.json")
    pot = np.zeros((1, g["T"], g["C"], g["C"]), dtype=np.float32)
    logz, _, _ = oracle.chain_marginals(pot)
    assert repr(float(logz[0])) == g["logZ"]


def test_golden_cfg1_enumeration():
    g = _golden("cfg1_brute.json")  # written by tests/golden/make_golden.py (brute.py only)
    cfg = tsgen.CONFIGS[1]
    pot = tsgen.config_potentials(cfg)
    assert hashlib_hex(pot) == g["pot_sha256"]
    logz, marg, _ = oracle.chain_marginals(pot)
    assert abs(logz[0] - g["logZ"]) < 1e-12 * abs(g["logZ"])
    np.testing.assert_allclose(marg[0], np.array(g["marginals"]), atol=1e-12, rtol=0)
    path, score, _ = oracle.chain_viterbi(pot)
    assert path[0].tolist() == g["viterbi_path"] and score[0] == g["viterbi_score"]


def hashlib_hex(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------- gradient identity

def test_marginals_equal_finite_differences():
    # mu = dA/dl; central differences, h = 2^-13 (dyadic: l +- h exact in fp32)
    N, C = 9, 5
    pot = dyadic((1, N - 1, C, C), seed=11)
    _, marg, _ = oracle.chain_marginals(pot)
    rng = np.random.default_rng(3)
    h = 2.0 ** -13
    for _ in range(20):
        t, i, j = rng.integers(N - 1), rng.integers(C), rng.integers(C)
        pp, pm = pot.copy(), pot.copy()
        pp[0, t, i, j] += np.float32(h)
        pm[0, t, i, j] -= np.float32(h)
        fd = (oracle.chain_marginals(pp, want_marg=False)[0][0]
              - oracle.chain_marginals(pm, want_marg=False)[0][0]) / (2 * h)
        assert abs(fd - marg[0, t, i, j]) < 1e-7


# ---------------------------------------------------------------- invariants

def test_marginal_invariants():
    B, N, C = 3, 40, 8
    pot = tsgen.potentials(B, N, C, seed=4)
    _, marg, _ = oracle.chain_marginals(pot)
    np.testing.assert_allclose(marg.sum(axis=(2, 3)), 1.0, atol=1e-12)  # per edge
    # node consistency: sum_i mu_t[i,j] = sum_k mu_{t+1}[j,k]
    np.testing.assert_allclose(marg[:, :-1].sum(axis=2), marg[:, 1:].sum(axis=3), atol=1e-12)
    np.testing.assert_allclose(marg.sum(axis=(1, 2, 3)), N - 1, rtol=1e-12)
    assert (marg >= 0).all() and (marg <= 1 + 1e-15).all()


def test_shift_invariance():
    # l + c gives A + E c; mu and z* unchanged (c dyadic: exact in fp32)
    B, N, C = 2, 30, 6
    pot = tsgen.potentials(B, N, C, seed=8, s=6)
    c = np.float32(3.5)
    lz0, m0, _ = oracle.chain_marginals(pot)
    lz1, m1, _ = oracle.chain_marginals(pot + c)
    np.testing.assert_allclose(lz1, lz0 + (N - 1) * 3.5, rtol=1e-13)
    np.testing.assert_allclose(m1, m0, atol=1e-12)
    p0, s0, _ = oracle.chain_viterbi(pot)
    p1, s1, _ = oracle.chain_viterbi(pot + c)
    np.testing.assert_array_equal(p0, p1)
    np.testing.assert_array_equal(s1, s0 + (N - 1) * 3.5)


def test_stabilisation_at_1e4():
    # magnitude 1e4 stays finite and equals the shifted result + analytic shift
    B, N, C = 2, 20, 5
    pot = tsgen.potentials(B, N, C, seed=12, s=6)
    big = (pot + np.float32(1e4)).astype(np.float32)
    assert ((big - np.float32(1e4)) == pot).all()  # exact in fp32
    lz0, m0, _ = oracle.chain_marginals(pot)
    lz1, m1, f1 = oracle.chain_marginals(big)
    assert np.isfinite(lz1).all() and (f1 == 0).all()
    np.testing.assert_allclose(lz1, lz0 + (N - 1) * 1e4, rtol=1e-13)
    np.testing.assert_allclose(m1, m0, atol=1e-10)
    neg = (pot - np.float32(1e4)).astype(np.float32)
    lz2, m2, _ = oracle.chain_marginals(neg)
    np.testing.assert_allclose(lz2, lz0 - (N - 1) * 1e4, rtol=1e-13)
    np.testing.assert_allclose(m2, m0, atol=1e-10)


def test_masks_and_structured_inputs_match_enumeration():
    pot = tsgen.tagging_potentials(3, 6, 4, seed=21, mask_frac=0.3)
    logz, marg, flags = oracle.chain_marginals(pot)
    path, score, _ = oracle.chain_viterbi(pot)
    for b in range(3):
        A = brute.log_partition(pot[b], 6)
        assert abs(logz[b] - A) <= 1e-12 * max(1, abs(A))
        np.testing.assert_allclose(marg[b], brute.marginals(pot[b], 6), atol=1e-12, rtol=0)
        z, best = brute.argmax(pot[b], 6)
        assert score[b] == best and (path[b] == z).all()
    assert (marg[np.isneginf(pot)] == 0).all()  # masked parts have zero marginal


# ---------------------------------------------------------------- flags / degenerate cases

def test_flags_and_degenerate_cases():
    B, N, C = 5, 6, 3
    pot = tsgen.potentials(B, N, C, seed=2)
    pot[1] = -np.inf                         # EMPTY
    pot[2, 3, 1, 2] = np.nan                 # NONFINITE on a used edge
    pot[4, 4, 0, 0] = np.nan                 # NaN beyond len: ignored
    lengths = np.array([0, N, N, 1, 4], dtype=np.int32)
    logz, marg, flags = oracle.chain_marginals(pot, lengths)
    path, score, vflags = oracle.chain_viterbi(pot, lengths)
    assert flags.tolist() == [oracle.F_BADLEN, oracle.F_EMPTY, oracle.F_NONFINITE, 0, 0]
    assert vflags.tolist() == flags.tolist()
    assert math.isnan(logz[0]) and math.isnan(logz[2]) and logz[1] == -math.inf
    assert abs(logz[3] - math.log(C)) < 1e-15 and score[3] == 0  # len=1: A = ln C
    assert path[3].tolist() == [0] + [-1] * (N - 1)
    assert (marg[:4] == 0).all() and (path[:3] == -1).all() and score[1] == -math.inf
    assert abs(logz[4] - brute.log_partition(pot[4], 4)) < 1e-12 * abs(logz[4])


# ---------------------------------------------------------------- §6(c) semiring product

def test_semiring_matmul_examples():
    # S:121-124
    assert oracle.semiring_matmul([[1.0]], [[2.0]])[0, 0] == 3.0
    assert abs(oracle.semiring_matmul([[0.0, 0.0]], [[0.0], [0.0]])[0, 0] - math.log(2)) < 1e-15
    v = oracle.semiring_matmul([[1000.0, 1000.0]], [[1000.0], [1000.0]])[0, 0]
    assert abs(v - (2000 + math.log(2))) < 1e-12
    assert (oracle.semiring_matmul(np.zeros((2, 2)), np.zeros((2, 2)), oracle.MAX) == 0).all()
    assert oracle.semiring_matmul([[-np.inf, 1.0]], [[2.0], [-np.inf]])[0, 0] == -np.inf


def test_semiring_matmul_reduces_to_real_matmul():
    # (LSE,+) product == log(exp(T) @ exp(U)) ("(sum,x) ... matrix multiplication")
    rng = np.random.default_rng(0)
    T, U = rng.normal(size=(7, 5)), rng.normal(size=(5, 9))
    np.testing.assert_allclose(oracle.semiring_matmul(T, U), np.log(np.exp(T) @ np.exp(U)),
                               rtol=1e-14)
    np.testing.assert_array_equal(oracle.semiring_matmul(T, U, oracle.MAX),
                                  (T[:, :, None] + U[None, :, :]).max(axis=1))


def test_summary_is_path_sum():
    # S[i,j] = (+) over all label paths from i to j through E edges (enumerated)
    E, C = 3, 3
    pot = dyadic((E, C, C), seed=31)
    S = oracle.chain_summary(pot)
    Smax = oracle.chain_summary(pot, oracle.MAX)
    Z = brute.labelings(E + 1, C)
    sc = sum(pot[t].astype(np.float64)[Z[:, t], Z[:, t + 1]] for t in range(E))
    for i in range(C):
        for j in range(C):
            sel = sc[(Z[:, 0] == i) & (Z[:, E] == j)]
            assert abs(S[i, j] - (np.log(np.exp(sel - sel.max()).sum()) + sel.max())) < 1e-12
            assert Smax[i, j] == sel.max()
    I = oracle.chain_summary(np.zeros((0, C, C), np.float32))
    assert (np.diag(I) == 0).all() and np.isneginf(I[~np.eye(C, dtype=bool)]).all()


@pytest.mark.parametrize("T", [1, 2, 3, 5, 7, 8, 17, 64])
def test_scan_order_equals_serial(T):
    # §6(a)/Fig. 4: balanced tree with I padding == left-to-right; ceil(log2 T) layers
    C = 4
    pot = tsgen.potentials(1, T + 1, C, seed=T)
    root, layers = oracle.scan_partition(pot[0])
    logz, _, _ = oracle.chain_marginals(pot)
    assert abs(root - logz[0]) <= 1e-12 * max(1, abs(root))
    assert layers == math.ceil(math.log2(T)) if T > 1 else layers == 0
    mroot, _ = oracle.scan_partition(pot[0], oracle.MAX)
    assert mroot == oracle.chain_viterbi(pot)[1][0]


# ---------------------------------------------------------------- generator

def test_generator_numpy_equals_host_c():
    for (B, N, C, seed, s) in [(2, 7, 5, 123, 15), (1, 30, 3, 9, 6), (3, 4, 20, 1, 12)]:
        a = tsgen.potentials(B, N, C, seed, s)
        b = tsgen.fill_host(B, N, C, seed, s)
        assert a.tobytes() == b.tobytes()
    # time-sliced generation uses global indices
    full = tsgen.potentials(2, 50, 4, 5, 6)
    part = tsgen.fill_host(2, 50, 4, 5, 6, t_begin=20, E_local=10, E_global=49)
    assert part.tobytes() == full[:, 20:30].tobytes()


def test_generator_recipe_properties():
    assert [c.quantum for c in tsgen.CONFIGS.values()] == [15, 15, 13, 12, 6]
    for c in tsgen.CONFIGS.values():
        assert c.E * 4 * 2 ** c.quantum <= 2 ** 24
    v = tsgen.potentials(4, 200, 20, 42, 15).astype(np.float64)
    assert np.abs(v).max() <= 4.0 and abs(v.mean()) < 0.02 and abs(v.std() - 1.155) < 0.02
    q = tsgen.potentials(1, 100, 8, 3, 6)
    assert ((q * 64) == np.round(q * 64)).all()  # on the 2^-s grid
