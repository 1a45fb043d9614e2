"""oracle — the plain, slow, float64 CPU oracle for the linear-chain CRF hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` leg may import this package.  The product
path (paper_2002_00876_b200/) never imports it, and it never imports the product
path.  See oracle/oracle.c for the definitions and their citations, and
oracle/brute.py for the independent brute-force enumerator that pins it.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

F_EMPTY, F_NONFINITE, F_BADLEN = 1, 2, 4  # the documented flag contract
LOG, MAX = 0, 1

_p = ctypes.c_void_p
_i64 = ctypes.c_int64


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc (no fast-math)."""
    import subprocess

    out = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-fPIC", "-shared", "-o", out, src,
                               "-lm", "-lpthread"])
    return out


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.oracle_semiring_matmul.argtypes = [ctypes.c_int, _p, _p, _i64, _i64, _i64, _p]
        L.oracle_chain_marginals.argtypes = [_p, _p, _i64, _i64, _i64, _p, _p, _p, ctypes.c_int]
        L.oracle_chain_viterbi.argtypes = [_p, _p, _i64, _i64, _i64, _p, _p, _p, ctypes.c_int]
        L.oracle_gen_marginals.argtypes = [ctypes.c_uint64, ctypes.c_int, _i64, _i64, _i64, _p,
                                           _i64, _p, _p, _p]
        L.oracle_gen_viterbi.argtypes = [ctypes.c_uint64, ctypes.c_int, _i64, _i64, _i64, _p, _p,
                                         _p]
        L.oracle_chain_summary.argtypes = [ctypes.c_int, _p, _i64, _i64, _p]
        L.oracle_scan_partition.argtypes = [ctypes.c_int, _p, _i64, _i64, _p, _p]
        for f in ("oracle_semiring_matmul", "oracle_chain_marginals", "oracle_chain_viterbi",
                  "oracle_gen_marginals", "oracle_gen_viterbi", "oracle_chain_summary",
                  "oracle_scan_partition"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _f32(pot):
    return np.ascontiguousarray(pot, dtype=np.float32)


def _lengths(lengths, B):
    if lengths is None:
        return None
    l = np.ascontiguousarray(lengths, dtype=np.int32)
    assert l.shape == (B,)
    return l


def semiring_matmul(T, U, semiring: int = LOG) -> np.ndarray:
    """V = T (x) U per §6(c), fp64."""
    T = np.ascontiguousarray(T, dtype=np.float64)
    U = np.ascontiguousarray(U, dtype=np.float64)
    n, m = T.shape
    m2, o = U.shape
    assert m == m2
    V = np.empty((n, o), dtype=np.float64)
    rc = lib().oracle_semiring_matmul(semiring, T.ctypes.data, U.ctypes.data, n, m, o, V.ctypes.data)
    assert rc == 0
    return V


def chain_marginals(pot, lengths=None, want_marg: bool = True, threads: int = 1):
    """pot [B, N-1, C, C] fp32 -> (logz [B] f64, marg [B,N-1,C,C] f64 or None, flags [B] u32)."""
    pot = _f32(pot)
    B, E, C, C2 = pot.shape
    assert C == C2
    N = E + 1
    l = _lengths(lengths, B)
    logz = np.empty(B, dtype=np.float64)
    marg = np.empty((B, E, C, C), dtype=np.float64) if want_marg else None
    flags = np.zeros(B, dtype=np.uint32)
    rc = lib().oracle_chain_marginals(pot.ctypes.data if pot.size else None,
                                      l.ctypes.data if l is not None else None, B, N, C,
                                      logz.ctypes.data, marg.ctypes.data if want_marg else None,
                                      flags.ctypes.data, threads)
    assert rc == 0
    return logz, marg, flags


def chain_viterbi(pot, lengths=None, threads: int = 1):
    """-> (path [B,N] i32 with -1 beyond len, score [B] f64, flags [B] u32)."""
    pot = _f32(pot)
    B, E, C, _ = pot.shape
    N = E + 1
    l = _lengths(lengths, B)
    path = np.empty((B, N), dtype=np.int32)
    score = np.empty(B, dtype=np.float64)
    flags = np.zeros(B, dtype=np.uint32)
    rc = lib().oracle_chain_viterbi(pot.ctypes.data if pot.size else None,
                                    l.ctypes.data if l is not None else None, B, N, C,
                                    path.ctypes.data, score.ctypes.data, flags.ctypes.data, threads)
    assert rc == 0
    return path, score, flags


def gen_marginals(seed: int, s: int, b: int, N: int, C: int, edges):
    """Full-size sampled mode: one generated sequence b; mu at the requested edges."""
    edges = np.ascontiguousarray(sorted(int(e) for e in edges), dtype=np.int64)
    marg = np.empty((len(edges), C, C), dtype=np.float64)
    logz = np.empty(1, dtype=np.float64)
    flags = np.zeros(1, dtype=np.uint32)
    rc = lib().oracle_gen_marginals(seed, s, b, N, C, edges.ctypes.data if len(edges) else None,
                                    len(edges), logz.ctypes.data,
                                    marg.ctypes.data if len(edges) else None, flags.ctypes.data)
    assert rc == 0
    return float(logz[0]), edges, marg, int(flags[0])


def gen_viterbi(seed: int, s: int, b: int, N: int, C: int):
    path = np.empty(N, dtype=np.int32)
    score = np.empty(1, dtype=np.float64)
    flags = np.zeros(1, dtype=np.uint32)
    rc = lib().oracle_gen_viterbi(seed, s, b, N, C, path.ctypes.data, score.ctypes.data,
                                  flags.ctypes.data)
    assert rc == 0
    return path, float(score[0]), int(flags[0])


def chain_summary(pot_seq, semiring: int = LOG) -> np.ndarray:
    """Transfer matrix S = l_0 (x) ... (x) l_{E-1} of one segment [E, C, C] -> [C, C] fp64."""
    pot_seq = _f32(pot_seq)
    E, C, _ = pot_seq.shape
    S = np.empty((C, C), dtype=np.float64)
    rc = lib().oracle_chain_summary(semiring, pot_seq.ctypes.data if E else None, E, C,
                                    S.ctypes.data)
    assert rc == 0
    return S


def scan_partition(pot_seq, semiring: int = LOG):
    """Fig. 4 ordering: balanced tree with I padding. -> (root, layers)."""
    pot_seq = _f32(pot_seq)
    T, C, _ = pot_seq.shape
    root = ctypes.c_double()
    layers = ctypes.c_int()
    rc = lib().oracle_scan_partition(semiring, pot_seq.ctypes.data, T, C, ctypes.byref(root),
                                     ctypes.byref(layers))
    assert rc == 0
    return root.value, layers.value


def max_indicator(path: np.ndarray, C: int, lengths=None) -> np.ndarray:
    """dA*/dl as the one-hot edge indicator of the Viterbi path: [B,N-1,C,C]."""
    B, N = path.shape
    out = np.zeros((B, N - 1, C, C), dtype=np.float64)
    for b in range(B):
        n = N if lengths is None else int(lengths[b])
        for t in range(max(n - 1, 0)):
            if path[b, t] >= 0 and path[b, t + 1] >= 0:
                out[b, t, path[b, t], path[b, t + 1]] = 1.0
    return out


# ---------------------------------------------------------------------------------------
# SURVEY §8(f) "next" rows: distribution properties of §3 on the same chain.
# ---------------------------------------------------------------------------------------

def chain_entropy(pot, lengths=None, threads: int = 1):
    """Entropy H_b = -Σ_z p(z) log p(z) (Table 2 'Entropy' P:206) written out via
    log p(z) = Score(z) - A and linearity of expectation over the parts:
        H = A - E_p[Score(z)] = A - Σ_t Σ_ij mu_t[i][j] l_t[i][j]
    fp64; terms with mu = 0 contribute 0 (masked -inf parts).  Flags as chain_marginals;
    H = NaN for EMPTY / NONFINITE / BADLEN sequences.  -> (H [B] f64, logz [B], flags)."""
    pot64 = np.asarray(pot, dtype=np.float64)
    logz, marg, flags = chain_marginals(pot, lengths, want_marg=True, threads=threads)
    B = pot64.shape[0]
    H = np.empty(B, dtype=np.float64)
    for b in range(B):
        if flags[b] != 0:
            H[b] = math.nan
            continue
        m = marg[b]
        nz = m != 0.0
        H[b] = logz[b] - float(np.sum(m[nz] * pot64[b][nz]))
    return H, logz, flags


def chain_expectation(pot, r, lengths=None, threads: int = 1):
    """Expectation of an additive feature (Table 2 'Exp.' row): the expectation
    semiring's moment over all structures divided by their total weight,
        E_p[Σ_{t<len-1} r_t[z_t][z_{t+1}]] = Σ_t Σ_ij mu_t[i][j] r_t[i][j]
    by linearity of expectation over the parts.  fp64; terms with mu = 0
    contribute 0.  NaN for EMPTY / NONFINITE / BADLEN sequences.
    -> (E [B] f64, logz [B], flags)."""
    r64 = np.asarray(r, dtype=np.float64)
    logz, marg, flags = chain_marginals(pot, lengths, want_marg=True, threads=threads)
    B = r64.shape[0]
    out = np.empty(B, dtype=np.float64)
    for b in range(B):
        if flags[b] != 0:
            out[b] = math.nan
            continue
        m = marg[b]
        nz = m != 0.0
        out[b] = float(np.sum(m[nz] * r64[b][nz]))
    return out, logz, flags


def chain_score(pot, z, lengths=None):
    """Score(z) = Σ_{t < len-1} l[t, z_t, z_{t+1}], fp64 (exact for fp32
    inputs up to rounding of the sum).  z [B, N] int; a label outside [0, C) on a used
    position gives NaN."""
    pot64 = np.asarray(pot, dtype=np.float64)
    z = np.asarray(z)
    B, E, C, _ = pot64.shape
    out = np.empty(B, dtype=np.float64)
    for b in range(B):
        n = E + 1 if lengths is None else int(lengths[b])
        if n < 1 or n > E + 1 or np.any((z[b, :n] < 0) | (z[b, :n] >= C)):
            out[b] = math.nan
            continue
        out[b] = math.fsum(pot64[b, t, z[b, t], z[b, t + 1]] for t in range(n - 1))
    return out


def chain_log_prob(pot, z, lengths=None, threads: int = 1):
    """log p(z) = Score(z) - A (P:119 'Density')."""
    logz, _, flags = chain_marginals(pot, lengths, want_marg=False, threads=threads)
    sc = chain_score(pot, z, lengths)
    out = sc - logz
    out[flags != 0] = math.nan
    return out


def forward_alpha(pot_seq, n: int) -> np.ndarray:
    """alpha [n, C] fp64 of one sequence: alpha_0 = 0, alpha_{t+1}[j] = LSE_i(alpha_t[i] +
    l_t[i][j]) with the per-cell max of §6(c)."""
    pot = np.asarray(pot_seq, dtype=np.float64)
    C = pot.shape[-1]
    al = np.zeros((n, C), dtype=np.float64)
    for t in range(n - 1):
        x = al[t][:, None] + pot[t]                      # [i, j]
        q = np.max(x, axis=0)
        with np.errstate(invalid="ignore", divide="ignore"):
            s = np.sum(np.exp(x - np.where(np.isfinite(q), q, 0.0)[None, :]), axis=0)
            al[t + 1] = np.where(np.isfinite(q), q + np.log(s), -math.inf)
    return al


def _draw(logw: np.ndarray, u: float) -> int:
    """Inverse-CDF draw from p_i ∝ exp(logw_i): the smallest i with cdf_i > u (fp64)."""
    m = float(np.max(logw))
    p = np.exp(logw - m)
    c = np.cumsum(p)
    k = int(np.searchsorted(c, u * c[-1], side="right"))
    return min(k, len(logw) - 1)


def ffbs_sample(pot, uniforms, lengths=None):
    """Forward-filtering backward-sampling (Table 2 'Sample' P:202): one exact draw
    z ~ p(z) per (k, b) from caller-supplied uniforms u [K, B, N] in [0, 1):
        z_{n-1} ~ p(z_{n-1}) ∝ exp(alpha_{n-1}[j])                      (u[k, b, n-1])
        z_t     ~ p(z_t | z_{t+1}) ∝ exp(alpha_t[i] + l_t[i][z_{t+1}])   (u[k, b, t])
    -> z [K, B, N] int32 (-1 beyond len or for EMPTY / NONFINITE / BADLEN sequences)."""
    pot64 = np.asarray(pot, dtype=np.float64)
    u = np.asarray(uniforms, dtype=np.float64)
    K = u.shape[0]
    B, E, C, _ = pot64.shape
    N = E + 1
    _, _, flags = chain_marginals(pot, lengths, want_marg=False)
    z = np.full((K, B, N), -1, dtype=np.int32)
    for b in range(B):
        if flags[b] != 0:
            continue
        n = N if lengths is None else int(lengths[b])
        al = forward_alpha(pot64[b], n)
        for k in range(K):
            zz = _draw(al[n - 1], u[k, b, n - 1])
            z[k, b, n - 1] = zz
            for t in range(n - 2, -1, -1):
                zz = _draw(al[t] + pot64[b, t, :, zz], u[k, b, t])
                z[k, b, t] = zz
    return z


def chain_kbest(pot, K: int, lengths=None):
    """K-best labelings (Table 2 'K-Max'): the first K labelings of the total order
    (Score descending, then reverse-lexicographic ascending — z_{n-1} first, the tie rule R5
    extended; reading R16), by the k-best max-plus DP written out in fp64:
        delta_0[j] = [(0, -)],  delta_{t+1}[j] = top-K over (i, r) of delta_t[i][r] + l_t[i][j]
    with candidates ordered by (score desc, i asc, r asc) — which is exactly the global order
    restricted to partial paths ending at (t+1, j) — and the final merge over (score desc,
    j asc, r asc).  -> (paths [B, K, N] int32 (-1 beyond len / missing), scores [B, K] f64
    (-inf missing), flags [B])."""
    pot64 = np.asarray(pot, dtype=np.float64)
    B, E, C, _ = pot64.shape
    N = E + 1
    _, _, flags = chain_viterbi(pot, lengths)
    paths = np.full((B, K, N), -1, dtype=np.int32)
    scores = np.full((B, K), -math.inf, dtype=np.float64)
    for b in range(B):
        n = N if lengths is None else int(lengths[b])
        if flags[b] & (F_NONFINITE | F_BADLEN):
            scores[b, :] = math.nan
            continue
        # lists[j] = [(score, i, r)] sorted by (score desc, i asc, r asc); bps[t][j] = list
        lists = [[(0.0, -1, -1)] for _ in range(C)]
        bps = []
        for t in range(n - 1):
            new = []
            for j in range(C):
                cand = []
                for i in range(C):
                    lv = pot64[b, t, i, j]
                    for r, (sc, _, _) in enumerate(lists[i]):
                        v = sc + lv
                        if v != -math.inf:
                            cand.append((v, i, r))
                cand.sort(key=lambda x: (-x[0], x[1], x[2]))
                new.append(cand[:K])
            bps.append(new)
            lists = new
        final = []
        for j in range(C):
            for r, (sc, _, _) in enumerate(lists[j]):
                if sc != -math.inf:
                    final.append((sc, j, r))
        final.sort(key=lambda x: (-x[0], x[1], x[2]))
        for q, (sc, j, r) in enumerate(final[:K]):
            scores[b, q] = sc
            z, slot = j, r
            paths[b, q, n - 1] = z
            for t in range(n - 2, -1, -1):
                _, i, rr = bps[t][z][slot]
                paths[b, q, t] = i
                z, slot = i, rr
    return paths, scores, flags


# ---------------------------------------------------------------------------------------
# semi-Markov CRF on the same chain machinery (Table 1 'Semi-Markov',
# P:44; "similar parallel approach can also be used for ... semi-Markov").
# Reading R17: pot [B, N-1, K, C, C]; l[b, n, k-1, c1, c2] scores a segment that
# covers the k steps n -> n+k with label c2, following label c1 at node n.  A labelled
# segmentation is 0 = p_0 < p_1 < ... < p_m = E_b (E_b = len_b - 1, p_s - p_{s-1} <= K) with
# labels y_0 (free) ... y_m; Score = Σ_s l[p_{s-1}, p_s - p_{s-1} - 1, y_{s-1}, y_s].
# K = 1 is exactly the linear chain.
# ---------------------------------------------------------------------------------------

def _lse_np(x, axis=None):
    m = np.max(x, axis=axis, keepdims=True)
    mf = np.where(np.isfinite(m), m, 0.0)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.log(np.sum(np.exp(x - mf), axis=axis, keepdims=True)) + mf
    r = np.where(np.isfinite(m), r, m)
    return np.squeeze(r, axis=axis) if axis is not None else float(r.reshape(()))


def semimarkov_marginals(pot, lengths=None, want_marg: bool = True):
    """Segmental forward-backward in fp64 (the per-cell max of §6(c) via LSE):
        alpha_0 = 0, alpha_p[c] = LSE_{k<=min(K,p), c'} alpha_{p-k}[c'] + l[p-k, k-1, c', c]
        beta_E  = 0, beta_p[c]  = LSE_{k<=min(K,E-p), c'} l[p, k-1, c, c'] + beta_{p+k}[c']
        A = LSE_c alpha_E[c],   mu[n,k-1,c1,c2] = exp(alpha_n[c1] + l + beta_{n+k}[c2] - A)
    Flags as chain_marginals (EMPTY: A = -inf -> mu = 0; NaN/+inf on a used part ->
    NONFINITE, A = NaN; bad length -> BADLEN).  -> (logz [B], marg [B,N-1,K,C,C] | None, flags)."""
    pot64 = np.asarray(pot, dtype=np.float64)
    B, E, K, C, _ = pot64.shape
    N = E + 1
    logz = np.empty(B)
    marg = np.zeros(pot64.shape) if want_marg else None
    flags = np.zeros(B, dtype=np.uint32)
    for b in range(B):
        n_b = N if lengths is None else int(lengths[b])
        if n_b < 1 or n_b > N:
            logz[b] = math.nan
            flags[b] = F_BADLEN
            continue
        Eb = n_b - 1
        used = np.zeros((E, K), bool)
        for n in range(Eb):
            used[n, :min(K, Eb - n)] = True
        if np.any(~np.isfinite(pot64[b][used]) & ~(pot64[b][used] == -np.inf)):
            logz[b] = math.nan
            flags[b] = F_NONFINITE
            continue
        al = np.full((Eb + 1, C), -np.inf)
        al[0] = 0.0
        for p in range(1, Eb + 1):
            terms = [al[p - k][:, None] + pot64[b, p - k, k - 1] for k in range(1, min(K, p) + 1)]
            al[p] = _lse_np(np.concatenate(terms, axis=0), axis=0)
        be = np.full((Eb + 1, C), -np.inf)
        be[Eb] = 0.0
        for p in range(Eb - 1, -1, -1):
            terms = [pot64[b, p, k - 1] + be[p + k][None, :] for k in range(1, min(K, Eb - p) + 1)]
            be[p] = _lse_np(np.concatenate(terms, axis=1), axis=1)
        A = _lse_np(al[Eb])
        logz[b] = A
        if A == -np.inf:
            flags[b] = F_EMPTY
            continue
        if want_marg:
            for n in range(Eb):
                for k in range(1, min(K, Eb - n) + 1):
                    with np.errstate(invalid="ignore"):
                        x = al[n][:, None] + pot64[b, n, k - 1] + be[n + k][None, :] - A
                    marg[b, n, k - 1] = np.where(np.isfinite(x), np.exp(x), 0.0)
    return logz, marg, flags


def semimarkov_viterbi(pot, lengths=None):
    """Semi-Markov Viterbi: the max semiring over the labelled segmentations
    of reading R17:
        delta_0[c] = 0,  delta_p[c] = max_{k <= min(K,p), c'} delta_{p-k}[c'] + l[p-k, k-1, c', c]
    backpointer of (p, c) = the first (k, c') in (k asc, c' asc) order attaining the max
    (strict >), end label = the smallest c attaining max_c delta_E[c] (reading R18: the
    labelled segmentation that is lexicographically smallest in (y_m, k_m, y_{m-1}, ..., y_0)
    read from the end).  fp64.
    -> (seg [B, N] int32: the label at every segment boundary node, -1 at interior nodes,
        beyond len and for flagged sequences; score [B] f64; flags as semimarkov_marginals
        with EMPTY -> score -inf)."""
    pot64 = np.asarray(pot, dtype=np.float64)
    B, E, K, C, _ = pot64.shape
    N = E + 1
    seg = np.full((B, N), -1, dtype=np.int32)
    score = np.empty(B)
    flags = np.zeros(B, dtype=np.uint32)
    for b in range(B):
        n_b = N if lengths is None else int(lengths[b])
        if n_b < 1 or n_b > N:
            score[b] = math.nan
            flags[b] = F_BADLEN
            continue
        Eb = n_b - 1
        used = np.zeros((E, K), bool)
        for n in range(Eb):
            used[n, :min(K, Eb - n)] = True
        if np.any(~np.isfinite(pot64[b][used]) & ~(pot64[b][used] == -np.inf)):
            score[b] = math.nan
            flags[b] = F_NONFINITE
            continue
        dl = np.full((Eb + 1, C), -np.inf)
        dl[0] = 0.0
        bk = np.zeros((Eb + 1, C), dtype=np.int64)
        bc = np.zeros((Eb + 1, C), dtype=np.int64)
        for p in range(1, Eb + 1):
            for k in range(1, min(K, p) + 1):
                cand = dl[p - k][:, None] + pot64[b, p - k, k - 1]    # [c', c]
                arg = np.argmax(cand, axis=0)                         # first c' on ties
                val = cand[arg, np.arange(C)]
                better = val > dl[p]                                  # strict: earlier k wins
                dl[p] = np.where(better, val, dl[p])
                bk[p] = np.where(better, k, bk[p])
                bc[p] = np.where(better, arg, bc[p])
        best = float(np.max(dl[Eb]))
        if best == -np.inf:
            score[b] = -np.inf
            flags[b] = F_EMPTY
            continue
        c = int(np.argmax(dl[Eb]))
        score[b] = best
        p = Eb
        while p > 0:
            seg[b, p] = c
            k, c = int(bk[p, c]), int(bc[p, c])
            p -= k
        seg[b, 0] = c
    return seg, score, flags
