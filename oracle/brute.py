"""brute.py — brute-force enumeration of every labelling z in [C]^n (TEST INFRASTRUCTURE).

The second, independent witness the oracle is pinned against (PAPER.md footnote,
P:149: "The test suite for each distribution enumerates over all structures to
ensure that properties hold ... for small sets").  It is written against the
structure definitions of §5.1, never the chart recursions:

  Score(z) = sum_t l[t, z_t, z_{t+1}]
  A        = log sum_z exp Score(z)
  mu[t,i,j] = sum_{z: z_t=i, z_{t+1}=j} exp(Score(z) - A)
  A*       = max_z Score(z)
  z*       = the optimal labelling that is lexicographically smallest when read
             from the last position backwards (reading R5)

Guarded at C^n <= 1e6.
"""
from __future__ import annotations

import math

import numpy as np

GUARD = 1_000_000


def labelings(n: int, C: int) -> np.ndarray:
    """All C^n labelings, [C^n, n] int64 (row k = base-C digits of k, position 0 first)."""
    count = C ** n
    if count > GUARD:
        raise ValueError(f"brute force refused: C^n = {count} > {GUARD}")
    k = np.arange(count, dtype=np.int64)
    Z = np.empty((count, n), dtype=np.int64)
    for pos in range(n):
        Z[:, pos] = (k // (C ** pos)) % C
    return Z


def scores(pot_seq: np.ndarray, n: int) -> tuple[np.ndarray, np.ndarray]:
    """(Z, Score(z)) for the first n positions of one sequence (fp64 sums)."""
    pot = np.asarray(pot_seq, dtype=np.float64)
    C = pot.shape[-1]
    Z = labelings(n, C)
    sc = np.zeros(Z.shape[0], dtype=np.float64)
    for t in range(n - 1):
        sc = sc + pot[t, Z[:, t], Z[:, t + 1]]
    return Z, sc


def _lse(x: np.ndarray) -> float:
    m = float(np.max(x))
    if m == -math.inf:
        return -math.inf
    return m + math.log(math.fsum(np.exp(x - m).tolist()))


def log_partition(pot_seq, n: int) -> float:
    _, sc = scores(pot_seq, n)
    return _lse(sc)


def marginals(pot_seq, n: int) -> np.ndarray:
    """mu [n-1, C, C] fp64 by direct summation over all labelings."""
    pot = np.asarray(pot_seq, dtype=np.float64)
    C = pot.shape[-1]
    Z, sc = scores(pot, n)
    A = _lse(sc)
    mu = np.zeros((max(n - 1, 0), C, C), dtype=np.float64)
    if A == -math.inf:
        return mu
    w = np.exp(sc - A)
    for t in range(n - 1):
        np.add.at(mu[t], (Z[:, t], Z[:, t + 1]), w)
    return mu


def argmax(pot_seq, n: int) -> tuple[np.ndarray, float]:
    """(z*, A*) with the canonical tie rule R5 (reverse-lexicographic minimum)."""
    Z, sc = scores(pot_seq, n)
    best = float(np.max(sc))
    opt = Z[sc == best]
    # lexicographic order on the reversed labelling: compare z_{n-1} first, then z_{n-2}, ...
    order = np.lexsort(opt.T)  # np.lexsort sorts by the LAST key first == position n-1 first
    return opt[order[0]].astype(np.int32), best


def optimal_set(pot_seq, n: int) -> np.ndarray:
    Z, sc = scores(pot_seq, n)
    return Z[sc == np.max(sc)]


def count(n: int, C: int) -> int:
    """Count semiring on zero potentials (Table 2 'Count'): |Z| = C^n."""
    return labelings(n, C).shape[0]


def probabilities(pot_seq, n: int) -> tuple[np.ndarray, np.ndarray]:
    """(Z, p(z)) for every labelling: p = exp(Score - A)."""
    Z, sc = scores(pot_seq, n)
    A = _lse(sc)
    return Z, np.exp(sc - A)


def entropy(pot_seq, n: int) -> float:
    """H = -Σ_z p(z) log p(z) by enumeration, terms with p = 0 omitted."""
    _, p = probabilities(pot_seq, n)
    p = p[p > 0]
    return -math.fsum((p * np.log(p)).tolist())


def expectation(pot_seq, r_seq, n: int) -> float:
    """E_p[Σ_t r_t[z_t][z_{t+1}]] = Σ_z p(z) Σ_t r_t[z_t][z_{t+1}] by enumeration (Table 2
    'Exp.'), structures with p = 0 omitted."""
    Z, p = probabilities(pot_seq, n)
    r = np.asarray(r_seq, np.float64)
    keep = p > 0
    Z, p = Z[keep], p[keep]
    f = np.zeros(len(Z))
    for t in range(n - 1):
        f += r[t, Z[:, t], Z[:, t + 1]]
    return math.fsum((p * f).tolist())


def kbest(pot_seq, n: int, K: int) -> tuple[np.ndarray, np.ndarray]:
    """The first K labelings in the order (Score desc, then reverse-lexicographic asc:
    z_{n-1} first) by sorting the enumeration — the definition of the K-Max result."""
    Z, sc = scores(pot_seq, n)
    keep = sc != -math.inf
    Z, sc = Z[keep], sc[keep]
    order = np.lexsort(tuple(Z.T) + (-sc,))  # last key first: -score, then z_{n-1}, ...
    order = order[:K]
    return Z[order].astype(np.int32), sc[order]


def segmentations(E: int, K: int):
    """All boundary sequences 0 = p_0 < ... < p_m = E with steps <= K (compositions of E)."""
    out = []

    def rec(p, acc):
        if p == E:
            out.append(list(acc))
            return
        for k in range(1, min(K, E - p) + 1):
            acc.append(p + k)
            rec(p + k, acc)
            acc.pop()

    rec(0, [0])
    return out


def semimarkov_argmax(pot_seq, n: int):
    """The canonical best labelled segmentation by enumeration (reading R18): among the
    maximisers of Score (R17), the one whose key (y_m, k_m, y_{m-1}, k_{m-1}, ..., k_1, y_0)
    — read from the end — is lexicographically smallest.  -> (seg [n] int32 as
    oracle.semimarkov_viterbi, score); score -inf and seg all -1 when nothing is finite."""
    pot = np.asarray(pot_seq, dtype=np.float64)
    _, K, C, _ = pot.shape
    E = n - 1
    best, best_key, best_seg = -math.inf, None, None
    for bnd in segmentations(E, K):
        m = len(bnd) - 1
        for ys in np.ndindex(*([C] * (m + 1))):
            sc = sum(pot[bnd[s - 1], bnd[s] - bnd[s - 1] - 1, ys[s - 1], ys[s]]
                     for s in range(1, m + 1)) if m else 0.0
            if sc == -math.inf:
                continue
            key = []
            for s in range(m, 0, -1):
                key += [ys[s], bnd[s] - bnd[s - 1]]
            key.append(ys[0])
            if sc > best or (sc == best and key < best_key):
                best, best_key, best_seg = sc, key, (bnd, ys)
    seg = np.full(n, -1, dtype=np.int32)
    if best_seg is not None:
        for p, y in zip(*best_seg):
            seg[p] = y
    return seg, best


def semimarkov(pot_seq, n: int):
    """(A, mu) of a semi-Markov chain by enumerating every segmentation x labelling (reading
    R17): Score = Σ_s l[p_{s-1}, p_s - p_{s-1} - 1, y_{s-1}, y_s]."""
    pot = np.asarray(pot_seq, dtype=np.float64)
    _, K, C, _ = pot.shape
    E = n - 1
    items = []
    for seg in segmentations(E, K):
        m = len(seg) - 1
        for ys in np.ndindex(*([C] * (m + 1))):
            sc = 0.0
            parts = []
            for s in range(1, m + 1):
                n0, k = seg[s - 1], seg[s] - seg[s - 1]
                sc += pot[n0, k - 1, ys[s - 1], ys[s]]
                parts.append((n0, k - 1, ys[s - 1], ys[s]))
            items.append((sc, parts))
    scs = np.array([it[0] for it in items])
    A = _lse(scs)
    mu = np.zeros(pot.shape)
    if A != -math.inf:
        for sc, parts in items:
            w = math.exp(sc - A)
            for q in parts:
                mu[q] += w
    return A, mu
