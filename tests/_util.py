"""Shared comparison helpers: the BASELINE.json parity gates.

  logZ      |dA| <= 1e-5 * max(1, |A|)            (reading R7)
  marginals max |d mu| <= 1e-4 absolute
  Viterbi   path bit-identical, fp32 score == fp32(oracle score)  (dyadic inputs)
  flags     identical
"""
import math

import numpy as np

LOGZ_RTOL = 1e-5
MARG_ATOL = 1e-4


def check_logz(gpu, ref, flags_ref=None):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    for b in range(len(ref)):
        r, g = ref[b], gpu[b]
        if math.isnan(r):
            assert math.isnan(g), (b, g, r)
        elif math.isinf(r):
            assert g == r, (b, g, r)
        else:
            assert abs(g - r) <= LOGZ_RTOL * max(1.0, abs(r)), (b, g, r, abs(g - r))


def check_marg(gpu, ref, atol=MARG_ATOL):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert gpu.shape == ref.shape
    assert np.isfinite(gpu).all()
    err = np.abs(gpu - ref)
    worst = float(err.max()) if err.size else 0.0
    assert worst <= atol, f"max |d mu| = {worst:.3e} at {np.unravel_index(err.argmax(), err.shape)}"
    return worst


def check_viterbi(path, score, ref_path, ref_score):
    np.testing.assert_array_equal(np.asarray(path), np.asarray(ref_path))
    s = np.asarray(score, dtype=np.float32)
    r = np.asarray(ref_score, dtype=np.float64).astype(np.float32)
    same = (s == r) | (np.isnan(s) & np.isnan(r))
    assert same.all(), (s[~same], r[~same])
