"""CPU-side checks of the C ABI boundary (no compute, no GPU needed).

* the shared library loads and exports every entry point include/ts_b200.h declares;
* argument validation returns TS_E_INVALID before touching any device;
* workspace sizing is consistent (monotone in B, zero-size for the fused small plan);
* the Python binding fails loudly (no CPU fallback) when the library is absent.
"""
import ctypes
import os
import re

import pytest

from paper_2002_00876_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ts_b200.h")).read()
    return sorted(set(re.findall(r"TS_API\s+[\w\s\*]+?\b(ts_\w+)\s*\(", src)))


def test_header_symbols_exported():
    L = _lib.load()
    decl = declared_symbols()
    assert len(decl) >= 13
    assert sorted(_lib.SYMBOLS) == decl
    for name in decl:
        assert hasattr(L, name), name
    assert L.ts_version().decode().startswith("ts_b200")
    assert b"WORKSPACE" in L.ts_status_str(3)


def _chain(B=2, N=5, C=3, pot=0x1000, lengths=None):
    return _lib.ts_chain(B, N, C, pot, lengths)


@pytest.mark.parametrize("kw", [dict(B=0), dict(N=0), dict(C=0), dict(C=257), dict(pot=0),
                                dict(pot=0x1004)])
def test_invalid_chains_rejected(kw):
    L = _lib.load()
    ch = _chain(**kw)
    logz = ctypes.c_void_p(0x2000)
    assert L.ts_logpartition(ctypes.byref(ch), 0, logz, None, None, 0, None) == 1
    assert L.ts_workspace_bytes(ctypes.byref(ch), 1, 0) == 0


def test_invalid_outputs_rejected():
    L = _lib.load()
    ch = _chain()
    assert L.ts_logpartition(ctypes.byref(ch), 0, None, None, None, 0, None) == 1  # logz NULL
    assert L.ts_marginals(ctypes.byref(ch), 0, 0x3008, 0x2000, None, None, 0, None) == 1  # misaligned
    assert L.ts_viterbi(ctypes.byref(ch), None, 0x2000, None, None, 0, None) == 1
    assert L.ts_logpartition(ctypes.byref(ch), 7, 0x2000, None, None, 0, None) == 1  # semiring
    assert L.ts_logpartition(None, 0, 0x2000, None, None, 0, None) == 1


def test_workspace_sizes():
    L = _lib.load()
    small = _chain(B=32, N=25, C=20)
    assert L.ts_workspace_bytes(ctypes.byref(small), _lib.TS_OP_MARG, _lib.TS_LOG) == 0
    big = _chain(B=4, N=512, C=64)
    big2 = _chain(B=8, N=512, C=64)
    w1 = L.ts_workspace_bytes(ctypes.byref(big), _lib.TS_OP_MARG, _lib.TS_LOG)
    w2 = L.ts_workspace_bytes(ctypes.byref(big2), _lib.TS_OP_MARG, _lib.TS_LOG)
    assert 0 < w1 < w2
    assert w1 >= 4 * 512 * 64 * 4  # holds the forward vectors [B][N][C]
    v = L.ts_workspace_bytes(ctypes.byref(_chain(B=64, N=1024, C=256)), _lib.TS_OP_VITERBI,
                             _lib.TS_MAX)
    assert v >= 64 * 1023 * 256  # uint8 backpointers
    h = L.ts_workspace_bytes(ctypes.byref(small), _lib.TS_OP_MARG_HOST, _lib.TS_LOG)
    assert h >= 2 * 32 * 24 * 400 * 4


def test_plan_knob_roundtrip():
    L = _lib.load()
    L.ts_set_plan_chunk(7)
    assert L.ts_get_plan_chunk() == 7
    L.ts_set_plan_chunk(0)
    assert L.ts_get_plan_chunk() == 0


def test_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.load()


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2002_00876_b200")
    banned = ("import oracle", "from oracle", "liboracle", "oracle.c", "oracle/")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                for b in banned:
                    assert b not in txt, (f, b)


def test_next_row_entry_points_validate_before_the_device():
    """The §8(f) / time-sharding entry points reject bad arguments with TS_E_INVALID and,
    with valid arguments on a machine without an sm_100 device, return TS_E_UNSUPPORTED
    (there is no CPU fallback) — never a silent success."""
    L = _lib.load()
    ch = _chain()
    A = 0x2000  # an aligned dummy device address (never dereferenced on these paths)
    # entropy: marg / logz / entropy required
    assert L.ts_entropy(ctypes.byref(ch), None, A, A, None, None, 0, None) == 1
    assert L.ts_entropy(ctypes.byref(ch), A, None, A, None, None, 0, None) == 1
    assert L.ts_entropy(ctypes.byref(ch), A, A, None, None, None, 0, None) == 1
    # expectation: the feature r is required too (and 16-byte aligned)
    assert L.ts_expectation(ctypes.byref(ch), None, A, A, A, None, None, 0, None) == 1
    assert L.ts_expectation(ctypes.byref(ch), A + 4, A, A, A, None, None, 0, None) == 1
    assert L.ts_expectation(ctypes.byref(ch), A, None, A, A, None, None, 0, None) == 1
    # log_prob: z and out required
    assert L.ts_log_prob(ctypes.byref(ch), None, None, A, None) == 1
    assert L.ts_log_prob(ctypes.byref(ch), A, None, None, None) == 1
    # sample: uniforms, K >= 1, z, logz
    assert L.ts_sample(ctypes.byref(ch), None, 1, A, A, None, None, 0, None) == 1
    assert L.ts_sample(ctypes.byref(ch), A, 0, A, A, None, None, 0, None) == 1
    # kbest: 1 <= K <= 16
    assert L.ts_kbest(ctypes.byref(ch), 0, A, A, None, None, 0, None) == 1
    assert L.ts_kbest(ctypes.byref(ch), 17, A, A, None, None, 0, None) == 1
    assert L.ts_kbest_workspace_bytes(ctypes.byref(ch), 17) == 0
    assert L.ts_kbest_workspace_bytes(ctypes.byref(ch), 4) >= 2 * 4 * 3 * 4 * 2
    # semimarkov: 1 <= K <= 16, logz required
    assert L.ts_semimarkov(ctypes.byref(ch), 0, None, A, None, None, 0, None) == 1
    assert L.ts_semimarkov(ctypes.byref(ch), 2, None, None, None, None, 0, None) == 1
    # time-sharded Viterbi: lengths must be NULL, rank in [0, world)
    chl = _chain(lengths=0x3000)
    assert L.ts_segment_viterbi_summary(ctypes.byref(chl), 0, 5, A, None) == 1
    assert L.ts_segment_viterbi_maps(ctypes.byref(ch), 0, 5, 2, 2, A, A, None, None, None, 0,
                                     None) == 1
    assert L.ts_segment_viterbi_summary_bytes(ctypes.byref(ch)) == 2 * 3 * 3 * 4
    # valid arguments, no sm_100 device here -> TS_E_UNSUPPORTED
    import torch

    if not torch.cuda.is_available():
        assert L.ts_log_prob(ctypes.byref(ch), A, None, A, None) == 2
        assert L.ts_kbest(ctypes.byref(ch), 4, A, A, None, A, 1 << 20, None) == 2
        assert L.ts_semimarkov(ctypes.byref(ch), 2, None, A, None, A, 1 << 20, None) == 2


def test_next_row_workspace_sizes():
    L = _lib.load()
    ch = _chain(B=4, N=100, C=20)
    assert L.ts_workspace_bytes(ctypes.byref(ch), _lib.TS_OP_ENTROPY, _lib.TS_LOG) >= 4 * 8
    assert (L.ts_workspace_bytes(ctypes.byref(ch), _lib.TS_OP_EXPECTATION, _lib.TS_LOG) ==
            L.ts_workspace_bytes(ctypes.byref(ch), _lib.TS_OP_ENTROPY, _lib.TS_LOG))
    assert L.ts_workspace_bytes(ctypes.byref(ch), _lib.TS_OP_SAMPLE, _lib.TS_LOG) >= 4 * 100 * 20 * 4
    assert L.ts_workspace_bytes(ctypes.byref(ch), _lib.TS_OP_SEGMENT_VITERBI,
                                _lib.TS_MAX) >= 4 * 99 * 20
    assert L.ts_semimarkov_workspace_bytes(ctypes.byref(ch), 4) >= 2 * 4 * 100 * 20 * 4
    big = _chain(B=4, N=100, C=200)
    # sampling for 128 < C <= 256 filters with the wide-label recursion (node vectors in ws)
    assert L.ts_workspace_bytes(ctypes.byref(big), _lib.TS_OP_SAMPLE, _lib.TS_LOG) >= 4 * 100 * 200 * 4
    assert L.ts_semimarkov_workspace_bytes(ctypes.byref(big), 4) >= 2 * 4 * 100 * 200 * 4
    # the log semiring for long chains with 128 < C <= 256 runs fb_wide (node vectors in ws)
    assert L.ts_workspace_bytes(ctypes.byref(big), _lib.TS_OP_MARG, _lib.TS_LOG) >= 2 * 4 * 100 * 200 * 4
