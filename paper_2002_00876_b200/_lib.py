"""ctypes binding of libts_b200.so (include/ts_b200.h).  Argument marshalling only.

The library is built in-tree by `make` / `__graft_entry__.build()`; importing this
module without it raises immediately — there is no CPU fallback anywhere.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# TS_B200_LIB: an alternative in-tree build of the same library (kernel-variant experiments)
LIB_PATH = os.environ.get("TS_B200_LIB") or os.path.join(_HERE, "libts_b200.so")

TS_LOG, TS_MAX = 0, 1
TS_OP_LOGZ, TS_OP_MARG, TS_OP_VITERBI, TS_OP_MARG_HOST, TS_OP_SEGMENT = 0, 1, 2, 3, 4
TS_OP_ENTROPY, TS_OP_SAMPLE, TS_OP_SEGMENT_VITERBI, TS_OP_KBEST = 5, 6, 7, 8
TS_OP_EXPECTATION = 9
TS_F_EMPTY, TS_F_NONFINITE, TS_F_BADLEN = 1, 2, 4
STATUS = {0: "TS_OK", 1: "TS_E_INVALID", 2: "TS_E_UNSUPPORTED", 3: "TS_E_WORKSPACE",
          4: "TS_E_CUDA"}

# Every symbol include/ts_b200.h declares (checked by tests/test_abi_cpu.py).
SYMBOLS = ("ts_workspace_bytes", "ts_logpartition", "ts_marginals", "ts_viterbi",
           "ts_marginals_host", "ts_segment_summary_bytes", "ts_segment_summary",
           "ts_segment_finish", "ts_set_plan_chunk", "ts_get_plan_chunk", "ts_set_small_cluster",
           "ts_set_tiny", "ts_set_wide_ring", "ts_set_tiny_early", "ts_set_host_pipeline", "ts_entropy", "ts_expectation", "ts_log_prob", "ts_sample",
           "ts_segment_viterbi_summary_bytes", "ts_segment_viterbi_summary",
           "ts_segment_viterbi_maps", "ts_segment_viterbi_finish",
           "ts_kbest_workspace_bytes", "ts_kbest", "ts_semimarkov_workspace_bytes",
           "ts_semimarkov", "ts_semimarkov_viterbi_workspace_bytes", "ts_semimarkov_viterbi",
           "ts_set_meet", "ts_set_vchunk_mm", "ts_set_kbest_split", "ts_set_viterbi_split", "ts_set_host_graphs",
           "ts_host_alloc", "ts_host_free", "ts_set_tc_summary", "ts_get_tc_summary",
           "ts_last_launch_count", "ts_last_kernel", "ts_status_str", "ts_version")


class ts_chain(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int64), ("N", ctypes.c_int64), ("C", ctypes.c_int64),
                ("pot", ctypes.c_void_p), ("lengths", ctypes.c_void_p)]


class TsError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)} "
                         f"({_lib.ts_status_str(status).decode() if _lib else ''})")


_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build the CUDA library first "
                           "(python -c 'import __graft_entry__ as g; g.build()'); "
                           "there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P, I64, SZ, INT = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t, ctypes.c_int
    CH = ctypes.POINTER(ts_chain)
    L.ts_workspace_bytes.argtypes = [CH, INT, INT]
    L.ts_workspace_bytes.restype = SZ
    L.ts_logpartition.argtypes = [CH, INT, P, P, P, SZ, P]
    L.ts_marginals.argtypes = [CH, INT, P, P, P, P, SZ, P]
    L.ts_viterbi.argtypes = [CH, P, P, P, P, SZ, P]
    L.ts_marginals_host.argtypes = [CH, INT, P, P, P, P, SZ, P]
    L.ts_segment_summary_bytes.argtypes = [CH]
    L.ts_segment_summary_bytes.restype = SZ
    L.ts_segment_summary.argtypes = [CH, I64, I64, INT, P, P, SZ, P]
    L.ts_segment_finish.argtypes = [CH, I64, I64, INT, INT, INT, P, P, P, P, P, SZ, P]
    L.ts_entropy.argtypes = [CH, P, P, P, P, P, SZ, P]
    L.ts_expectation.argtypes = [CH, P, P, P, P, P, P, SZ, P]
    L.ts_semimarkov_workspace_bytes.argtypes = [CH, I64]
    L.ts_semimarkov_workspace_bytes.restype = SZ
    L.ts_semimarkov.argtypes = [CH, I64, P, P, P, P, SZ, P]
    L.ts_semimarkov_viterbi_workspace_bytes.argtypes = [CH, I64]
    L.ts_semimarkov_viterbi_workspace_bytes.restype = SZ
    L.ts_semimarkov_viterbi.argtypes = [CH, I64, P, P, P, P, SZ, P]
    L.ts_kbest_workspace_bytes.argtypes = [CH, I64]
    L.ts_kbest_workspace_bytes.restype = SZ
    L.ts_kbest.argtypes = [CH, I64, P, P, P, P, SZ, P]
    L.ts_segment_viterbi_summary_bytes.argtypes = [CH]
    L.ts_segment_viterbi_summary_bytes.restype = SZ
    L.ts_segment_viterbi_summary.argtypes = [CH, I64, I64, P, P]
    L.ts_segment_viterbi_maps.argtypes = [CH, I64, I64, INT, INT, P, P, P, P, P, SZ, P]
    L.ts_segment_viterbi_finish.argtypes = [CH, I64, I64, INT, INT, P, P, P, SZ, P]
    L.ts_log_prob.argtypes = [CH, P, P, P, P]
    L.ts_sample.argtypes = [CH, P, I64, P, P, P, P, SZ, P]
    for f in ("ts_logpartition", "ts_marginals", "ts_viterbi", "ts_marginals_host",
              "ts_segment_summary", "ts_segment_finish", "ts_entropy", "ts_expectation", "ts_log_prob",
              "ts_sample", "ts_segment_viterbi_summary", "ts_segment_viterbi_maps",
              "ts_segment_viterbi_finish", "ts_kbest", "ts_semimarkov", "ts_semimarkov_viterbi"):
        getattr(L, f).restype = INT
    L.ts_set_plan_chunk.argtypes = [I64]
    L.ts_set_plan_chunk.restype = None
    L.ts_get_plan_chunk.restype = I64
    L.ts_set_small_cluster.argtypes = [INT]
    L.ts_set_small_cluster.restype = None
    L.ts_last_kernel.argtypes = []
    L.ts_last_kernel.restype = ctypes.c_char_p
    L.ts_set_tiny.argtypes = [INT]
    L.ts_set_tiny.restype = None
    L.ts_set_wide_ring.argtypes = [INT]
    L.ts_set_wide_ring.restype = None
    L.ts_set_tiny_early.argtypes = [INT]
    L.ts_set_tiny_early.restype = None
    L.ts_set_host_pipeline.argtypes = [INT]
    L.ts_set_host_pipeline.restype = None
    L.ts_set_meet.argtypes = [INT]
    L.ts_set_meet.restype = None
    L.ts_set_vchunk_mm.argtypes = [INT]
    L.ts_set_vchunk_mm.restype = None
    L.ts_set_kbest_split.argtypes = [INT]
    L.ts_set_kbest_split.restype = None
    L.ts_set_viterbi_split.argtypes = [INT]
    L.ts_set_viterbi_split.restype = None
    L.ts_set_host_graphs.argtypes = [INT]
    L.ts_set_host_graphs.restype = None
    L.ts_set_tc_summary.argtypes = [INT]
    L.ts_set_tc_summary.restype = None
    L.ts_get_tc_summary.restype = INT
    L.ts_host_alloc.argtypes = [SZ]
    L.ts_host_alloc.restype = P
    L.ts_host_free.argtypes = [P]
    L.ts_host_free.restype = None
    L.ts_last_launch_count.restype = INT
    L.ts_status_str.argtypes = [INT]
    L.ts_status_str.restype = ctypes.c_char_p
    L.ts_version.restype = ctypes.c_char_p
    _lib = L
    return L


def check(status: int, where: str) -> None:
    if status != 0:
        raise TsError(status, where)
