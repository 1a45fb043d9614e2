"""paper_2002_00876_b200 — B200-native linear-chain CRF hot path of Torch-Struct
(Rush 2020, arXiv 2002.00876): log-partition A(l), marginals dA/dl and the Viterbi
argmax, computed by hand-written sm_100a CUDA kernels behind a C ABI
(include/ts_b200.h).  This module only marshals arguments: torch provides device
memory and the current stream; every step of the computation runs in the kernels.

    logz, flags         = logpartition(pot, lengths=None, semiring="log")
    marg, logz, flags   = marginals(pot, lengths=None, semiring="log")
    path, score, flags  = viterbi(pot, lengths=None)

pot: float32 CUDA tensor [B, N-1, C, C] with pot[b, t, i, j] = l(z_t=i, z_{t+1}=j);
lengths: int32 CUDA tensor [B] in [1, N] or None.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import TS_F_BADLEN, TS_F_EMPTY, TS_F_NONFINITE, TsError  # noqa: F401

__all__ = ["logpartition", "marginals", "viterbi", "marginals_host", "host_empty", "set_plan_chunk",
           "get_plan_chunk", "last_launch_count", "workspace_bytes", "Workspace", "TsError",
           "Segment"]

_SEMI = {"log": _lib.TS_LOG, "max": _lib.TS_MAX}


def _semi(s) -> int:
    if isinstance(s, int):
        return s
    return _SEMI[s]


def _chain(pot: torch.Tensor, lengths, N: int | None = None) -> _lib.ts_chain:
    if pot.dim() != 4 or pot.shape[2] != pot.shape[3]:
        raise ValueError("pot must be [B, N-1, C, C]")
    if pot.dtype != torch.float32 or not pot.is_contiguous():
        raise ValueError("pot must be a contiguous float32 tensor")
    B, E, C, _ = pot.shape
    if lengths is not None:
        if lengths.dtype != torch.int32 or lengths.shape != (B,) or lengths.device != pot.device:
            raise ValueError("lengths must be an int32 tensor [B] on pot's device")
    return _lib.ts_chain(B, E + 1, C, pot.data_ptr() if pot.numel() else None,
                         lengths.data_ptr() if lengths is not None else None)


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class Workspace:
    """Caller-owned device workspace, grown on demand (one per device)."""

    _per_device: dict = {}

    def __init__(self, device):
        self.device = torch.device(device)
        self.buf = torch.empty(0, dtype=torch.uint8, device=self.device)

    @classmethod
    def get(cls, device, tag: str = "") -> "Workspace":
        d = torch.device(device)
        key = (d.type, d.index if d.index is not None else torch.cuda.current_device(), tag)
        ws = cls._per_device.get(key)
        if ws is None:
            ws = cls._per_device[key] = Workspace(d)
        return ws

    def ptr(self, nbytes: int) -> int:
        if nbytes == 0:
            return 0
        if self.buf.numel() < nbytes + 256:
            self.buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        p = self.buf.data_ptr()
        return (p + 255) & ~255


def workspace_bytes(pot, lengths=None, op: int = _lib.TS_OP_MARG, semiring="log") -> int:
    L = _lib.load()
    ch = _chain(pot, lengths)
    return int(L.ts_workspace_bytes(ctypes.byref(ch), op, _semi(semiring)))


def _ws(pot, ch, op, semi, ws):
    L = _lib.load()
    need = int(L.ts_workspace_bytes(ctypes.byref(ch), op, semi))
    ws = ws or Workspace.get(pot.device)
    return ws.ptr(need), need


def logpartition(pot: torch.Tensor, lengths=None, semiring="log", ws: Workspace | None = None):
    """A(l) per sequence (semiring='max' gives A*(l))."""
    L = _lib.load()
    ch = _chain(pot, lengths)
    semi = _semi(semiring)
    B = pot.shape[0]
    logz = torch.empty(B, dtype=torch.float32, device=pot.device)
    flags = torch.empty(B, dtype=torch.int32, device=pot.device)
    wp, wn = _ws(pot, ch, _lib.TS_OP_LOGZ, semi, ws)
    _lib.check(L.ts_logpartition(ctypes.byref(ch), semi, logz.data_ptr(), flags.data_ptr(), wp,
                                 wn, _stream(pot.device)), "ts_logpartition")
    return logz, flags


def marginals(pot: torch.Tensor, lengths=None, semiring="log", ws: Workspace | None = None,
              out: torch.Tensor | None = None):
    """dA/dl [B, N-1, C, C], logZ [B], flags [B]."""
    L = _lib.load()
    ch = _chain(pot, lengths)
    semi = _semi(semiring)
    B = pot.shape[0]
    marg = out if out is not None else torch.empty_like(pot)
    logz = torch.empty(B, dtype=torch.float32, device=pot.device)
    flags = torch.empty(B, dtype=torch.int32, device=pot.device)
    wp, wn = _ws(pot, ch, _lib.TS_OP_MARG, semi, ws)
    _lib.check(L.ts_marginals(ctypes.byref(ch), semi, marg.data_ptr(), logz.data_ptr(),
                              flags.data_ptr(), wp, wn, _stream(pot.device)), "ts_marginals")
    return marg, logz, flags


def viterbi(pot: torch.Tensor, lengths=None, ws: Workspace | None = None):
    """Canonical argmax labelling (reading R5): path [B, N], score [B], flags."""
    L = _lib.load()
    ch = _chain(pot, lengths)
    B, E = pot.shape[0], pot.shape[1]
    path = torch.empty((B, E + 1), dtype=torch.int32, device=pot.device)
    score = torch.empty(B, dtype=torch.float32, device=pot.device)
    flags = torch.empty(B, dtype=torch.int32, device=pot.device)
    wp, wn = _ws(pot, ch, _lib.TS_OP_VITERBI, _lib.TS_MAX, ws)
    _lib.check(L.ts_viterbi(ctypes.byref(ch), path.data_ptr(), score.data_ptr(), flags.data_ptr(),
                            wp, wn, _stream(pot.device)), "ts_viterbi")
    return path, score, flags


def entropy(pot: torch.Tensor, lengths=None, ws: Workspace | None = None,
            out: torch.Tensor | None = None):
    """Entropy H = A - Σ mu·l of the CRF: (H [B], marg, logZ, flags)."""
    L = _lib.load()
    ch = _chain(pot, lengths)
    B = pot.shape[0]
    marg = out if out is not None else torch.empty_like(pot)
    logz = torch.empty(B, dtype=torch.float32, device=pot.device)
    H = torch.empty(B, dtype=torch.float32, device=pot.device)
    flags = torch.empty(B, dtype=torch.int32, device=pot.device)
    wp, wn = _ws(pot, ch, _lib.TS_OP_ENTROPY, _lib.TS_LOG, ws)
    _lib.check(L.ts_entropy(ctypes.byref(ch), marg.data_ptr(), logz.data_ptr(), H.data_ptr(),
                            flags.data_ptr(), wp, wn, _stream(pot.device)), "ts_entropy")
    return H, marg, logz, flags


def expectation(pot: torch.Tensor, r: torch.Tensor, lengths=None, ws: Workspace | None = None,
                out: torch.Tensor | None = None):
    """E_p[Σ_p r_p z_p] = Σ mu·r of an additive feature r (same shape as pot; Table 2 'Exp.',
    P:207): (E [B], marg, logZ, flags)."""
    L = _lib.load()
    ch = _chain(pot, lengths)
    if r.shape != pot.shape or r.dtype != torch.float32 or r.device != pot.device:
        raise ValueError("expectation: r must be a float32 tensor shaped and placed like pot")
    r = r.contiguous()
    B = pot.shape[0]
    marg = out if out is not None else torch.empty_like(pot)
    logz = torch.empty(B, dtype=torch.float32, device=pot.device)
    ev = torch.empty(B, dtype=torch.float32, device=pot.device)
    flags = torch.empty(B, dtype=torch.int32, device=pot.device)
    wp, wn = _ws(pot, ch, _lib.TS_OP_EXPECTATION, _lib.TS_LOG, ws)
    _lib.check(L.ts_expectation(ctypes.byref(ch), r.data_ptr(), marg.data_ptr(), logz.data_ptr(),
                                ev.data_ptr(), flags.data_ptr(), wp, wn, _stream(pot.device)),
               "ts_expectation")
    return ev, marg, logz, flags


def log_prob(pot: torch.Tensor, z: torch.Tensor, lengths=None, logz: torch.Tensor | None = None):
    """log p(z) = Score(z) - A for labellings z [B, N] int32; with logz=None the
    partition is computed first (ts_logpartition)."""
    L = _lib.load()
    ch = _chain(pot, lengths)
    if logz is None:
        logz, _ = logpartition(pot, lengths)
    z = z.to(torch.int32).contiguous()
    out = torch.empty(pot.shape[0], dtype=torch.float32, device=pot.device)
    _lib.check(L.ts_log_prob(ctypes.byref(ch), z.data_ptr(), logz.data_ptr(), out.data_ptr(),
                             _stream(pot.device)), "ts_log_prob")
    return out


def score(pot: torch.Tensor, z: torch.Tensor, lengths=None):
    """Score(z) = Σ_t l[t, z_t, z_{t+1}] for labellings z [B, N]."""
    L = _lib.load()
    ch = _chain(pot, lengths)
    z = z.to(torch.int32).contiguous()
    out = torch.empty(pot.shape[0], dtype=torch.float32, device=pot.device)
    _lib.check(L.ts_log_prob(ctypes.byref(ch), z.data_ptr(), None, out.data_ptr(),
                             _stream(pot.device)), "ts_log_prob")
    return out


def sample(pot: torch.Tensor, uniforms: torch.Tensor, lengths=None, ws: Workspace | None = None):
    """K exact samples per sequence by forward-filtering backward-sampling
    driven by caller-supplied uniforms [K, B, N] in [0, 1): (z [K, B, N] int32, logZ, flags)."""
    L = _lib.load()
    ch = _chain(pot, lengths)
    u = uniforms.to(torch.float32).contiguous()
    K = u.shape[0]
    B, E = pot.shape[0], pot.shape[1]
    assert u.shape == (K, B, E + 1), u.shape
    z = torch.empty((K, B, E + 1), dtype=torch.int32, device=pot.device)
    logz = torch.empty(B, dtype=torch.float32, device=pot.device)
    flags = torch.empty(B, dtype=torch.int32, device=pot.device)
    wp, wn = _ws(pot, ch, _lib.TS_OP_SAMPLE, _lib.TS_LOG, ws)
    _lib.check(L.ts_sample(ctypes.byref(ch), u.data_ptr(), K, z.data_ptr(), logz.data_ptr(),
                           flags.data_ptr(), wp, wn, _stream(pot.device)), "ts_sample")
    return z, logz, flags


_HOST_NEED: dict = {}


def marginals_host(pot_host: torch.Tensor, marg_host: torch.Tensor, logz_host: torch.Tensor,
                   flags_host: torch.Tensor | None = None, lengths_host=None, semiring="log",
                   device=None, ws: Workspace | None = None):
    """End-to-end call with HOST (ideally pinned) buffers; copies happen inside the C ABI call.

    Enqueued on the current stream of `device`; synchronise before reading the outputs.
    Repeated calls with the same buffers replay a CUDA graph of the whole pipeline
    (include/ts_b200.h, ts_marginals_host).
    """
    L = _lib.load()
    device = torch.device(device or "cuda")
    B, E, C, _ = pot_host.shape
    ch = _lib.ts_chain(B, E + 1, C, pot_host.data_ptr() if pot_host.numel() else None,
                       lengths_host.data_ptr() if lengths_host is not None else None)
    semi = _semi(semiring)
    key = (B, E, C, semi, lengths_host is not None)
    need = _HOST_NEED.get(key)
    if need is None:
        need = _HOST_NEED[key] = int(L.ts_workspace_bytes(ctypes.byref(ch), _lib.TS_OP_MARG_HOST,
                                                          semi))
    # a workspace of its own: the cross-call copy pipeline writes the next call's input
    # staging while earlier work on the stream may still run (include/ts_b200.h)
    ws = ws or Workspace.get(device, "host")
    wp = ws.ptr(need)
    _lib.check(L.ts_marginals_host(ctypes.byref(ch), semi, marg_host.data_ptr(),
                                   logz_host.data_ptr(),
                                   flags_host.data_ptr() if flags_host is not None else None, wp,
                                   need, _stream(device)), "ts_marginals_host")


class _HostBlock:
    """Owner of one ts_host_alloc block; freed when the last tensor view is collected."""

    def __init__(self, nbytes: int):
        self.ptr = _lib.load().ts_host_alloc(nbytes)
        if not self.ptr:
            raise MemoryError(f"ts_host_alloc({nbytes}) failed")
        self.nbytes = nbytes

    def __del__(self):
        if getattr(self, "ptr", None):
            _lib.load().ts_host_free(self.ptr)
            self.ptr = None


def host_empty(shape, dtype=torch.float32) -> torch.Tensor:
    """Page-locked host tensor from the library allocator (ts_host_alloc), for the
    host-buffer entry point marginals_host."""
    n = 1
    for d in shape:
        n *= int(d)
    itemsize = torch.empty(0, dtype=dtype).element_size()
    nbytes = max(n * itemsize, 1)
    blk = _HostBlock(nbytes)
    buf = (ctypes.c_uint8 * nbytes).from_address(blk.ptr)
    buf._ts_owner = blk  # keep the block alive as long as the buffer is
    t = torch.frombuffer(buf, dtype=torch.uint8, count=n * itemsize)
    return t.view(dtype).view(*shape) if n else torch.empty(shape, dtype=dtype)


def set_tc_summary(mode: int) -> None:
    """Debug/testing: scan leaf summaries on tensor cores (3 = 3xTF32 default, 1 = 1xTF32,
    0 = SIMT fp32)."""
    _lib.load().ts_set_tc_summary(int(mode))


def get_tc_summary() -> int:
    return int(_lib.load().ts_get_tc_summary())


def set_host_pipeline(mode) -> None:
    """Debug knob: cross-call pipeline of marginals_host for single-chunk payloads: 2 (default,
    or True) = three stages on library streams, 1 = two-stream copy pipeline, 0 (or False) =
    every call fully ordered on its stream."""
    m = 2 if mode is True else (0 if mode is False else int(mode))
    _lib.load().ts_set_host_pipeline(m)


def set_host_graphs(enable: bool) -> None:
    """Debug/testing: graph replay of repeated ts_marginals_host bindings (default on)."""
    _lib.load().ts_set_host_graphs(1 if enable else 0)


class Segment:
    """One rank's contiguous time segment of a long chain (time sharding).

    Holds the device workspace (the local scan tree) between `summary()` and `finish()`.
    `local_pot` [B, E_local, C, C] holds global edges [edge_begin, edge_begin + E_local) of
    chains with `n_global` positions (full length; no per-sequence lengths).
    """

    def __init__(self, local_pot: torch.Tensor, edge_begin: int, n_global: int):
        self.pot = local_pot
        self.edge_begin = int(edge_begin)
        self.n_global = int(n_global)
        self.ch = _chain(local_pot, None)
        L = _lib.load()
        self.nbytes = int(L.ts_segment_summary_bytes(ctypes.byref(self.ch)))
        self.ws_bytes = int(L.ts_workspace_bytes(ctypes.byref(self.ch), _lib.TS_OP_SEGMENT,
                                                 _lib.TS_LOG))
        self.ws = Workspace(local_pot.device)
        self.wptr = self.ws.ptr(self.ws_bytes)

    def summary(self) -> torch.Tensor:
        """This segment's C x C transfer matrices (the local semiring product) as
        float32 words (ts_segment_summary_bytes / 4: the [B, C, C] matrices padded to 16 bytes,
        then the [B, C] fp64 row offsets, include/ts_b200.h)."""
        L = _lib.load()
        out = torch.empty(self.nbytes // 4, dtype=torch.float32, device=self.pot.device)
        _lib.check(L.ts_segment_summary(ctypes.byref(self.ch), self.edge_begin, self.n_global,
                                        _lib.TS_LOG, out.data_ptr(), self.wptr, self.ws_bytes,
                                        _stream(self.pot.device)), "ts_segment_summary")
        return out

    def finish(self, all_summaries: torch.Tensor, rank: int, world: int, want_marg: bool = True):
        """Combine the gathered summaries [world, nbytes/4] (rank order) -> (marg|None, logz, flags)."""
        L = _lib.load()
        B = self.pot.shape[0]
        dev = self.pot.device
        all_summaries = all_summaries.contiguous()
        marg = torch.empty_like(self.pot) if want_marg else None
        logz = torch.empty(B, dtype=torch.float32, device=dev)
        flags = torch.empty(B, dtype=torch.int32, device=dev)
        _lib.check(L.ts_segment_finish(ctypes.byref(self.ch), self.edge_begin, self.n_global,
                                       int(rank), int(world), _lib.TS_LOG,
                                       all_summaries.data_ptr(),
                                       marg.data_ptr() if want_marg else None, logz.data_ptr(),
                                       flags.data_ptr(), self.wptr, self.ws_bytes, _stream(dev)),
                   "ts_segment_finish")
        return marg, logz, flags


def semimarkov(pot: torch.Tensor, lengths=None, want_marg: bool = True,
               ws: Workspace | None = None):
    """Semi-Markov CRF (Table 1; reading R17): pot [B, N-1, K, C, C] ->
    (marg (same shape) | None, logZ [B], flags [B])."""
    L = _lib.load()
    assert pot.dim() == 5 and pot.is_contiguous()
    B, E, K, C, _ = pot.shape
    ch = _lib.ts_chain(B, E + 1, C, pot.data_ptr(),
                       lengths.data_ptr() if lengths is not None else None)
    marg = torch.empty_like(pot) if want_marg else None
    logz = torch.empty(B, dtype=torch.float32, device=pot.device)
    flags = torch.empty(B, dtype=torch.int32, device=pot.device)
    need = int(L.ts_semimarkov_workspace_bytes(ctypes.byref(ch), int(K)))
    ws = ws or Workspace.get(pot.device)
    _lib.check(L.ts_semimarkov(ctypes.byref(ch), int(K), marg.data_ptr() if want_marg else None,
                               logz.data_ptr(), flags.data_ptr(), ws.ptr(need), need,
                               _stream(pot.device)), "ts_semimarkov")
    return marg, logz, flags


def semimarkov_viterbi(pot: torch.Tensor, lengths=None, ws: Workspace | None = None):
    """Semi-Markov Viterbi (readings R17/R18): pot [B, N-1, K, C, C] -> (seg [B, N] int32:
    the label at each segment boundary node, -1 elsewhere; score [B]; flags [B])."""
    L = _lib.load()
    assert pot.dim() == 5 and pot.is_contiguous()
    B, E, K, C, _ = pot.shape
    ch = _lib.ts_chain(B, E + 1, C, pot.data_ptr(),
                       lengths.data_ptr() if lengths is not None else None)
    seg = torch.empty((B, E + 1), dtype=torch.int32, device=pot.device)
    score = torch.empty(B, dtype=torch.float32, device=pot.device)
    flags = torch.empty(B, dtype=torch.int32, device=pot.device)
    need = int(L.ts_semimarkov_viterbi_workspace_bytes(ctypes.byref(ch), int(K)))
    ws = ws or Workspace.get(pot.device)
    _lib.check(L.ts_semimarkov_viterbi(ctypes.byref(ch), int(K), seg.data_ptr(), score.data_ptr(),
                                       flags.data_ptr(), ws.ptr(need), need, _stream(pot.device)),
               "ts_semimarkov_viterbi")
    return seg, score, flags


def kbest(pot: torch.Tensor, K: int, lengths=None, ws: Workspace | None = None):
    """The K best labelings (Table 2 'K-Max'; order: score desc, then reverse-
    lexicographic): (paths [B, K, N] int32, scores [B, K], flags [B])."""
    L = _lib.load()
    ch = _chain(pot, lengths)
    B, E = pot.shape[0], pot.shape[1]
    paths = torch.empty((B, K, E + 1), dtype=torch.int32, device=pot.device)
    scores = torch.empty((B, K), dtype=torch.float32, device=pot.device)
    flags = torch.empty(B, dtype=torch.int32, device=pot.device)
    need = int(L.ts_kbest_workspace_bytes(ctypes.byref(ch), int(K)))
    ws = ws or Workspace.get(pot.device)
    _lib.check(L.ts_kbest(ctypes.byref(ch), int(K), paths.data_ptr(), scores.data_ptr(),
                          flags.data_ptr(), ws.ptr(need), need, _stream(pot.device)), "ts_kbest")
    return paths, scores, flags


class ViterbiSegment:
    """One rank's contiguous time segment for time-sharded Viterbi: the
    max-plus summary, then (after gathering every rank's summary) the end-label maps, then
    (after gathering the maps) the local path.  Holds the backpointer workspace between
    maps() and finish()."""

    def __init__(self, local_pot: torch.Tensor, edge_begin: int, n_global: int):
        self.pot = local_pot
        self.edge_begin = int(edge_begin)
        self.n_global = int(n_global)
        self.ch = _chain(local_pot, None)
        L = _lib.load()
        self.nbytes = int(L.ts_segment_viterbi_summary_bytes(ctypes.byref(self.ch)))
        self.ws_bytes = int(L.ts_workspace_bytes(ctypes.byref(self.ch),
                                                 _lib.TS_OP_SEGMENT_VITERBI, _lib.TS_MAX))
        self.ws = Workspace(local_pot.device)
        self.wptr = self.ws.ptr(self.ws_bytes)

    def summary(self) -> torch.Tensor:
        """Max-plus transfer matrices of the local edges [B, C, C] (Table 2 'Max')."""
        L = _lib.load()
        B, _, C, _ = self.pot.shape
        out = torch.empty((B, C, C), dtype=torch.float32, device=self.pot.device)
        _lib.check(L.ts_segment_viterbi_summary(ctypes.byref(self.ch), self.edge_begin,
                                                self.n_global, out.data_ptr(),
                                                _stream(self.pot.device)),
                   "ts_segment_viterbi_summary")
        return out

    def maps(self, all_summaries: torch.Tensor, rank: int, world: int):
        """-> (maps [B, C] int32, global score [B], flags [B])."""
        L = _lib.load()
        B, _, C, _ = self.pot.shape
        dev = self.pot.device
        all_summaries = all_summaries.contiguous()
        maps = torch.empty((B, C), dtype=torch.int32, device=dev)
        score = torch.empty(B, dtype=torch.float32, device=dev)
        flags = torch.empty(B, dtype=torch.int32, device=dev)
        _lib.check(L.ts_segment_viterbi_maps(ctypes.byref(self.ch), self.edge_begin,
                                             self.n_global, int(rank), int(world),
                                             all_summaries.data_ptr(), maps.data_ptr(),
                                             score.data_ptr(), flags.data_ptr(), self.wptr,
                                             self.ws_bytes, _stream(dev)),
                   "ts_segment_viterbi_maps")
        return maps, score, flags

    def finish(self, all_maps: torch.Tensor, rank: int, world: int) -> torch.Tensor:
        """-> local path [B, E_local + 1] int32 (global nodes edge_begin ...)."""
        L = _lib.load()
        B, E = self.pot.shape[0], self.pot.shape[1]
        dev = self.pot.device
        all_maps = all_maps.to(torch.int32).contiguous()
        path = torch.empty((B, E + 1), dtype=torch.int32, device=dev)
        _lib.check(L.ts_segment_viterbi_finish(ctypes.byref(self.ch), self.edge_begin,
                                               self.n_global, int(rank), int(world),
                                               all_maps.data_ptr(), path.data_ptr(), self.wptr,
                                               self.ws_bytes, _stream(dev)),
                   "ts_segment_viterbi_finish")
        return path


def set_plan_chunk(L: int) -> None:
    """Debug knob: 0 auto, 1 = pure Fig. 4 tree, >= N-1 = serial sweep."""
    _lib.load().ts_set_plan_chunk(int(L))


def set_small_cluster(G: int) -> None:
    """Plan knob for short C % 4 == 0, C <= 28 chains: the §6(a) chunked scan on a G-CTA
    cluster per sequence (fb_cscan.cu).  0 = one CTA per sequence (default), -1 = auto,
    2 / 4 = force G where the shape fits."""
    _lib.load().ts_set_small_cluster(int(G))


def set_tiny(enable: bool) -> None:
    """Debug knob: latency-optimised short-chain kernel for C % 4 == 0, C <= 28 (default on)."""
    _lib.load().ts_set_tiny(1 if enable else 0)


def set_wide_ring(enable: bool) -> None:
    """Debug knob: bulk-copy SMEM ring for the wide-label (128 < C <= 256) log path."""
    _lib.load().ts_set_wide_ring(1 if enable else 0)


def set_tiny_early(enable: bool) -> None:
    """Debug knob: fb_tiny reads its inputs before the PDL wait when no recent call's outputs
    overlap them (default on); off = wait first.  Identical results."""
    _lib.load().ts_set_tiny_early(1 if enable else 0)


def set_meet(enable: bool) -> None:
    """Debug knob: meet-in-the-middle fused marginals kernel for C = 64 (default on)."""
    _lib.load().ts_set_meet(1 if enable else 0)


def set_vchunk_mm(enable: bool) -> None:
    """Debug knob: register-blocked max-plus chunk summaries of the chunked Viterbi for
    C in {32, 64, 128} (default on; off = row-chain summaries, auto plan serial)."""
    _lib.load().ts_set_vchunk_mm(1 if enable else 0)


def set_kbest_split(S: int) -> None:
    """Debug knob: K-best lanes per label column (0 auto, 1/2/4/8); results bit-identical."""
    _lib.load().ts_set_kbest_split(int(S))


def set_viterbi_split(G: int) -> None:
    """Debug knob: Viterbi C in {128,256} cluster size (0 auto, 1/2/4/8 forced, -1 legacy)."""
    _lib.load().ts_set_viterbi_split(int(G))


def get_plan_chunk() -> int:
    return int(_lib.load().ts_get_plan_chunk())


def last_kernel() -> str:
    """Dominant kernel of this thread's last hot-path call (measurement / profiling)."""
    return _lib.load().ts_last_kernel().decode()


def last_launch_count() -> int:
    return int(_lib.load().ts_last_launch_count())
