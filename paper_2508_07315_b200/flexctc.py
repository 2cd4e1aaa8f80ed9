"""Thin Python binding of libflexctc.so (include/flexctc.h): argument marshalling only.

Every step of the decode runs in the library's CUDA kernels; torch provides device memory and
streams. There is no CPU path: if the shared library is missing or cannot be loaded, importing
this module raises, and `decode` refuses tensors that are not on a CUDA device.

Names follow the C ABI: lm_load, boost_build, decode, decode_host, workspace_bytes, check.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

FLEXCTC_OK = 0
_STATUS = {0: "OK", 1: "INVALID_ARG", 2: "PARSE", 3: "VOCAB_BIND", 4: "CAPACITY", 5: "CUDA", 6: "OOM", 7: "IO"}
FLAG_LENGTH_CLAMPED_HIGH = 1
FLAG_LENGTH_CLAMPED_LOW = 2


class FlexCTCError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"flexctc {_STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    """flexctc_config (Eq. (1) weights P:96-98, θ P:237)."""
    _fields_ = [("beam", ctypes.c_int32), ("alpha_lm", ctypes.c_float), ("alpha_bt", ctypes.c_float),
                ("beta", ctypes.c_float), ("theta", ctypes.c_float), ("merge_mode", ctypes.c_int32),
                ("retract_boost_at_eos", ctypes.c_int32), ("fuse_repeats", ctypes.c_int32),
                ("merge_first", ctypes.c_int32)]


def config(beam: int, alpha_lm: float = 0.0, alpha_bt: float = 0.0, beta: float = 0.0,
           theta: float = 12.0, merge_mode: int = 0, retract_boost_at_eos: int = 0, fuse_repeats: int = 0,
           merge_first: int = 0) -> Config:
    return Config(int(beam), float(alpha_lm), float(alpha_bt), float(beta), float(theta), int(merge_mode),
                  int(retract_boost_at_eos), int(fuse_repeats), int(merge_first))


class LmInfo(ctypes.Structure):
    _fields_ = [("order", ctypes.c_int32), ("vocab_size", ctypes.c_int32), ("n_states", ctypes.c_int32),
                ("start_state", ctypes.c_int32), ("n_arcs", ctypes.c_int64), ("device_bytes", ctypes.c_int64)]


EXPORTS = [
    "flexctc_last_error", "flexctc_version", "flexctc_lm_load", "flexctc_lm_free", "flexctc_lm_get_info",
    "flexctc_lm_host_query", "flexctc_lm_host_query_batch", "flexctc_lm_host_bound", "flexctc_boost_build", "flexctc_boost_free", "flexctc_boost_host_query",
    "flexctc_boost_num_nodes", "flexctc_boost_host_query_batch", "flexctc_boost_host_signature", "flexctc_workspace_bytes", "flexctc_decode", "flexctc_check",
    "flexctc_host_scratch_bytes", "flexctc_decode_host", "flexctc_host_streaming", "flexctc_decode_nbest", "flexctc_decode_logits_bf16", "flexctc_logits_workspace_bytes", "flexctc_set_profile_events", "flexctc_set_stage_events", "flexctc_last_kernel", "flexctc_get_stats",
    "flexctc_host_scratch_bytes_bf16", "flexctc_decode_host_bf16",
]
STAT_NAMES = ["frames", "alive_slots", "listed_tokens", "exact_sparse", "dense_frames", "lm_rows_built",
              "exact_dense", "compactions", "top_token_stages", "deferred_next",
              "cyc_phase1_3", "cyc_phase4", "cyc_lm_rows", "cyc_phase5", "cyc_phase6_7", "heavy_frames",
              "cyc_heavy_frames", "cyc_frame_top", "cyc_phase2", "cyc_phase3", "cyc_p4_setup", "cyc_p4_collect",
              "cyc_p4_eval", "light_frames", "lcyc_p1", "lcyc_p2", "lcyc_p3", "lcyc_b1", "lcyc_p5", "lcyc_p6",
              "lcyc_p7", "lcyc_p7a", "lcyc_p7b", "lcyc_p7c", "lcyc_p7d", "fast_frames", "cyc_fast"]


def _load() -> ctypes.CDLL:
    path = os.environ.get("FLEXCTC_LIB_AB")  # A/B timing of two builds (tools/ab.sh); never a fallback
    if path:
        return _declare(ctypes.CDLL(path))
    path = _build.lib_path()  # libflexctc.so, or libflexctc_timers.so under FLEXCTC_PHASE_TIMERS=1
    if not _build.up_to_date():
        _build.build()  # missing or stale (sources newer); nvcc is part of the image, failures raise
    return _declare(ctypes.CDLL(path))


def _declare(L: ctypes.CDLL) -> ctypes.CDLL:
    vp, i32, i64, f32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_size_t
    P = ctypes.POINTER
    L.flexctc_last_error.restype = ctypes.c_char_p
    L.flexctc_version.restype = ctypes.c_char_p
    L.flexctc_lm_load.argtypes = [ctypes.c_char_p, i32, vp, i32, P(vp)]
    L.flexctc_lm_free.argtypes = [vp]
    L.flexctc_lm_free.restype = None
    L.flexctc_lm_get_info.argtypes = [vp, P(LmInfo)]
    L.flexctc_lm_host_query.argtypes = [vp, i32, i32, P(f32), P(i32)]
    L.flexctc_boost_build.argtypes = [vp, vp, i32, f32, i32, i32, P(vp)]
    L.flexctc_boost_free.argtypes = [vp]
    L.flexctc_boost_free.restype = None
    L.flexctc_boost_host_query.argtypes = [vp, i32, i32, P(f32), P(i32), P(f32)]
    L.flexctc_boost_num_nodes.argtypes = [vp, P(i32)]
    L.flexctc_lm_host_query_batch.argtypes = [vp, i64, vp, vp, vp, vp]
    L.flexctc_lm_host_bound.argtypes = [vp, i32, P(f32), P(f32)]
    L.flexctc_boost_host_query_batch.argtypes = [vp, i64, vp, vp, vp, vp]
    L.flexctc_boost_host_signature.argtypes = [vp, i32, P(ctypes.c_uint64)]
    L.flexctc_workspace_bytes.argtypes = [i32, i32, i32, P(Config)]
    L.flexctc_workspace_bytes.restype = sz
    L.flexctc_decode.argtypes = [vp, i64, i64, vp, i32, i32, i32, P(Config), vp, vp, vp, sz, vp,
                                 vp, vp, vp, vp, vp]
    L.flexctc_decode_nbest.argtypes = [vp, i64, i64, vp, i32, i32, i32, P(Config), vp, vp, vp, sz, vp, i32,
                                       vp, vp, vp, vp]
    L.flexctc_logits_workspace_bytes.argtypes = [i32, i32, i32, P(Config)]
    L.flexctc_logits_workspace_bytes.restype = sz
    L.flexctc_decode_logits_bf16.argtypes = [vp, i64, i64, vp, i32, i32, i32, P(Config), vp, vp, vp, sz, vp,
                                             vp, vp, vp, vp, vp]
    L.flexctc_check.argtypes = [vp, P(ctypes.c_uint32)]
    L.flexctc_host_scratch_bytes.argtypes = [i32, i32, i32, P(Config)]
    L.flexctc_host_scratch_bytes.restype = sz
    L.flexctc_decode_host.argtypes = [vp, vp, i32, i32, i32, P(Config), vp, vp, vp, sz, vp, vp, vp, vp, vp,
                                      P(ctypes.c_uint32)]
    L.flexctc_host_scratch_bytes_bf16.argtypes = [i32, i32, i32, P(Config)]
    L.flexctc_host_scratch_bytes_bf16.restype = sz
    L.flexctc_decode_host_bf16.argtypes = [vp, vp, i32, i32, i32, P(Config), vp, vp, vp, sz, vp, vp, vp, vp, vp,
                                           P(ctypes.c_uint32)]
    L.flexctc_host_streaming.argtypes = []
    L.flexctc_host_streaming.restype = i32
    L.flexctc_set_profile_events.argtypes = [vp, vp]
    L.flexctc_set_profile_events.restype = None
    L.flexctc_set_stage_events.argtypes = [ctypes.c_int32, vp, vp]
    L.flexctc_set_stage_events.restype = ctypes.c_int
    L.flexctc_last_kernel.restype = ctypes.c_char_p
    L.flexctc_get_stats.argtypes = [vp, vp, i32]
    for name in EXPORTS:
        getattr(L, name)  # AttributeError if a declared symbol is missing
    return L


lib = _load()


def last_error() -> str:
    return lib.flexctc_last_error().decode()


def _check(st: int):
    if st != FLEXCTC_OK:
        raise FlexCTCError(st, last_error())


def version() -> str:
    return lib.flexctc_version().decode()


class LM:
    """flexctc_lm handle (flexctc_lm_load). device=-1 builds a host-only handle for inspection."""

    def __init__(self, arpa_path: str, vocab_size: int, symbols=None, device: int = 0):
        syms = None
        if symbols is not None:
            self._syms = (ctypes.c_char_p * vocab_size)(*[s.encode() for s in symbols])
            syms = ctypes.cast(self._syms, ctypes.c_void_p)
        h = ctypes.c_void_p()
        _check(lib.flexctc_lm_load(arpa_path.encode(), int(vocab_size), syms, int(device), ctypes.byref(h)))
        self.h = h
        self.vocab_size = vocab_size
        self.device = device

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:
            lib.flexctc_lm_free(self.h)
            self.h = None

    def info(self) -> LmInfo:
        i = LmInfo()
        _check(lib.flexctc_lm_get_info(self.h, ctypes.byref(i)))
        return i

    def host_query(self, state: int, token: int):
        lp, nx = ctypes.c_float(), ctypes.c_int32()
        _check(lib.flexctc_lm_host_query(self.h, int(state), int(token), ctypes.byref(lp), ctypes.byref(nx)))
        return lp.value, nx.value

    def host_query_batch(self, states, tokens):
        """(logp f32[n], next i32[n]) for the (state, token) pairs."""
        st = np.ascontiguousarray(states, dtype=np.int32)
        tk = np.ascontiguousarray(tokens, dtype=np.int32)
        lp = np.empty(st.shape[0], dtype=np.float32)
        nx = np.empty(st.shape[0], dtype=np.int32)
        _check(lib.flexctc_lm_host_query_batch(self.h, st.shape[0], st.ctypes.data, tk.ctypes.data, lp.ctypes.data,
                                               nx.ctypes.data))
        return lp, nx

    def host_bound(self, state: int):
        """(ub, LM.Final) of a state: the kernels' pre-prune bound ub >= max_w log P(w | state)."""
        ub, eos = ctypes.c_float(), ctypes.c_float()
        _check(lib.flexctc_lm_host_bound(self.h, int(state), ctypes.byref(ub), ctypes.byref(eos)))
        return ub.value, eos.value


class Boost:
    """flexctc_boost handle (flexctc_boost_build)."""

    def __init__(self, phrases, token_weight: float, vocab_size: int, device: int = 0):
        toks = np.ascontiguousarray([t for p in phrases for t in p], dtype=np.int32)
        offs = np.zeros(len(phrases) + 1, dtype=np.int64)
        offs[1:] = np.cumsum([len(p) for p in phrases])
        h = ctypes.c_void_p()
        _check(lib.flexctc_boost_build(toks.ctypes.data_as(ctypes.c_void_p), offs.ctypes.data_as(ctypes.c_void_p),
                                       len(phrases), float(token_weight), int(vocab_size), int(device),
                                       ctypes.byref(h)))
        self.h = h
        self.vocab_size = vocab_size

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:
            lib.flexctc_boost_free(self.h)
            self.h = None

    def num_nodes(self) -> int:
        n = ctypes.c_int32()
        _check(lib.flexctc_boost_num_nodes(self.h, ctypes.byref(n)))
        return n.value

    def host_query(self, node: int, token: int):
        d, nx, u = ctypes.c_float(), ctypes.c_int32(), ctypes.c_float()
        _check(lib.flexctc_boost_host_query(self.h, int(node), int(token), ctypes.byref(d), ctypes.byref(nx),
                                            ctypes.byref(u)))
        return d.value, nx.value, u.value

    def host_query_batch(self, nodes, tokens):
        """(delta f32[n], next i32[n]) for the (node, token) pairs."""
        nd = np.ascontiguousarray(nodes, dtype=np.int32)
        tk = np.ascontiguousarray(tokens, dtype=np.int32)
        d = np.empty(nd.shape[0], dtype=np.float32)
        nx = np.empty(nd.shape[0], dtype=np.int32)
        _check(lib.flexctc_boost_host_query_batch(self.h, nd.shape[0], nd.ctypes.data, tk.ctypes.data, d.ctypes.data,
                                                  nx.ctypes.data))
        return d, nx

    def host_signature(self, node: int) -> int:
        sg = ctypes.c_uint64()
        _check(lib.flexctc_boost_host_signature(self.h, int(node), ctypes.byref(sg)))
        return sg.value


def _check_lengths(lengths, B: int, device=None, host: bool = False):
    """lengths must be int32, contiguous, exactly B entries, on log_probs' device (or on the host
    for decode_host): the C ABI reads int32[B] (an int64 tensor would be misread silently)."""
    import torch
    if not isinstance(lengths, torch.Tensor):
        raise FlexCTCError(1, "lengths must be a torch tensor")
    if lengths.dtype != torch.int32:
        raise FlexCTCError(1, f"lengths must be int32 (got {lengths.dtype})")
    if not lengths.is_contiguous() or lengths.dim() != 1 or lengths.numel() != B:
        raise FlexCTCError(1, f"lengths must be a contiguous 1-D tensor of B = {B} entries")
    if host:
        if lengths.is_cuda:
            raise FlexCTCError(1, "decode_host takes host lengths")
    elif not lengths.is_cuda or (device is not None and lengths.device != device):
        raise FlexCTCError(1, "lengths must be on the same CUDA device as the inputs")


def workspace_bytes(B: int, T: int, Vp1: int, cfg: Config) -> int:
    return int(lib.flexctc_workspace_bytes(int(B), int(T), int(Vp1), ctypes.byref(cfg)))


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


@dataclass
class Workspace:
    buf: object  # torch.uint8 cuda tensor
    nbytes: int


def make_workspace(B: int, T: int, Vp1: int, cfg: Config, device=None):
    import torch
    n = workspace_bytes(B, T, Vp1, cfg)
    return Workspace(torch.empty(max(n, 1), dtype=torch.uint8, device=device or "cuda"), n)


def make_logits_workspace(B: int, T: int, Vp1: int, cfg: Config, device=None):
    """Workspace for decode_logits_bf16 (flexctc_logits_workspace_bytes)."""
    import torch
    n = int(lib.flexctc_logits_workspace_bytes(int(B), int(T), int(Vp1), ctypes.byref(cfg)))
    return Workspace(torch.empty(max(n, 1), dtype=torch.uint8, device=device or "cuda"), n)


def decode(log_probs, lengths, cfg: Config, lm: LM | None = None, boost: Boost | None = None,
           Vp1: int | None = None, workspace: Workspace | None = None, stream=None, outputs=None,
           alignment: bool = False):
    """Enqueue flexctc_decode on `stream` (default: torch's current stream).

    log_probs: CUDA float32 tensor [B, T, >=Vp1] with unit stride on the last axis (the first
    Vp1 columns are used; blank = Vp1-1). lengths: CUDA int32 [B]. Returns a dict of CUDA
    tensors (tokens, num_tokens, scores, timestamps[, alignment]); valid once the stream syncs.
    """
    import torch
    if not (log_probs.is_cuda and lengths.is_cuda):
        raise FlexCTCError(1, "decode needs CUDA tensors (there is no CPU path)")
    if log_probs.dtype != torch.float32 or log_probs.dim() != 3 or log_probs.stride(2) != 1:
        raise FlexCTCError(1, "log_probs must be float32 [B, T, V'] with unit stride on V'")
    B, T, W = log_probs.shape
    _check_lengths(lengths, B, log_probs.device)
    Vp1 = W if Vp1 is None else Vp1
    dev = log_probs.device
    if workspace is None:
        workspace = make_workspace(B, T, Vp1, cfg, dev)
    if outputs is None:
        outputs = {
            "tokens": torch.empty((B, T), dtype=torch.int32, device=dev),
            "num_tokens": torch.empty(B, dtype=torch.int32, device=dev),
            "scores": torch.empty(B, dtype=torch.float32, device=dev),
            "timestamps": torch.empty((B, T), dtype=torch.int32, device=dev),
        }
        if alignment:
            outputs["alignment"] = torch.empty((B, T), dtype=torch.int32, device=dev)
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        _check(lib.flexctc_decode(_ptr(log_probs), log_probs.stride(0), log_probs.stride(1), _ptr(lengths), B, T,
                                  Vp1, ctypes.byref(cfg), lm.h if lm else None, boost.h if boost else None,
                                  _ptr(workspace.buf), workspace.nbytes, ctypes.c_void_p(stream.cuda_stream),
                                  _ptr(outputs["tokens"]), _ptr(outputs["num_tokens"]), _ptr(outputs["scores"]),
                                  _ptr(outputs.get("timestamps")), _ptr(outputs.get("alignment"))))
    return outputs


def decode_nbest(log_probs, lengths, cfg: Config, nbest: int, lm: LM | None = None, boost: Boost | None = None,
                 Vp1: int | None = None, workspace: Workspace | None = None, stream=None):
    """Enqueue flexctc_decode_nbest: the `nbest` best final hypotheses per utterance, ranked by
    (score desc, slot asc). Returns CUDA tensors tokens [B, N, T], num_tokens [B, N], scores [B, N],
    timestamps [B, N, T]; rows past the surviving hypotheses are empty (0 tokens, -inf)."""
    import torch
    if not (log_probs.is_cuda and lengths.is_cuda):
        raise FlexCTCError(1, "decode needs CUDA tensors (there is no CPU path)")
    if log_probs.dtype != torch.float32 or log_probs.dim() != 3 or log_probs.stride(2) != 1:
        raise FlexCTCError(1, "log_probs must be float32 [B, T, V'] with unit stride on V'")
    B, T, W = log_probs.shape
    _check_lengths(lengths, B, log_probs.device)
    Vp1 = W if Vp1 is None else Vp1
    dev = log_probs.device
    if workspace is None:
        workspace = make_workspace(B, T, Vp1, cfg, dev)
    out = {"tokens": torch.empty((B, nbest, T), dtype=torch.int32, device=dev),
           "num_tokens": torch.empty((B, nbest), dtype=torch.int32, device=dev),
           "scores": torch.empty((B, nbest), dtype=torch.float32, device=dev),
           "timestamps": torch.empty((B, nbest, T), dtype=torch.int32, device=dev)}
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        _check(lib.flexctc_decode_nbest(_ptr(log_probs), log_probs.stride(0), log_probs.stride(1), _ptr(lengths), B,
                                        T, Vp1, ctypes.byref(cfg), lm.h if lm else None, boost.h if boost else None,
                                        _ptr(workspace.buf), workspace.nbytes, ctypes.c_void_p(stream.cuda_stream),
                                        int(nbest), _ptr(out["tokens"]), _ptr(out["num_tokens"]), _ptr(out["scores"]),
                                        _ptr(out["timestamps"])))
    return out


def decode_logits_bf16(logits, lengths, cfg: Config, lm: LM | None = None, boost: Boost | None = None,
                       Vp1: int | None = None, workspace: Workspace | None = None, stream=None, outputs=None,
                       alignment: bool = False):
    """Enqueue flexctc_decode_logits_bf16: like decode() but over bf16 logits [B, T, >=Vp1]
    (torch.bfloat16, unit stride on the last axis), normalised on the GPU (reading R25) first."""
    import torch
    if not (logits.is_cuda and lengths.is_cuda):
        raise FlexCTCError(1, "decode needs CUDA tensors (there is no CPU path)")
    if logits.dtype != torch.bfloat16 or logits.dim() != 3 or logits.stride(2) != 1:
        raise FlexCTCError(1, "logits must be bfloat16 [B, T, V'] with unit stride on V'")
    B, T, W = logits.shape
    _check_lengths(lengths, B, logits.device)
    Vp1 = W if Vp1 is None else Vp1
    dev = logits.device
    if workspace is None:
        workspace = make_logits_workspace(B, T, Vp1, cfg, dev)
    if outputs is None:
        outputs = {"tokens": torch.empty((B, T), dtype=torch.int32, device=dev),
                   "num_tokens": torch.empty(B, dtype=torch.int32, device=dev),
                   "scores": torch.empty(B, dtype=torch.float32, device=dev),
                   "timestamps": torch.empty((B, T), dtype=torch.int32, device=dev)}
        if alignment:
            outputs["alignment"] = torch.empty((B, T), dtype=torch.int32, device=dev)
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        _check(lib.flexctc_decode_logits_bf16(_ptr(logits), logits.stride(0), logits.stride(1), _ptr(lengths), B, T,
                                              Vp1, ctypes.byref(cfg), lm.h if lm else None,
                                              boost.h if boost else None, _ptr(workspace.buf), workspace.nbytes,
                                              ctypes.c_void_p(stream.cuda_stream), _ptr(outputs["tokens"]),
                                              _ptr(outputs["num_tokens"]), _ptr(outputs["scores"]),
                                              _ptr(outputs.get("timestamps")), _ptr(outputs.get("alignment"))))
    return outputs


def set_profile_events(start=None, stop=None):
    """Record torch.cuda.Event `start`/`stop` around the beam kernel of later decode calls."""
    lib.flexctc_set_profile_events(ctypes.c_void_p(start.cuda_event) if start is not None else None,
                                   ctypes.c_void_p(stop.cuda_event) if stop is not None else None)


def last_kernel() -> str:
    """Name of the frame-loop kernel the last decode on this thread launched."""
    return lib.flexctc_last_kernel().decode()


def set_stage_events(stage: int, start=None, stop=None):
    """Record torch.cuda.Event `start`/`stop` around a stage of later decode calls: 0 the beam
    kernel, 1 the frame compaction pass (warp path only)."""
    _check(lib.flexctc_set_stage_events(stage, ctypes.c_void_p(start.cuda_event) if start is not None else None,
                                        ctypes.c_void_p(stop.cuda_event) if stop is not None else None))


def stats(workspace: Workspace) -> dict:
    """Device counters of the last decode on `workspace` (after the stream has synchronised)."""
    out = np.zeros(len(STAT_NAMES), dtype=np.uint64)
    _check(lib.flexctc_get_stats(_ptr(workspace.buf), out.ctypes.data_as(ctypes.c_void_p), len(STAT_NAMES)))
    return {k: int(v) for k, v in zip(STAT_NAMES, out)}


def check(workspace: Workspace) -> int:
    """Device flags of the last decode on `workspace` (call after the stream has synchronised)."""
    f = ctypes.c_uint32()
    _check(lib.flexctc_check(_ptr(workspace.buf), ctypes.byref(f)))
    return f.value


def host_scratch_bytes(B: int, T: int, Vp1: int, cfg: Config) -> int:
    return int(lib.flexctc_host_scratch_bytes(int(B), int(T), int(Vp1), ctypes.byref(cfg)))


def host_streaming() -> bool:
    """flexctc_host_streaming: does decode_host overlap its H2D copy with the decode here?"""
    return bool(lib.flexctc_host_streaming())


def decode_host(log_probs: np.ndarray, lengths: np.ndarray, cfg: Config, lm: LM | None = None,
                boost: Boost | None = None, scratch=None, stream=None, out=None):
    """End-to-end flexctc_decode_host: host (ideally pinned) float32 [B, T, V'] in, host outputs
    out; H2D, decode and D2H all run inside the call (which synchronises the stream). The
    device flags of the decode come back in out["flags"]."""
    return _decode_host(log_probs, lengths, cfg, lm, boost, scratch, stream, out, bf16=False)


def decode_host_bf16(logits, lengths, cfg: Config, lm: LM | None = None, boost: Boost | None = None,
                     scratch=None, stream=None, out=None):
    """flexctc_decode_host_bf16: host (ideally pinned) bf16 logits [B, T, V'] (torch.bfloat16, or
    uint16 bit patterns), normalised on the GPU (reading R25); otherwise as decode_host."""
    return _decode_host(logits, lengths, cfg, lm, boost, scratch, stream, out, bf16=True)


def _decode_host(x, lengths, cfg, lm, boost, scratch, stream, out, bf16):
    import torch
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(x)
    if isinstance(lengths, np.ndarray):
        lengths = torch.from_numpy(lengths)
    want = (torch.bfloat16, torch.uint16) if bf16 else (torch.float32,)
    if x.dtype not in want or x.dim() != 3 or not x.is_contiguous() or x.is_cuda:
        raise FlexCTCError(1, f"decode_host{'_bf16' if bf16 else ''} takes a contiguous host {want[0]} [B, T, V'] tensor")
    B, T, Vp1 = x.shape
    _check_lengths(lengths, B, host=True)
    nscratch = (lib.flexctc_host_scratch_bytes_bf16 if bf16 else lib.flexctc_host_scratch_bytes)(
        int(B), int(T), int(Vp1), ctypes.byref(cfg))
    if scratch is None:
        scratch = torch.empty(max(int(nscratch), 1), dtype=torch.uint8, device="cuda")
    if out is None:
        pin = x.is_pinned()
        out = {"tokens": torch.empty((B, T), dtype=torch.int32, pin_memory=pin),
               "num_tokens": torch.empty(B, dtype=torch.int32, pin_memory=pin),
               "scores": torch.empty(B, dtype=torch.float32, pin_memory=pin),
               "timestamps": torch.empty((B, T), dtype=torch.int32, pin_memory=pin)}
    if stream is None:
        stream = torch.cuda.current_stream()
    flags = ctypes.c_uint32()
    fn = lib.flexctc_decode_host_bf16 if bf16 else lib.flexctc_decode_host
    _check(fn(_ptr(x), _ptr(lengths), B, T, Vp1, ctypes.byref(cfg), lm.h if lm else None, boost.h if boost else None,
              _ptr(scratch), scratch.numel(), ctypes.c_void_p(stream.cuda_stream), _ptr(out["tokens"]),
              _ptr(out["num_tokens"]), _ptr(out["scores"]), _ptr(out["timestamps"]), ctypes.byref(flags)))
    out["flags"] = flags.value
    return out
