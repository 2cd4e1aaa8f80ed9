"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``liboracle.so`` (oracle.cpp): the plain CPU implementation of FlexCTC's
Algorithm 1 (§III-C) with a direct ARPA backoff evaluator and a naive
suffix-matching phrase booster. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. It shares no code with the
CUDA product (``paper_2508_07315_b200``) and never imports it.

Parity status per function (details in DESIGN.md "Oracle pins"):
  decode (acoustic part + merging, lse and max) ...... pinned: brute force, CTC forward, ctc_loss
  decode with LM/BT/β ................................ pinned: exhaustive enumerator (tests/exact)
  decode K=1 .......................................... pinned: greedy decoding
  lm_logp / lm_seq .................................... pinned: hand-computed ARPA fixtures
  boost_delta / boost_U ............................... pinned: SPEC S:259-285 hand values, telescoping
  log_softmax_bf16 (input side, reading R25) .......... pinned: numpy fp64 log-softmax, hand cases,
        normalisation
  decode at K < #prefixes, θ < ∞ (the beam heuristic) . follows Alg. 1 step by step; the
        truncation itself has no closed form ("parity unpinned" beyond the pins above)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain -O2 (no fast-math, no FMA contraction)."""
    if not force and os.path.exists(_LIB_PATH) and os.path.getmtime(_LIB_PATH) >= max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           "-pthread", _SRC, "-o", tmp]
    subprocess.check_call(cmd)
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class Cfg(ctypes.Structure):
    _fields_ = [("beam", ctypes.c_int32), ("alpha_lm", ctypes.c_double), ("alpha_bt", ctypes.c_double),
                ("beta", ctypes.c_double), ("theta", ctypes.c_double), ("merge_mode", ctypes.c_int32),
                ("retract_boost_at_eos", ctypes.c_int32), ("fuse_repeats", ctypes.c_int32),
                ("merge_first", ctypes.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        P = ctypes.POINTER
        L.oracle_last_error.restype = ctypes.c_char_p
        L.oracle_lm_load.restype = vp
        L.oracle_lm_load.argtypes = [ctypes.c_char_p, i32, vp]
        L.oracle_lm_free.argtypes = [vp]
        L.oracle_lm_order.argtypes = [vp]
        L.oracle_lm_logp.restype = dbl
        L.oracle_lm_logp.argtypes = [vp, vp, i32, i32, i32]
        L.oracle_lm_logp_many.restype = None
        L.oracle_lm_logp_many.argtypes = [vp, vp, i32, vp, i32, i32, vp]
        L.oracle_lm_seq.restype = dbl
        L.oracle_lm_seq.argtypes = [vp, vp, i32]
        L.oracle_boost_build.restype = vp
        L.oracle_boost_build.argtypes = [vp, vp, i32, dbl, i32]
        L.oracle_boost_free.argtypes = [vp]
        L.oracle_boost_delta.restype = dbl
        L.oracle_boost_delta.argtypes = [vp, vp, i32, i32, i32]
        L.oracle_boost_U.restype = dbl
        L.oracle_boost_U.argtypes = [vp, vp, i32, i32]
        L.oracle_boost_state_depth.restype = i32
        L.oracle_boost_state_depth.argtypes = [vp, vp, i32]
        L.oracle_decode_f32.restype = i32
        L.oracle_decode_f32.argtypes = [vp, i64, i64, vp, i32, i32, i32, P(Cfg), vp, vp, i32,
                                        vp, vp, vp, vp, vp]
        L.oracle_decode_nbest.restype = i32
        L.oracle_decode_nbest.argtypes = [vp, i32, i32, i32, P(Cfg), vp, vp, i32, i32, vp, vp, vp]
        L.oracle_log_softmax_bf16.restype = i32
        L.oracle_log_softmax_bf16.argtypes = [vp, i64, i64, i32, vp]
    return _lib


def _err() -> str:
    return lib().oracle_last_error().decode()


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


class LM:
    """Direct ARPA backoff evaluator (R7)."""

    def __init__(self, arpa_path: str, vocab_size: int, symbols=None):
        syms = None
        if symbols is not None:
            arr = (ctypes.c_char_p * vocab_size)(*[s.encode() for s in symbols])
            syms = ctypes.cast(arr, ctypes.c_void_p)
            self._syms = arr
        self.h = lib().oracle_lm_load(arpa_path.encode(), vocab_size, syms)
        if not self.h:
            raise ValueError(_err())
        self.V = vocab_size

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_lm_free(self.h)
            self.h = None

    @property
    def order(self) -> int:
        return lib().oracle_lm_order(self.h)

    def logp_many(self, hist, ws, f32: bool = False):
        """log P(w | hist) for every w in ws (float64 array; f32: the fp32 evaluation)."""
        h = np.ascontiguousarray(hist, dtype=np.int32)
        w = np.ascontiguousarray(ws, dtype=np.int32)
        out = np.empty(w.shape[0], dtype=np.float64)
        lib().oracle_lm_logp_many(self.h, _ptr(h), len(h), w.ctypes.data, w.shape[0], int(f32), out.ctypes.data)
        return out

    def logp(self, hist, w: int, f32: bool = False) -> float:
        """log P(w | <s> hist) in nats; w = -1 means </s>."""
        h = _i32(hist)
        return lib().oracle_lm_logp(self.h, _ptr(h), len(h), int(w), int(f32))

    def seq(self, toks) -> float:
        t = _i32(toks)
        return lib().oracle_lm_seq(self.h, _ptr(t), len(t))


class Boost:
    """Naive suffix-matching phrase booster (R17)."""

    def __init__(self, phrases, token_weight: float, vocab_size: int):
        toks = _i32([t for p in phrases for t in p])
        offs = np.zeros(len(phrases) + 1, dtype=np.int64)
        offs[1:] = np.cumsum([len(p) for p in phrases])
        self.h = lib().oracle_boost_build(_ptr(toks), _ptr(offs), len(phrases), float(token_weight), vocab_size)
        if not self.h:
            raise ValueError(_err())

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_boost_free(self.h)
            self.h = None

    def delta(self, prefix, w: int, f32: bool = False) -> float:
        p = _i32(prefix)
        return lib().oracle_boost_delta(self.h, _ptr(p), len(p), int(w), int(f32))

    def U(self, prefix, f32: bool = False) -> float:
        p = _i32(prefix)
        return lib().oracle_boost_U(self.h, _ptr(p), len(p), int(f32))

    def state_depth(self, prefix) -> int:
        p = _i32(prefix)
        return lib().oracle_boost_state_depth(self.h, _ptr(p), len(p))


def make_cfg(beam, alpha_lm=0.0, alpha_bt=0.0, beta=0.0, theta=float("inf"), merge_mode=0, retract=0,
             fuse_repeats=0, merge_first=0) -> Cfg:
    return Cfg(int(beam), float(alpha_lm), float(alpha_bt), float(beta), float(theta), int(merge_mode), int(retract),
               int(fuse_repeats), int(merge_first))


def decode(D: np.ndarray, lengths, cfg: Cfg, lm: LM | None = None, boost: Boost | None = None,
           nthreads: int | None = None, with_alignment: bool = False):
    """fp32 Algorithm 1 over a batch; D is float32 [B, T, >=Vp1] (last axis contiguous)
    with Vp1 given by cfg-independent D.shape unless `Vp1` columns are sliced by the caller."""
    assert D.dtype == np.float32 and D.ndim == 3 and D.strides[2] == 4
    B, T, _ = D.shape
    return decode_strided(D, D.shape[2], lengths, cfg, lm, boost, nthreads, with_alignment)


def decode_strided(D: np.ndarray, Vp1: int, lengths, cfg: Cfg, lm=None, boost=None, nthreads=None,
                   with_alignment=False):
    B, T = D.shape[0], D.shape[1]
    L = _i32(lengths)
    tok = np.empty((B, T), np.int32)
    n = np.empty(B, np.int32)
    sc = np.empty(B, np.float32)
    ts = np.empty((B, T), np.int32)
    al = np.empty((B, T), np.int32) if with_alignment else None
    nthreads = nthreads or os.cpu_count() or 1
    rc = lib().oracle_decode_f32(_ptr(D), D.strides[0] // 4, D.strides[1] // 4, _ptr(L), B, T, Vp1,
                                 ctypes.byref(cfg), lm.h if lm else None, boost.h if boost else None,
                                 int(nthreads), _ptr(tok), _ptr(n), _ptr(sc), _ptr(ts), _ptr(al))
    if rc != 0:
        raise ValueError(_err())
    out = {"tokens": tok, "num_tokens": n, "scores": sc, "timestamps": ts}
    if with_alignment:
        out["alignment"] = al
    return out


def decode_nbest(D: np.ndarray, cfg: Cfg, lm: LM | None = None, boost: Boost | None = None,
                 L: int | None = None, f32: bool = False, max_out: int = 100000):
    """One utterance D [T, Vp1] (float64). Returns [(tokens tuple, score)] for every final
    merged hypothesis, sorted by (score desc, slot asc)."""
    D = np.ascontiguousarray(D, dtype=np.float64)
    T, Vp1 = D.shape
    L = T if L is None else L
    cap = min(max_out, cfg.beam)
    tok = np.empty((cap, max(T, 1)), np.int32)
    lens = np.empty(cap, np.int32)
    sc = np.empty(cap, np.float64)
    n = lib().oracle_decode_nbest(_ptr(D), T, Vp1, L, ctypes.byref(cfg), lm.h if lm else None,
                                  boost.h if boost else None, int(f32), cap, _ptr(tok), _ptr(lens), _ptr(sc))
    if n < 0:
        raise ValueError(_err())
    return [(tuple(int(x) for x in tok[i, :lens[i]]), float(sc[i])) for i in range(min(n, cap))]


def log_softmax_bf16(x_bits: np.ndarray) -> np.ndarray:
    """Log-softmax over the last axis of bf16 logits given as uint16 bit patterns [..., Vp1]
    (reading R25): fp32 result of (x - lse) with lse = m + log(sum exp(x - m)) in fp64."""
    x = np.ascontiguousarray(x_bits, dtype=np.uint16)
    Vp1 = x.shape[-1]
    rows = x.reshape(-1, Vp1)
    out = np.empty(rows.shape, np.float32)
    rc = lib().oracle_log_softmax_bf16(_ptr(rows), rows.shape[0], Vp1, Vp1, _ptr(out))
    if rc != 0:
        raise ValueError(_err())
    return out.reshape(x.shape)
