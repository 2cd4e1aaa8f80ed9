"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle's tests.

This module holds NONE of the decoding method's arithmetic (no candidate scoring,
no top-K, no LM/boost queries). It only manufactures inputs with the shapes and
statistics of the paper's workloads:

* ``logprobs``  — Parakeet-CTC-like log-softmax tensors D [B, T, V+1] (blank = V),
                  40 ms frames, peaky spikes, competitors, leakage (PAPER.md P:157-159,
                  §III-C "output log probabilities is tensor D").
* ``arpa_text`` — a 4-gram backoff ARPA LM (~1M n-grams) estimated with interpolated
                  absolute discounting from a corpus drawn from a sparse Markov source
                  (stands in for the paper's KenLM subword LMs).
* ``phrases``   — 1000 boosted phrases of 2-5 tokens (stands in for "~1,000 medical
                  terms").
* ``lengths``   — fixed T=400 (c2-c4) or LibriSpeech-shaped lognormal durations (c5).

Everything is a pure function of its seed.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

FRAME_SECONDS = 0.04  # BASELINE.json north_star: "40 ms frames"

# --------------------------------------------------------------------------------------
# Workload configurations (BASELINE.json configs[0..4])
# --------------------------------------------------------------------------------------


@dataclass(frozen=True)
class Workload:
    name: str
    B: int
    T: int                 # padded frame count (max length)
    V: int                 # non-blank vocabulary; V' = V + 1, blank id = V
    beam: int
    lm: bool
    boost: bool
    seed: int
    lengths: str = "fixed"  # "fixed" | "librispeech"
    alpha_lm: float = 0.5
    alpha_bt: float = 1.0
    beta: float = 0.5
    theta: float = 12.0     # P:237 "we set the pruning threshold θ to 12"
    merge_mode: int = 0     # 0 = log-sum-exp, 1 = max

    @property
    def Vp1(self) -> int:
        return self.V + 1


WORKLOADS = {
    "c1": Workload("c1", B=1, T=50, V=128, beam=4, lm=False, boost=False, seed=101, beta=0.0),
    "c2": Workload("c2", B=32, T=400, V=1024, beam=8, lm=False, boost=False, seed=102, beta=0.0),
    "c3": Workload("c3", B=64, T=400, V=1024, beam=16, lm=True, boost=False, seed=103),
    "c4": Workload("c4", B=64, T=400, V=1024, beam=16, lm=True, boost=True, seed=104),
    "c5": Workload("c5", B=512, T=875, V=1024, beam=128, lm=True, boost=True, seed=105,
                   lengths="librispeech"),
}

LM_SEED = 7
PHRASE_SEED = 11

# --------------------------------------------------------------------------------------
# Sparse Markov token source (corpus for the LM and transcripts for the log-probs)
# --------------------------------------------------------------------------------------

_P = np.uint64(0x9E3779B97F4A7C15)


def _mix(*xs: np.ndarray) -> np.ndarray:
    """Deterministic integer hash (splitmix-style) of integer arrays, vectorised."""
    h = np.zeros(np.broadcast(*xs).shape, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for x in xs:
            h = h ^ (np.asarray(x).astype(np.uint64) + _P + (h << np.uint64(6)) + (h >> np.uint64(2)))
            h = h ^ (h >> np.uint64(30))
            h = h * np.uint64(0xBF58476D1CE4E5B9)
            h = h ^ (h >> np.uint64(27))
            h = h * np.uint64(0x94D049BB133111EB)
            h = h ^ (h >> np.uint64(31))
    return h


class MarkovSource:
    """Random sparse order-3 (two-token context) Markov source over V tokens.

    next(a, b) = with prob p2: one of n2 successors hashed from (a, b)
                 with prob p1: one of n1 successors hashed from (b)
                 else        : a Zipf(s) unigram draw.
    """

    def __init__(self, V: int, seed: int, n2: int = 3, n1: int = 8, p2: float = 0.45,
                 p1: float = 0.30, zipf_s: float = 1.1):
        self.V, self.seed, self.n2, self.n1, self.p2, self.p1 = V, seed, n2, n1, p2, p1
        rng = np.random.default_rng(seed)
        ranks = np.arange(1, V + 1, dtype=np.float64)
        w = ranks ** (-zipf_s)
        perm = rng.permutation(V)           # which token gets which Zipf rank
        p = np.empty(V)
        p[perm] = w / w.sum()
        self.unigram = p
        self.cdf = np.cumsum(p)
        self.cdf[-1] = 1.0

    def zipf(self, rng: np.random.Generator, n) -> np.ndarray:
        return np.searchsorted(self.cdf, rng.random(n), side="right").astype(np.int64).clip(0, self.V - 1)

    def step(self, rng: np.random.Generator, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        n = a.shape[0]
        u = rng.random(n)
        i2 = rng.integers(0, self.n2, n)
        i1 = rng.integers(0, self.n1, n)
        s2 = (_mix(a, b, i2, np.uint64(self.seed)) % np.uint64(self.V)).astype(np.int64)
        s1 = (_mix(b, i1, np.uint64(self.seed + 1)) % np.uint64(self.V)).astype(np.int64)
        z = self.zipf(rng, n)
        return np.where(u < self.p2, s2, np.where(u < self.p2 + self.p1, s1, z))

    def sequences(self, rng: np.random.Generator, n: int, length: int) -> np.ndarray:
        """n sequences of exactly `length` tokens, each started from a fresh Zipf pair."""
        out = np.empty((n, max(length, 0)), dtype=np.int64)
        if length == 0:
            return out
        a = self.zipf(rng, n)
        b = self.zipf(rng, n)
        for j in range(length):
            c = self.step(rng, a, b)
            out[:, j] = c
            a, b = b, c
        return out


# --------------------------------------------------------------------------------------
# 4-gram ARPA estimation: interpolated absolute discounting -> backoff ARPA
# --------------------------------------------------------------------------------------

_BASE = 2048  # token code width for packing n-grams into int64 keys


def _pack(cols) -> np.ndarray:
    k = np.zeros(cols[0].shape, dtype=np.int64)
    for c in cols:
        k = k * _BASE + c.astype(np.int64)
    return k


def _unpack(keys: np.ndarray, n: int) -> list:
    cols = []
    k = keys.copy()
    for _ in range(n):
        cols.append(k % _BASE)
        k //= _BASE
    return cols[::-1]


@dataclass
class _Order:
    keys: np.ndarray          # packed n-grams, sorted
    lnp: np.ndarray           # natural-log probability of the listed n-gram
    bw: np.ndarray = field(default=None)  # natural-log backoff of the n-gram as a context (0 if none)


def _lookup(keys: np.ndarray, q: np.ndarray):
    idx = np.searchsorted(keys, q)
    idx_c = np.minimum(idx, len(keys) - 1)
    found = (idx < len(keys)) & (keys[idx_c] == q)
    return found, idx_c


def _prob(orders: list, m: int, ctx: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Natural-log backoff probability P_m(w | ctx) with |ctx| = m-1 (vectorised)."""
    if m == 1:
        found, idx = _lookup(orders[0].keys, w)
        assert found.all()
        return orders[0].lnp[idx]
    o = orders[m - 1]
    found, idx = _lookup(o.keys, ctx * _BASE + w)
    out = np.empty(len(w))
    out[found] = o.lnp[idx[found]]
    nf = ~found
    if nf.any():
        c = ctx[nf]
        cf, cidx = _lookup(orders[m - 2].keys, c)
        bw = np.where(cf, orders[m - 2].bw[cidx], 0.0)
        shorter = c % (_BASE ** (m - 2)) if m > 2 else np.zeros_like(c)
        out[nf] = bw + _prob(orders, m - 1, shorter, w[nf])
    return out


def arpa_text(V: int = 1024, seed: int = LM_SEED, order: int = 4, n_tokens: int = 3_000_000,
              mean_sentence: int = 24, discount: float = 0.75, prune_min_count: int = 2) -> str:
    """Synthetic backoff ARPA (log10), symbols "0".."V-1", "<s>", "</s>".

    Interpolated absolute discounting: p(w|h) = max(c(h,w)-D,0)/c(h.) + D*N1+(h.)/c(h.) * P(w|h')
    for listed n-grams; singleton n-grams of order >= 3 are pruned; backoff weights are
    normalised so that sum_w P(w|h) = 1 for every context.
    """
    rng = np.random.default_rng(seed)
    src = MarkovSource(V, seed)
    BOS, EOS = V, V + 1
    n_sent = max(1, n_tokens // mean_sentence)
    lens = np.clip(rng.geometric(1.0 / mean_sentence, n_sent), 2, 4 * mean_sentence)
    Lmax = int(lens.max())
    seqs = src.sequences(rng, n_sent, Lmax)
    # padded sentence matrix: <s> tokens... </s> then -1
    W = np.full((n_sent, Lmax + 2), -1, dtype=np.int64)
    W[:, 0] = BOS
    pos = np.arange(Lmax)[None, :]
    W[:, 1:Lmax + 1] = np.where(pos < lens[:, None], seqs, -1)
    W[np.arange(n_sent), lens + 1] = EOS

    orders: list = []
    # ---- unigrams: add-one over V tokens + </s>; <s> listed with log10 -99
    toks = W[:, 1:].ravel()
    toks = toks[toks >= 0]
    cnt = np.bincount(toks, minlength=V + 2).astype(np.float64)
    syms = np.arange(V + 2)
    uni = np.where(syms == BOS, -99.0 * math.log(10.0), np.log((cnt + 1.0) / (cnt[syms != BOS].sum() + (V + 1))))
    orders.append(_Order(keys=syms.astype(np.int64), lnp=uni))

    for n in range(2, order + 1):
        # all n-gram windows
        cols = [W[:, i:W.shape[1] - n + 1 + i] for i in range(n)]
        valid = np.ones(cols[0].shape, dtype=bool)
        for c in cols:
            valid &= c >= 0
        grams = _pack([c[valid] for c in cols])
        keys, counts = np.unique(grams, return_counts=True)
        ctx = keys // _BASE
        w = keys % _BASE
        # per-context totals and distinct-successor counts (unpruned)
        uctx, inv = np.unique(ctx, return_inverse=True)
        c_h = np.bincount(inv, weights=counts).astype(np.float64)
        n1_h = np.bincount(inv).astype(np.float64)
        lower_ctx = ctx % (_BASE ** (n - 2)) if n > 2 else np.zeros_like(ctx)
        p_lower = np.exp(_prob(orders, n - 1, lower_ctx, w))
        p = np.maximum(counts - discount, 0.0) / c_h[inv] + discount * n1_h[inv] / c_h[inv] * p_lower
        keep = counts >= prune_min_count if n >= 3 else np.ones(len(keys), dtype=bool)
        keys, p, p_lower, ctx = keys[keep], p[keep], p_lower[keep], ctx[keep]
        # backoff weights for the (n-1)-gram contexts that have listed children
        prev = orders[n - 2]
        bw = np.zeros(len(prev.keys))
        uctx, inv = np.unique(ctx, return_inverse=True)
        num = 1.0 - np.bincount(inv, weights=p)
        den = 1.0 - np.bincount(inv, weights=p_lower)
        found, cidx = _lookup(prev.keys, uctx)
        assert found.all(), "listed n-gram whose context is not listed"
        bw[cidx] = np.log(np.maximum(num, 1e-12)) - np.log(np.maximum(den, 1e-12))
        prev.bw = bw
        orders.append(_Order(keys=keys, lnp=np.log(p)))
    orders[-1].bw = np.zeros(len(orders[-1].keys))

    # ---- write ARPA text (log10)
    names = [str(i) for i in range(V)] + ["<s>", "</s>"]
    L10 = 1.0 / math.log(10.0)
    out = ["", "\\data\\"]
    for n, o in enumerate(orders, 1):
        out.append(f"ngram {n}={len(o.keys)}")
    for n, o in enumerate(orders, 1):
        out.append("")
        out.append(f"\\{n}-grams:")
        cols = _unpack(o.keys, n)
        words = [" ".join(names[int(t)] for t in row) for row in zip(*[c.tolist() for c in cols])]
        lp = o.lnp * L10
        bw = o.bw * L10
        has_bw = (o.bw != 0.0) & (n < order)
        for i, ws in enumerate(words):
            if has_bw[i]:
                out.append(f"{lp[i]:.6f}\t{ws}\t{bw[i]:.6f}")
            else:
                out.append(f"{lp[i]:.6f}\t{ws}")
    out.append("")
    out.append("\\end\\")
    out.append("")
    return "\n".join(out)


def arpa_file(path: str | None = None, V: int = 1024, seed: int = LM_SEED, **kw) -> str:
    """Write the synthetic ARPA to `path` (default: a cache file under the repo) and return it."""
    if path is None:
        cache = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), ".cache")
        os.makedirs(cache, exist_ok=True)
        tag = "_".join(f"{k}{v}" for k, v in sorted(kw.items()))
        path = os.path.join(cache, f"lm_V{V}_s{seed}{('_' + tag) if tag else ''}.arpa")
        if os.path.exists(path):
            return path
    text = arpa_text(V=V, seed=seed, **kw)
    tmp = path + f".tmp{os.getpid()}"
    with open(tmp, "w") as f:
        f.write(text)
    os.replace(tmp, path)
    return path


# --------------------------------------------------------------------------------------
# Boosted phrases
# --------------------------------------------------------------------------------------


def phrases(V: int = 1024, n: int = 1000, seed: int = PHRASE_SEED) -> list:
    """n distinct phrases of 2-5 tokens (30/35/25/10 %); half Markov-corpus subsequences,
    half random 'rare terms'."""
    rng = np.random.default_rng(seed)
    src = MarkovSource(V, LM_SEED)
    out, seen = [], set()
    while len(out) < n:
        L = int(rng.choice([2, 3, 4, 5], p=[0.30, 0.35, 0.25, 0.10]))
        if len(out) % 2 == 0:
            ph = tuple(int(x) for x in src.sequences(rng, 1, L)[0])
        else:
            ph = tuple(int(x) for x in rng.integers(0, V, L))
        if ph not in seen:
            seen.add(ph)
            out.append(ph)
    return out


def phrases_csr(ph: list):
    toks = np.array([t for p in ph for t in p], dtype=np.int32)
    offs = np.zeros(len(ph) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([len(p) for p in ph])
    return toks, offs


# --------------------------------------------------------------------------------------
# Lengths and log-probs
# --------------------------------------------------------------------------------------


def lengths(wl: Workload, B: int | None = None, seed: int | None = None) -> np.ndarray:
    B = wl.B if B is None else B
    rng = np.random.default_rng((wl.seed if seed is None else seed) + 1000)
    if wl.lengths == "fixed":
        return np.full(B, wl.T, dtype=np.int32)
    # LibriSpeech test-clean shaped: lognormal, mean 7.42 s, sigma_log 0.65, clipped [1.3, 35] s
    sigma = 0.65
    mu = math.log(7.42) - sigma * sigma / 2
    dur = np.clip(rng.lognormal(mu, sigma, B), 1.3, 35.0)
    L = np.round(dur / FRAME_SECONDS).astype(np.int32)
    return np.minimum(L, wl.T)


def logprobs(B: int, T: int, V: int, L: np.ndarray, seed: int, phrase_list: list | None = None,
             token_rate: float = 0.16, pad_value: float = 0.0, row_stride: int | None = None,
             flat: bool = False, markov_seed: int = LM_SEED, return_frames: bool = False):
    """Parakeet-CTC-like log-softmax output, blank = V (last index).

    Returns (D float32 [B, T, stride] with the first V+1 columns valid, transcripts list), plus,
    with return_frames, the planted spike frame of every transcript token (the first frame of
    its span; the RNG stream is the same either way).
    Recipe: logits N(0,1); target (blank on non-spike frames) + U(14,20)
    (U(4,8) for the 'flat' stress variant); on spike frames, p=0.25 a competitor + U(10,16)
    (half random token, half a boosted-phrase continuation); p=0.3 the spike leaks + U(8,14)
    into the next frame; 20% of spikes span 2 frames; D = log_softmax in float64 -> float32.
    """
    Vp1 = V + 1
    stride = Vp1 if row_stride is None else row_stride
    assert stride >= Vp1
    rng = np.random.default_rng(seed)
    src = MarkovSource(V, markov_seed) if V >= 16 else None
    D = np.full((B, T, stride), pad_value, dtype=np.float32)
    transcripts = []
    spike_frames = []
    tlo, thi = (4.0, 8.0) if flat else (14.0, 20.0)
    for b in range(B):
        Lb = int(L[b])
        n_tok = int(round(token_rate * Lb))
        n_tok = min(n_tok, max(0, (Lb + 1) // 2 - 1))
        if src is not None and n_tok > 0:
            y = src.sequences(rng, 1, n_tok)[0].copy()
        else:
            y = rng.integers(0, V, n_tok)
        if phrase_list and n_tok >= 6:
            n_inj = rng.poisson(1.5)
            for _ in range(n_inj):
                ph = phrase_list[int(rng.integers(len(phrase_list)))]
                if len(ph) < n_tok:
                    at = int(rng.integers(0, n_tok - len(ph) + 1))
                    y[at:at + len(ph)] = ph
        transcripts.append([int(t) for t in y])
        logits = rng.standard_normal((Lb, Vp1)).astype(np.float64)
        target = np.full(Lb, V, dtype=np.int64)
        if n_tok > 0:
            q = np.sort(rng.integers(0, Lb - 2 * n_tok + 1, n_tok))
            pos = q + 2 * np.arange(n_tok)
            target[pos] = y
            spike_frames.append([int(x) for x in pos])
        else:
            spike_frames.append([])
        if n_tok > 0:
            for i in range(n_tok):
                nxt = pos[i + 1] if i + 1 < n_tok else Lb
                same_next = i + 1 < n_tok and y[i + 1] == y[i]
                if rng.random() < 0.2 and pos[i] + 1 < nxt and not (same_next and pos[i] + 2 >= nxt):
                    target[pos[i] + 1] = y[i]
        logits[np.arange(Lb), target] += rng.uniform(tlo, thi, Lb)
        spike = target != V
        for t in np.nonzero(spike)[0]:
            if rng.random() < 0.25:
                if phrase_list and rng.random() < 0.5:
                    ph = phrase_list[int(rng.integers(len(phrase_list)))]
                    c = ph[int(rng.integers(len(ph)))]
                else:
                    c = int(rng.integers(0, V))
                logits[t, c] += rng.uniform(10.0, 16.0)
            if t + 1 < Lb and rng.random() < 0.3:
                logits[t + 1, target[t]] += rng.uniform(8.0, 14.0)
        m = logits.max(axis=1, keepdims=True)
        lse = m + np.log(np.exp(logits - m).sum(axis=1, keepdims=True))
        D[b, :Lb, :Vp1] = (logits - lse).astype(np.float32)
    if return_frames:
        return D, transcripts, spike_frames
    return D, transcripts


def random_logprobs(rng: np.random.Generator, B: int, T: int, Vp1: int, peak: float = 0.0):
    """Small dense random log-softmax inputs for exactness tests (float64)."""
    x = rng.standard_normal((B, T, Vp1)) * 1.5
    if peak:
        idx = rng.integers(0, Vp1, (B, T))
        np.put_along_axis(x, idx[..., None], np.take_along_axis(x, idx[..., None], -1) + peak, -1)
    m = x.max(-1, keepdims=True)
    return x - (m + np.log(np.exp(x - m).sum(-1, keepdims=True)))


def workload_inputs(name: str, B: int | None = None, seed_offset: int = 0, row_stride: int | None = None,
                    pad_value: float = 0.0):
    """Everything a run of workload `name` needs: (wl, D, L, arpa_path|None, phrases|None)."""
    wl = WORKLOADS[name]
    B = wl.B if B is None else B
    L = lengths(wl, B, wl.seed + seed_offset)
    T = int(L.max()) if wl.lengths != "fixed" else wl.T
    ph = phrases(wl.V) if wl.boost else None
    D, _ = logprobs(B, T, wl.V, L, wl.seed + seed_offset, phrase_list=ph, row_stride=row_stride,
                    pad_value=pad_value)
    arpa = arpa_file(V=wl.V) if wl.lm else None
    return wl, D, L, arpa, ph
