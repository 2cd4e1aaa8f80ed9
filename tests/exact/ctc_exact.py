"""Brute force, CTC forward algorithm and greedy decoding in fp64 / fp32 (test pins)."""
from __future__ import annotations

import itertools
import math

import numpy as np


def collapse(align, blank):
    """CTC collapse: merge repeats, drop blanks."""
    out, prev = [], None
    for a in align:
        if a != blank and a != prev:
            out.append(int(a))
        prev = a
    return tuple(out)


def _lse(xs):
    m = max(xs)
    if m == -math.inf:
        return -math.inf
    return m + math.log(sum(math.exp(x - m) for x in xs))


def brute_force(D, blank, mode="lse"):
    """Every transcript's score over all V'^T alignments: lse (= log P_CTC(y|x)) or max."""
    D = np.asarray(D, dtype=np.float64)
    T, Vp1 = D.shape
    groups = {}
    for align in itertools.product(range(Vp1), repeat=T):
        s = float(sum(D[t, a] for t, a in enumerate(align)))
        groups.setdefault(collapse(align, blank), []).append(s)
    return {y: (_lse(v) if mode == "lse" else max(v)) for y, v in groups.items()}


def ctc_forward(D, y, blank):
    """log P(y | x) by the textbook CTC forward (alpha) recursion over l' = (b, y1, b, ..., b)."""
    D = np.asarray(D, dtype=np.float64)
    T = D.shape[0]
    ext = [blank]
    for c in y:
        ext += [c, blank]
    S = len(ext)
    if T == 0:
        return 0.0 if len(y) == 0 else -math.inf
    NEG = -math.inf
    a = [NEG] * S
    a[0] = D[0, ext[0]]
    if S > 1:
        a[1] = D[0, ext[1]]
    for t in range(1, T):
        b = [NEG] * S
        for s in range(S):
            terms = [a[s]]
            if s >= 1:
                terms.append(a[s - 1])
            if s >= 2 and ext[s] != blank and ext[s] != ext[s - 2]:
                terms.append(a[s - 2])
            b[s] = _lse(terms) + D[t, ext[s]]
        a = b
    return _lse([a[S - 1]] + ([a[S - 2]] if S >= 2 else []))


def greedy(D32, blank):
    """Greedy CTC: per-frame argmax (lowest index wins ties), collapse; score = fp32 running
    sum of the chosen log-probs."""
    D32 = np.asarray(D32, dtype=np.float32)
    align = [int(np.argmax(row)) for row in D32]
    s = np.float32(0.0)
    for t, a in enumerate(align):
        s = np.float32(s + D32[t, a])
    return collapse(align, blank), float(s), align
