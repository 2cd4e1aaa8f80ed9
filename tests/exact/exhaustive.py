"""Exhaustive ground truth for Eq. (1): every transcript y gets
  combine_{alignments of y}(Σ_t D[t, a_t]) + α_LM·log P_LM(y, incl. EOS) + α_BT·Σ bt-deltas(y) + β·|y|
(SPEC S:432-440). Only for tiny T, V'."""
from __future__ import annotations

from .ctc_exact import brute_force


def exhaustive(D, blank, mode="lse", alpha_lm=0.0, lm=None, symbols=None, alpha_bt=0.0, boost=None,
               beta=0.0, retract=False):
    ac = brute_force(D, blank, mode)
    out = {}
    for y, s in ac.items():
        tot = s + beta * len(y)
        if lm is not None:
            tot += alpha_lm * lm.seq([symbols[t] for t in y])
        if boost is not None:
            bsum, u = boost.total(y)
            tot += alpha_bt * bsum
            if retract:
                tot -= alpha_bt * boost.U[u]
        out[y] = tot
    return out


def exhaustive_paths(D, blank, mode="lse", alpha_lm=0.0, lm=None, symbols=None, alpha_bt=0.0, boost=None,
                     beta=0.0, retract=False, fuse_repeats=False):
    """Path-level ground truth (V'^T alignments, fp64): each alignment a scores
    Σ_t D[t, a_t] + Σ_emissions (β + α_LM·log P(w | <s> y) + α_BT·delta) and, with fuse_repeats
    (PAPER.md P:167 variant), + α_LM·log P(w | <s> y) + α_BT·delta on every repeat frame (the
    prefix y already ends with w; the states do not advance). Transcript score = combine over
    its alignments + α_LM·log P(</s> | <s> y) (- α_BT·U at EOS with retract)."""
    import itertools
    import math
    T, Vp1 = len(D), len(D[0])
    groups = {}
    for a in itertools.product(range(Vp1), repeat=T):
        s, y, prev, u, hist = 0.0, [], blank, 0, ["<s>"]
        for t, w in enumerate(a):
            s += D[t][w]
            if w != blank and w != prev:
                s += beta
                if lm is not None:
                    s += alpha_lm * lm.logp(hist, symbols[w])
                if boost is not None:
                    d, u = boost.delta(u, w)
                    s += alpha_bt * d
                y.append(w)
                hist.append(symbols[w] if symbols else w)
            elif w != blank and fuse_repeats:
                if lm is not None:
                    s += alpha_lm * lm.logp(hist, symbols[w])
                if boost is not None:
                    s += alpha_bt * boost.delta(u, w)[0]
            prev = w
        key = tuple(y)
        end = 0.0
        if lm is not None:
            end += alpha_lm * lm.logp(hist, "</s>")
        if boost is not None and retract:
            end -= alpha_bt * boost.U[u]
        groups.setdefault(key, ([], end))[0].append(s)
    out = {}
    for y, (ss, end) in groups.items():
        m = max(ss)
        c = m if mode == "max" else m + math.log(sum(math.exp(x - m) for x in ss))
        out[y] = c + end
    return out
