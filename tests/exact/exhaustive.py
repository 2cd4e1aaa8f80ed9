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
