"""Minimal ARPA reader + textbook backoff recursion in fp64 (independent of the oracle)."""
from __future__ import annotations

import math


class ArpaPy:
    def __init__(self, path):
        self.p, self.bw, self.order = {}, {}, 0
        sec = None
        for line in open(path):
            s = line.strip()
            if not s:
                continue
            if s == "\\data\\":
                sec = "data"
                continue
            if s == "\\end\\":
                break
            if s.startswith("\\") and s.endswith("-grams:"):
                sec = int(s[1:s.index("-")])
                self.order = max(self.order, sec)
                continue
            if sec == "data" or sec is None:
                continue
            f = s.split()
            n = sec
            key = tuple(f[1:1 + n])
            self.p[key] = float(f[0]) * math.log(10.0)
            if len(f) == n + 2:
                self.bw[key] = float(f[n + 1]) * math.log(10.0)

    def logp(self, hist, w):
        """P(w | hist): explicit entry, else bw(hist) + P(w | hist[1:])."""
        h = tuple(hist)[-(self.order - 1):] if self.order > 1 else ()
        return self._rec(h, w)

    def _rec(self, h, w):
        if h + (w,) in self.p:
            return self.p[h + (w,)]
        if not h:
            raise KeyError(w)
        return self.bw.get(h, 0.0) + self._rec(h[1:], w)

    def seq(self, toks):
        """Σ log P(tok_i | <s> tok_<i) + log P(</s> | <s> toks)."""
        hist = ["<s>"]
        s = 0.0
        for t in toks:
            s += self.logp(hist, t)
            hist.append(t)
        return s + self.logp(hist, "</s>")
