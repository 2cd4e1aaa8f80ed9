"""Aho-Corasick booster in fp64 (independent of the oracle's naive suffix matcher).

Reward law: C(n) = w*depth(n); committed(n) = C(deepest final
ancestor-or-self); U = C - committed; pcom = C(deepest final strict ancestor);
delta(u, a) = [v final](C(v) - pcom(v)) + U(v) - U(u), v = AC transition.
"""
from __future__ import annotations

from collections import deque


class BoostPy:
    def __init__(self, phrases, w):
        self.goto = [{}]
        self.depth = [0]
        self.final = [False]
        self.parent = [0]
        for ph in phrases:
            n = 0
            for a in ph:
                if a not in self.goto[n]:
                    self.goto.append({})
                    self.depth.append(self.depth[n] + 1)
                    self.final.append(False)
                    self.parent.append(n)
                    self.goto[n][a] = len(self.goto) - 1
                n = self.goto[n][a]
            self.final[n] = True
        N = len(self.goto)
        self.fail = [0] * N
        q = deque(self.goto[0].values())
        while q:
            u = q.popleft()
            for a, v in self.goto[u].items():
                f = self.fail[u]
                while f and a not in self.goto[f]:
                    f = self.fail[f]
                self.fail[v] = self.goto[f][a] if (a in self.goto[f] and self.goto[f][a] != v) else 0
                q.append(v)
        self.C = [w * d for d in self.depth]
        self.committed = [0.0] * N
        self.pcom = [0.0] * N
        order = sorted(range(N), key=lambda n: self.depth[n])
        for n in order:
            if n == 0:
                continue
            p = self.parent[n]
            self.pcom[n] = self.committed[p]
            self.committed[n] = self.C[n] if self.final[n] else self.committed[p]
        self.U = [self.C[n] - self.committed[n] for n in range(N)]

    def step(self, u, a):
        while u and a not in self.goto[u]:
            u = self.fail[u]
        return self.goto[u].get(a, 0)

    def delta(self, u, a):
        v = self.step(u, a)
        dC = (self.C[v] - self.pcom[v]) if self.final[v] else 0.0
        return dC + self.U[v] - self.U[u], v

    def total(self, toks):
        u, s = 0, 0.0
        for a in toks:
            d, u = self.delta(u, a)
            s += d
        return s, u
