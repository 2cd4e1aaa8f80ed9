"""Speed trends of PAPER.md Fig. 1 (RTFx vs batch size, beams 4/8/16 and greedy, LM on) and
Fig. 2 (RTFx vs beam size up to 128, LM + phrase boosting, B = 32) on B200 with the synthetic
c4 inputs. Greedy = Algorithm 1 at K = 1 (fused greedy, Table II rows).

  python sweep.py [--fig 1|2|both] [--steps 5]

Prints one JSON line per point: {"fig", "B", "K", "lm", "boost", "ms", "rtfx", "frames_beams_per_s"}.
Timing: CUDA events around flexctc_decode, inputs resident, L2 flushed before each step."""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_07315_b200 as F  # noqa: E402
import synth  # noqa: E402


def timed(Dd, Ld, cfg, lm, bt, steps, flush):
    ws = F.make_workspace(Dd.shape[0], Dd.shape[1], Dd.shape[2], cfg)
    out = None
    for _ in range(2):
        out = F.decode(Dd, Ld, cfg, lm, bt, workspace=ws, outputs=out)
    tot = 0.0
    for _ in range(steps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = F.decode(Dd, Ld, cfg, lm, bt, workspace=ws, outputs=out)
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fig", default="both")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--bmax", type=int, default=1024)
    a = ap.parse_args()
    wl = synth.WORKLOADS["c4"]
    base_B = 256
    _, D, L, arpa, ph = synth.workload_inputs("c4", B=base_B)
    lm = F.LM(arpa, wl.V)
    bt = F.Boost(ph, 1.0, wl.V)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    Dall = torch.from_numpy(D).cuda()
    Lall = torch.from_numpy(L).cuda()

    def batch(B):
        reps = (B + base_B - 1) // base_B
        Dd = Dall.repeat(reps, 1, 1)[:B].contiguous() if reps > 1 else Dall[:B].contiguous()
        Ld = Lall.repeat(reps)[:B].contiguous() if reps > 1 else Lall[:B].contiguous()
        return Dd, Ld

    def point(fig, B, K, use_lm, use_bt):
        Dd, Ld = batch(B)
        cfg = F.config(K, wl.alpha_lm if use_lm else 0.0, wl.alpha_bt if use_bt else 0.0, wl.beta, wl.theta)
        ms = timed(Dd, Ld, cfg, lm if use_lm else None, bt if use_bt else None, a.steps, flush)
        frames = float(Ld.sum())
        print(json.dumps({"fig": fig, "B": B, "K": K, "lm": use_lm, "boost": use_bt, "ms": round(ms, 4),
                          "rtfx": frames * synth.FRAME_SECONDS / (ms / 1e3),
                          "frames_beams_per_s": frames * K / (ms / 1e3)}), flush=True)

    if a.fig in ("1", "both"):
        for K in (1, 4, 8, 16):
            for B in (1, 4, 16, 32, 64, 128, 256, 512, 1024):
                if B <= a.bmax:
                    point(1, B, K, True, False)
    if a.fig in ("2", "both"):
        for K in (1, 4, 8, 16, 32, 64, 128):
            point(2, 32, K, True, True)


if __name__ == "__main__":
    main()
