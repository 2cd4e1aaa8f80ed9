"""Time flexctc_decode on a workload under variations of the configuration (kernel-time
ablations for DESIGN.md). CUDA events around each decode, L2 flushed before each, mean of N.

  python tools/ablate.py --workload c4 [--steps 20]
Prints one JSON line per variant."""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2508_07315_b200 as F  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--only", default="", help="run only this variant")
    a = ap.parse_args()
    wl = synth.WORKLOADS[a.workload]
    _, D, L, arpa, ph = synth.workload_inputs(a.workload)
    lm = F.LM(arpa, wl.V) if arpa is not None else None
    bt = F.Boost(ph, 1.0, wl.V) if ph is not None else None
    Dd, Ld = torch.from_numpy(D).cuda(), torch.from_numpy(L).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    base = dict(beam=wl.beam, alpha_lm=wl.alpha_lm if lm else 0.0, alpha_bt=wl.alpha_bt if bt else 0.0,
                beta=wl.beta, theta=wl.theta, merge_mode=wl.merge_mode)
    variants = [("baseline", {}, True, True), ("max merge", {"merge_mode": 1}, True, True),
                ("no boost", {}, True, False), ("no LM", {}, False, True), ("no LM, no boost", {}, False, False),
                ("theta 8", {"theta": 8.0}, True, True), ("beam 8", {"beam": 8}, True, True),
                ("beam 32", {"beam": 32}, True, True)]
    for name, over, use_lm, use_bt in variants:
        if a.only and name != a.only:
            continue
        kw = dict(base)
        kw.update(over)
        cfg = F.config(**kw)
        ws = F.make_workspace(Dd.shape[0], Dd.shape[1], Dd.shape[2], cfg)
        g_lm, g_bt = (lm if use_lm else None), (bt if use_bt else None)
        out = None
        for _ in range(3):
            out = F.decode(Dd, Ld, cfg, g_lm, g_bt, workspace=ws, outputs=out)
        ts = []
        for _ in range(a.steps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = F.decode(Dd, Ld, cfg, g_lm, g_bt, workspace=ws, outputs=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        s = F.stats(ws)
        print(json.dumps({"workload": a.workload, "variant": name, "ms": round(sum(ts) / len(ts), 4),
                          "heavy_frames": s["heavy_frames"], "exact_sparse": s["exact_sparse"],
                          "top_token_stages": s["top_token_stages"]}), flush=True)


if __name__ == "__main__":
    main()
