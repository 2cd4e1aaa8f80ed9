"""Per-frame cycle split of the beam kernel from its device counters (needs the library built with
`python paper_2508_07315_b200/build.py --force --timers`; the default build compiles the timers out).

  python profiles/phase_split.py [--workload c4] [--nt 256]

Prints one JSON line: counters per step and cycles per frame for each phase (thread 0's clock)."""
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
    ap.add_argument("--beam", type=int, default=0)
    a = ap.parse_args()
    wl = synth.WORKLOADS[a.workload]
    _, D, L, arpa, ph = synth.workload_inputs(a.workload)
    K = a.beam or wl.beam
    lm = F.LM(arpa, wl.V) if arpa is not None else None
    bt = F.Boost(ph, 1.0, wl.V) if ph is not None else None
    cfg = F.config(K, wl.alpha_lm if lm else 0.0, wl.alpha_bt if bt else 0.0, wl.beta, wl.theta, wl.merge_mode)
    Dd, Ld = torch.from_numpy(D).cuda(), torch.from_numpy(L).cuda()
    ws = F.make_workspace(Dd.shape[0], Dd.shape[1], Dd.shape[2], cfg)
    F.decode(Dd, Ld, cfg, lm, bt, workspace=ws)
    torch.cuda.synchronize()
    s = F.stats(ws)
    fr = max(1, s["frames"])
    per = {k: round(v / fr, 1) for k, v in s.items() if k.startswith("cyc_")}
    hv = max(1, s["heavy_frames"])
    lf = max(1, s.get("light_frames", 0))
    light = {k: round(v / lf, 1) for k, v in s.items() if k.startswith("lcyc_")}
    out = {"workload": a.workload, "K": K, "counters": s, "cycles_per_frame": per,
           "heavy_fraction": round(s["heavy_frames"] / fr, 3),
           "cycles_per_heavy_frame": round(s["cyc_heavy_frames"] / hv, 1),
           "light_frame_split": light}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
