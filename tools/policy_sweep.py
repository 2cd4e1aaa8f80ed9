"""Warp-per-utterance kernel vs the persistent CTA kernel on c4-shaped batches of B utterances
(launch-policy evidence): CUDA events around flexctc_decode, inputs resident, L2
flushed before each step. FLEXCTC_WARP=1 forces the warp path, =0 the CTA kernel.

  python tools/policy_sweep.py [--bs 64,148,256,512,1024,2048] [--workload c4] [--steps 5]"""
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
    ap.add_argument("--bs", default="64,148,256,512,1024,2048")
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--modes", default="0,1")
    a = ap.parse_args()
    wl = synth.WORKLOADS[a.workload]
    bs = [int(x) for x in a.bs.split(",")]
    base = 256
    _, D, L, arpa, ph = synth.workload_inputs(a.workload, B=base)
    lm = F.LM(arpa, wl.V) if arpa else None
    bt = F.Boost(ph, 1.0, wl.V) if ph else None
    cfg = F.config(wl.beam, wl.alpha_lm if lm else 0.0, wl.alpha_bt if bt else 0.0, wl.beta, wl.theta, wl.merge_mode)
    Dall, Lall = torch.from_numpy(D).cuda(), torch.from_numpy(L).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for B in bs:
        reps = (B + base - 1) // base
        Dd = Dall.repeat(reps, 1, 1)[:B].contiguous()
        Ld = Lall.repeat(reps)[:B].contiguous()
        ws = F.make_workspace(B, Dd.shape[1], Dd.shape[2], cfg)
        for mode in a.modes.split(","):
            # "0" / "1": FLEXCTC_WARP; "0nt128": the CTA kernel at 128 threads per utterance
            if mode[0] == "d":  # the library's own launch policy
                os.environ.pop("FLEXCTC_WARP", None)
            else:
                os.environ["FLEXCTC_WARP"] = mode[0]
            if "nt" in mode:
                os.environ["FLEXCTC_NT"] = mode.split("nt")[1]
            else:
                os.environ.pop("FLEXCTC_NT", None)
            out = None
            for _ in range(2):
                out = F.decode(Dd, Ld, cfg, lm, bt, workspace=ws, outputs=out)
            tot = 0.0
            for _ in range(a.steps):
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                out = F.decode(Dd, Ld, cfg, lm, bt, workspace=ws, outputs=out)
                e1.record()
                torch.cuda.synchronize()
                tot += e0.elapsed_time(e1)
            ms = tot / a.steps
            frames = int(Ld.sum())
            print(json.dumps({"workload": a.workload, "B": B, "mode": mode, "ms": round(ms, 4),
                              "rtfx": round(frames * 0.04 / (ms / 1000.0), 1)}), flush=True)


if __name__ == "__main__":
    main()
