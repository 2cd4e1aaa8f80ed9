"""Per-frame cycle split of the warp beam kernel (K <= 32) from its device counters. Needs the
timers library: FLEXCTC_PHASE_TIMERS=1 python tools/warp_split.py [--workload c4]
(builds libflexctc_timers.so on first use). One JSON line: per frame class (frames with scored
pairs / with a row scan only / light) the mean cycles of: ring wait, blank+repeat candidates and
ranks, token filter + pair scoring, TopK + beams.update, recombination."""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["FLEXCTC_PHASE_TIMERS"] = "1"

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_07315_b200 as F  # noqa: E402
from paper_2508_07315_b200 import flexctc as FX  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    a = ap.parse_args()
    wl = synth.WORKLOADS[a.workload]
    _, D, L, arpa, ph = synth.workload_inputs(a.workload)
    lm = F.LM(arpa, wl.V) if arpa is not None else None
    bt = F.Boost(ph, 1.0, wl.V) if ph is not None else None
    cfg = F.config(wl.beam, wl.alpha_lm if lm else 0.0, wl.alpha_bt if bt else 0.0, wl.beta, wl.theta, wl.merge_mode)
    Dd, Ld = torch.from_numpy(D).cuda(), torch.from_numpy(L).cuda()
    ws = F.make_workspace(Dd.shape[0], Dd.shape[1], Dd.shape[2], cfg)
    F.decode(Dd, Ld, cfg, lm, bt, workspace=ws)
    torch.cuda.synchronize()
    raw = np.zeros(48, dtype=np.uint64)
    FX.lib.flexctc_get_stats(FX._ptr(ws.buf), raw.ctypes.data_as(ctypes.c_void_p), 48)
    names = ["wait", "rb_rank", "pairs", "topk_update", "merge"]
    out = {"workload": a.workload, "frames": int(raw[0]), "evals": int(raw[3]), "tokens": int(raw[2]),
           "scan_frames": int(raw[4]), "pair_frames": int(raw[15]), "batches": int(raw[24]),
           "row_loads": int(raw[25]), "lm_global": int(raw[26]), "lm_cached_row": int(raw[27]),
           "jobs": int(raw[28]), "job_pairs": int(raw[29]), "job_candidates": int(raw[23]), "job_overflows": int(raw[22]), "lm_arc_cache": int(raw[21]),
           "kernel": FX.last_kernel()}
    out["pair_detail_cycles_per_pair_frame"] = {k: round(int(raw[36 + i]) / max(1, int(raw[35])), 1) for i, k in
                                                enumerate(["phaseA", "staging", "scan", "gather", "global_evals"])}
    out["pair_detail_cycles_per_pair_frame"]["pushes_with_keys"] = int(raw[41])
    for ci, cls in enumerate(["pair", "scan_only", "light"]):
        if cls == "scan_only":
            continue
        n = int(raw[30 + 6 * ci + 5])
        out[cls] = {"frames": n, **{k: round(int(raw[30 + 6 * ci + j]) / max(1, n), 1) for j, k in enumerate(names)}}
        out[cls]["total"] = round(sum(out[cls][k] for k in names), 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
