"""Summarise ncu evidence for profiles/ (run here, on the CPU box, on reports brought back by gpurun).

  python profiles/summarize.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
      --workload c4 --tag r1 [--frames 25600]

Writes profiles/<tag>_ncu_summary.md and merges the dominant kernel's DRAM traffic per launch into
profiles/ncu_summary.json (read by bench.py for roofline.traffic)."""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warp_latency_issue_stalled_barrier", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]
UNIT = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "usecond": 1e-6,
        "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9, "s": 1.0, "second": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    res = []
    for v in vals:
        d = {}
        for i, h in enumerate(hdr):
            d[h] = (v[i], units[i])
        res.append(d)
    return res


def to_si(v, u):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * UNIT.get(u, 1.0)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    iu = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    agg = {}
    for r in rows[1:]:
        name = r[ik]
        if "flexctc::" in name:  # our kernels: bare name without namespace / template / arguments
            short = name.replace("<unnamed>::", "").replace("void ", "").split("(")[0].split("<")[0].split("::")[-1]
        else:
            short = name[:60]
        t = float(r[iv].replace(",", "")) * (UNIT.get(r[iu], 1e-9) if iu is not None else 1e-9)
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += t
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--frames", type=int, default=25600)
    ap.add_argument("--note", default="")
    ap.add_argument("--kernel", default="ctc_beam_kernel", help="substring of the captured kernel's name")
    ap.add_argument("--alg-per-frame", type=float, default=4 * 1025 + 3 * 16,
                    help="algorithmic bytes per utterance-frame (DESIGN.md)")
    a = ap.parse_args()
    md = [f"# ncu summary ({a.tag}, workload {a.workload})", ""]
    if a.note:
        md += [a.note, ""]
    js_path = os.path.join(HERE, "ncu_summary.json")
    js = json.load(open(js_path)) if os.path.exists(js_path) else {}
    if a.rep:
        k = [d for d in raw(a.rep) if a.kernel in d.get("Kernel Name", ("", ""))[0]]
        d = k[0]
        md += [f"## `ncu --set full` capture of `{a.kernel}` (one launch, cold L2 after the bench's flush)", "",
               "| metric | value | unit |", "|---|---|---|"]
        for m in METRICS:
            if m in d:
                md.append(f"| {m} | {d[m][0]} | {d[m][1]} |")
        rd = to_si(*d["dram__bytes_read.sum"])
        wr = to_si(*d["dram__bytes_write.sum"])
        dur = to_si(*d["gpu__time_duration.sum"])
        alg = a.frames * a.alg_per_frame
        md += ["", f"DRAM traffic per launch: {(rd + wr) / 1e6:.1f} MB (read {rd / 1e6:.1f} + write {wr / 1e6:.1f}); "
               f"algorithmic bytes {alg / 1e6:.1f} MB; duration under ncu {dur * 1e3:.3f} ms.", ""]
        js[a.workload] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                          "algorithmic_bytes": alg, "duration_s_under_ncu": dur,
                          "source": f"profiles/{a.tag}_ncu_summary.md ({os.path.basename(a.rep)})"}
        json.dump(js, open(js_path, "w"), indent=1)
    if a.launches:
        agg = launches(a.launches)
        tot = sum(v[1] for v in agg.values())
        md += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`)", "",
               "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            md.append(f"| {name} | {n} | {t * 1e3:.3f} | {100 * t / tot:.1f}% |")
        md.append("")
    out = os.path.join(HERE, f"{a.tag}_ncu_summary.md")
    open(out, "w").write("\n".join(md) + "\n")
    print(out)


if __name__ == "__main__":
    main()
