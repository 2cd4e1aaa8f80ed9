"""Summarise an ncu source export (--page source --csv --print-source cuda,sass) by CUDA line:
samples per stall reason. Usage: python profiles/ncu_lines.py export.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[2]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {h: hdr.index(h) for h in reasons + ["Warp Stall Sampling (All Samples)", "Instructions Executed"]}


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


tot = {h: 0 for h in reasons}
lines = []
for r in rows[3:]:
    if r[0] != "" and r[0].isdigit():
        d = {h: num(r[idx[h]]) for h in reasons}
        for h in reasons:
            tot[h] += d[h]
        lines.append((num(r[idx["Warp Stall Sampling (All Samples)"]]), int(r[0]), r[1][:70], d))
S = sum(tot.values())
print("stall totals:", ", ".join(f"{h[6:]} {100 * v / S:.1f}%" for h, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
for s, ln, src, d in sorted(lines, reverse=True)[:top]:
    main = sorted(d.items(), key=lambda x: -x[1])[:3]
    print(f"{100 * s / S:5.1f}% L{ln:4d} {src:70s} " + " ".join(f"{h[6:]}={v}" for h, v in main if v))
