"""Per-CUDA-line summary of an ncu source export (ncu -i X.ncu-rep --page source --csv
--print-source cuda,sass): warp-stall samples (with the top stall reasons) and executed warp
instructions per source line of one file. Usage: python tools/ncu_src.py export.csv file_substring [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cur = None
hdr = None
out = []
tot_reason = {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if cur is None or want not in cur or not r or not r[0].isdigit():
        continue
    num = lambda x: int(x) if x.isdigit() else 0
    s = num(r[4])
    ins = num(r[7])
    reasons = {}
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            reasons[h[6:]] = num(r[i])
            tot_reason[h[6:]] = tot_reason.get(h[6:], 0) + num(r[i])
    out.append((s, ins, int(r[0]), r[1][:80], reasons))
S = sum(x[0] for x in out) or 1
I = sum(x[1] for x in out) or 1
RS = sum(tot_reason.values()) or 1
print(f"samples {S}, warp instructions {I}")
print("stalls:", ", ".join(f"{k} {100 * v / RS:.1f}%" for k, v in sorted(tot_reason.items(), key=lambda x: -x[1]) if v > 0.01 * RS))
for s, ins, ln, src, rs in sorted(out, reverse=True)[:top]:
    main = sorted(rs.items(), key=lambda x: -x[1])[:2]
    print(f"{100 * s / S:5.1f}% {100 * ins / I:5.1f}%i L{ln:4d} {src:80s} " + " ".join(f"{k}={v}" for k, v in main if v))
