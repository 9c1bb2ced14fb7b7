"""Top source lines by warp-stall samples from `ncu --page source --csv --print-source cuda,sass`.
usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass | python tools/ncu_lines.py [topN]"""
import csv, sys

top = int(sys.argv[1]) if len(sys.argv) > 1 else 25
rows = list(csv.reader(sys.stdin))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
iS = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
lines = []
total = 0
for r in rows[hi + 1:]:
    if not r or r[0] in ("", "Line No") or len(r) <= iS:
        continue
    try:
        s = int(float(r[iS] or 0))
    except ValueError:
        continue
    total += s
    br = sorted(((int(float(r[i] or 0)), c[6:]) for i, c in stall_cols if r[i] not in ("", "0")), reverse=True)[:3]
    lines.append((s, r[0], r[1][:90], br))
lines.sort(reverse=True)
print("total samples", total)
for s, ln, src, br in lines[:top]:
    print(f"{s:6d} {100*s/max(total,1):5.1f}% L{ln:>5} {src}  {br}")
