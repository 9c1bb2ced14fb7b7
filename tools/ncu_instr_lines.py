"""Top source lines by executed instructions (and stall samples) of each kernel in
an .ncu-rep.  python tools/ncu_instr_lines.py REP [topN]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
agg = {}
for k, i in enumerate(hi):
    h = rows[i]
    if "Instructions Executed" not in h:
        continue
    ie, iss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    end = hi[k + 1] - 1 if k + 1 < len(hi) else len(rows)
    for r in rows[i + 1:end]:
        if len(r) <= ie or not r[ie]:
            continue
        try:
            v, st = float(r[ie]), float(r[iss] or 0)
        except ValueError:
            continue
        a = agg.setdefault((r[0], r[1][:100]), [0.0, 0.0])
        a[0] += v
        a[1] += st
tot = sum(v[0] for v in agg.values())
tots = sum(v[1] for v in agg.values())
print(f"total instructions {tot/1e6:.1f}M, stall samples {tots:.0f}")
for key, (v, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v/1e6:8.1f}M {100*v/tot:5.1f}%  st {100*st/max(tots,1):5.1f}%  L{key[0]:>4} {key[1]}")
