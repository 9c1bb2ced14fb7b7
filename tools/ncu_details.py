"""Print section / metric / value of an .ncu-rep (details page), compactly.
python tools/ncu_details.py REP [regex]"""
import csv, io, re, subprocess, sys
rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, si, mi, ui, vi = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
for r in rows[1:]:
    line = f"{r[ki].split('(')[0][:28]:28s} | {r[si][:28]:28s} | {r[mi][:45]:45s} | {r[vi]} {r[ui]}"
    if not pat or pat.search(line):
        print(line)
