"""Summarise ncu output brought back by gpurun into profiles/ (committed evidence).

    python tools/ncu_summarize.py --round 1 --launches gpurun_out/launches_c3.csv \
        --full gpurun_out/prof_fused_c3.ncu-rep --kernel fused --workload c3bulk

Writes profiles/r<NN>_<workload>_launches.csv (the per-launch list as captured),
profiles/r<NN>_<workload>_ncu.md (per-kernel medians + the full-capture
metrics) and profiles/ncu_traffic.json (dram bytes per launch of the dominant
kernel, read by bench.py for its roofline "traffic" key).
"""
import argparse
import collections
import csv
import io
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_selected",
    "smsp__pcsamp_sample_count",
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
              "ms": 1e-3, "nsecond": 1e-9, "msecond": 1e-3}


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in data:
        agg[r[ki].split("(")[0]][(r[mi], r[ui])].append(float(r[vi].replace(",", "")))
    return agg


def full_capture(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for m in FULL_METRICS:
            if m in h:
                d[m] = (r[h.index(m)], units[h.index(m)])
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", type=int, required=True)
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--kernel", default="fused")
    ap.add_argument("--workload", default="c3bulk")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    prof = os.environ.get("CT_PROFILES_DIR") or os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    os.makedirs(prof, exist_ok=True)
    tag = f"r{a.round:02d}_{a.workload}"
    md = [f"# ncu summary, round {a.round}, workload {a.workload}", ""]
    if a.note:
        md += [a.note, ""]
    if a.launches:
        shutil.copy(a.launches, os.path.join(prof, f"{tag}_launches.csv"))
        agg = launch_table(a.launches)
        md += ["## Launch list (`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
               "--clock-control none`; cold-cache, serialised: compare shares, not absolutes)", "",
               "| kernel | launches | median time | median DRAM read | median DRAM write | share of kernel time |",
               "|---|---|---|---|---|---|"]
        tot = sum(sum(v.get(("gpu__time_duration.sum", u), []) or [0]) for v in agg.values()
                  for u in ("ns", "nsecond", "us", "usecond"))
        for k, v in agg.items():
            t = next((x for key, x in v.items() if key[0] == "gpu__time_duration.sum"), [0])
            tu = next((key[1] for key in v if key[0] == "gpu__time_duration.sum"), "ns")
            rd = next((x for key, x in v.items() if key[0] == "dram__bytes_read.sum"), [0])
            wr = next((x for key, x in v.items() if key[0] == "dram__bytes_write.sum"), [0])
            med = lambda xs: sorted(xs)[len(xs) // 2]
            share = sum(t) / tot if tot else 0
            md.append(f"| `{k}` | {len(t)} | {med(t):.0f} {tu} | {med(rd) / 1e6:.2f} MB | {med(wr) / 1e6:.2f} MB | {share:.1%} |")
        md.append("")
    if a.full:
        caps = full_capture(a.full)
        md += [f"## Full capture (`ncu --set full --clock-control none --import-source on`) of `{a.kernel}`", "",
               "| metric | " + " | ".join(f"launch {i}" for i in range(len(caps))) + " |",
               "|---|" + "---|" * len(caps)]
        for m in FULL_METRICS:
            vals = [c.get(m) for c in caps]
            if all(v is None for v in vals):
                continue
            md.append(f"| `{m}` | " + " | ".join(f"{v[0]} {v[1]}" if v else "" for v in vals) + " |")
        md.append("")
        per = []
        for c in caps:
            rd, ru = c["dram__bytes_read.sum"]
            wr, wu = c["dram__bytes_write.sum"]
            per.append(float(rd.replace(",", "")) * UNIT_SCALE.get(ru, 1) + float(wr.replace(",", "")) * UNIT_SCALE.get(wu, 1))
        tj = {"workload": a.workload, "n_gpus": 1, "kernel": a.kernel, "round": a.round,
              "dram_bytes_per_launch": sum(per) / len(per), "launches_captured": len(per),
              "source": os.path.basename(a.full)}
        tpath = os.path.join(prof, "ncu_traffic.json")
        try:
            allj = json.load(open(tpath))
            if "workload" in allj:            # old single-entry format
                allj = {allj["workload"]: allj}
        except Exception:
            allj = {}
        allj[a.workload] = tj
        json.dump(allj, open(tpath, "w"), indent=1)
        md.append(f"DRAM traffic per launch (read + write): {tj['dram_bytes_per_launch'] / 1e6:.1f} MB")
    open(os.path.join(prof, f"{tag}_ncu.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
