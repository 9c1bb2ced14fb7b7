#!/usr/bin/env python
"""Benchmark of the Compact-Table propagation hot path on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c3bulk|c3b|c4|c5|lin]

Default workload (BASELINE config 3, "c3bulk"): random positive table, arity 8,
domain 100, 1e7 tuples (1.0 GB of support bitsets); one step = restore the
root state (device copy) + one ct_propagate of a seeded bulk removal (a random
50 % of every variable's values), i.e. one pass of every §8(a) row: ingest,
updateTable (dense, HBM-bound), index compaction, emptiness check, residue
filter, finalize.  At N > 1 (torchrun) the table is tuple-range sharded over
the N GPUs and the per-row support flags are OR-combined with an in-library
NCCL all-reduce inside every step (strong scaling: the table is fixed).

`value` = propagations/s with inputs resident in HBM (device-buffer entry
point, CUDA events on the library stream, max over ranks).  `e2e` = the same
metric through the synchronous host-buffer C call ct_propagate (H2D of the
removal set and D2H of status+domains inside every step).  `roofline` = the
dominant kernel (k_fast, the whole call in one launch): bytes it loads/stores per launch (counted by the
kernel itself) / its CUDA-event duration, against MEASURED_PEAKS.json's HBM
copy bandwidth.  `cpu_baseline` = the CPU oracle (oracle/, plain C brute
force) on the host cores, rank 0 at N = 1 only.  `latency` = p50/p90/p99 of
ct_propagate on BASELINE config 2 (arity 5, domain 20, 1e5 tuples, 1000
random-removal calls, policy P(2, 0.5)).

--workload c3b: the banded C3b table (x_i = (x0*c_i + u_i) mod 100, u_i < 10);
each step fixes x0 to one seeded value, so 630 values of x1..x7 lose every
support and the filter scans their whole rows over the compacted index: the
HBM-bound filterDomains workload.  c4 / c5 / lin: see run_c4 /
run_c5 / run_lin (lin = the paper-shaped knapsack table).

--impl reference times the oracle (the reference arm of this tier) on the same
workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0   # GB/s, /opt/skills/guides/B200_PROFILING.md fallback


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: copy_ of 1 Gi bf16)"
    except Exception:
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------- clocks sampler
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.2)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(workload, world, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/ncu_traffic.json, written by tools/ncu_summarize.py), or None."""
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        allj = json.load(open(tpath))
        if "workload" in allj:
            allj = {allj["workload"]: allj}
        tj = allj.get(workload) or {}

        def base(name):   # "void ctk::k_bupdate<32>" / "k_bupdate" -> "k_bupdate"
            return str(name).replace("void ", "").split("::")[-1].split("<")[0].strip()

        if tj.get("n_gpus", 1) == world and base(tj.get("kernel")) == base(kernel):
            return tj.get("dram_bytes_per_launch")
    except Exception:
        pass
    return None


# ---------------------------------------------------------------- workloads
def c3_problem(t=10_000_000):
    from workloads import random_table
    return random_table(8, 100, t, seed=3, name=f"C3 random n=8 d=100 t={t:.0e} seed=3")


def c3b_problem(t=10_000_000):
    from workloads import banded_table
    return banded_table(8, 100, t, seed=4, name=f"C3b banded n=8 d=100 t={t:.0e} seed=4")


# C3 workload -> (problem builder, tuples, i.i.d.?): SURVEY §8(d) evaluates the
# HBM target also on the same two workloads rebuilt at t = 1e6 ("c3bulk6" /
# "c3b6"; their 100 MB of supports may sit in L2 across back-to-back calls, so
# their CUDA-event bandwidth is L2-assisted, and the HBM fraction comes from
# ncu with the caches flushed between replays)
C3_FAMILY = {"c3bulk": (c3_problem, 10_000_000, True), "c3b": (c3b_problem, 10_000_000, False),
             "c3bulk6": (c3_problem, 1_000_000, True), "c3b6": (c3b_problem, 1_000_000, False)}


def fix_patterns(root_member, d, count: int, seed: int = 12):
    """C3b calls: remove all but one seeded value of x0."""
    from workloads import Rng, fix_one_value_removal
    rng = Rng(seed)
    return [fix_one_value_removal(rng, root_member, d, var=0) for _ in range(count)]


WORKLOADS = {
    "c3bulk": dict(metric="propagations/s (C3 bulk ct_propagate, 1e7-tuple table)",
                   table="arity 8, domain 100, 1e7 tuples, seed 3",
                   step="ct_propagate_from_async(work, root) of a bulk removal (50% of every var); the root "
                        "is only read, so a step needs no restore copy"),
    "c3b": dict(metric="propagations/s (C3b banded ct_propagate, filter-heavy, 1e7-tuple table)",
                table="banded arity 8, domain 100, 1e7 tuples, seed 4 (x_i = (x0*c_i + u_i) mod 100, u_i < 10)",
                step="ct_propagate_from_async(work, root) fixing x0 to one seeded value "
                     "(630 unsupported values -> full filter scans)"),
    "c3bulk6": dict(metric="propagations/s (C3 bulk ct_propagate, 1e6-tuple table)",
                    table="arity 8, domain 100, 1e6 tuples, seed 3",
                    step="as c3bulk, on the table rebuilt at t = 1e6 (SURVEY 8(d))"),
    "c3b6": dict(metric="propagations/s (C3b banded ct_propagate, filter-heavy, 1e6-tuple table)",
                 table="banded arity 8, domain 100, 1e6 tuples, seed 4",
                 step="as c3b, on the table rebuilt at t = 1e6 (SURVEY 8(d))"),
}


def c2_problem():
    from workloads import random_table
    return random_table(5, 20, 100_000, seed=1, name="C2 random n=5 d=20 t=1e5 seed=1")


def c4_problem():
    from workloads import random_table
    return random_table(6, 50, 1_000_000, seed=5, name="C4 random n=6 d=50 t=1e6 seed=5")


def bulk_patterns(root_member, d, count: int, seed: int = 11):
    from workloads import Rng, bulk_removal
    rng = Rng(seed)
    return [bulk_removal(rng, root_member, d, q=0.5) for _ in range(count)]


# ---------------------------------------------------------------- f2: LIN-shaped (knapsack) table
def run_lin(args):
    """a knapsack-configuration table shaped like the paper's
    LIN_B set (Table tbl:instances: 120 variables, max domain
    600, 1e4 tuples; many support rows over few words, filter-heavy) driven by a
    policy P(2, 0.5) walk (restore the root after FAIL or when solved).  The
    walk is first run with the synchronous host-buffer call (e2e and per-call
    latency), recording every call's removal set and restores; the same
    sequence is then replayed with the device-buffer call for the device-timed
    value (identical states: the library is deterministic).  Latency-bound:
    the roofline object reports the bytes the kernels count against HBM peak
    only for completeness.  Replicas only (one table per GPU, no collective)."""
    import ctypes
    import torch
    from paper_2507_18413_b200 import CT_OK, Table
    from paper_2507_18413_b200 import ct as C
    from workloads import Rng, knapsack_table, LIN_PRESETS, member_to_bitmap, bitmap_to_member
    from workloads.policies import walk_removal
    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    preset = LIN_PRESETS["lin_b"]
    p = knapsack_table(seed=21, **preset)
    t0 = time.perf_counter()
    tab = Table(p.lo, p.d, p.tuples, device=dev)
    build_s = time.perf_counter() - t0
    root_m = bitmap_to_member(tab.root_dom, p.d)
    wd = tab.Wd
    n_calls = args.steps
    # ---- e2e + latency: the synchronous C call on host buffers, recording the walk
    st = tab.root.clone()
    rem = np.zeros(wd, np.uint64)
    out = np.zeros(wd, np.uint64)
    pr = np.zeros(wd, np.uint64)
    fn = C.lib().ct_propagate
    cargs = (st.handle, rem.ctypes.data_as(ctypes.c_void_p), out.ctypes.data_as(ctypes.c_void_p),
             pr.ctypes.data_as(ctypes.c_void_p))
    rng = Rng(2, lanes=1)
    cur = root_m.copy()
    seq = []             # (restore_before, removal bitmap)
    lat = []
    restore = False
    fails = solved = 0
    t_e2e = 0.0
    k = 0
    while len(seq) < args.warmup + n_calls:
        r = walk_removal(rng, cur, p.d)
        if r is None:
            cur = root_m.copy()
            restore = True
            solved += 1
            continue
        rem[:] = member_to_bitmap(r, p.d)
        if restore:
            st.copy_from(tab.root)
        a = time.perf_counter()
        s = fn(*cargs)
        b = time.perf_counter()
        if s < 0:
            raise RuntimeError(C.ct_last_error())
        if len(seq) >= args.warmup:
            lat.append((b - a) * 1e6)
            t_e2e += b - a
        seq.append((restore, rem.copy()))
        restore = False
        if s == CT_OK:
            cur = bitmap_to_member(out, p.d)
        else:
            fails += 1
            cur = root_m.copy()
            restore = True
    st.close()
    # ---- device-timed replay (device buffers, async), same sequence
    work = tab.root.clone()
    rem_dev = torch.from_numpy(np.stack([x[1] for x in seq]).view(np.int64)).to(f"cuda:{dev}")
    od = torch.zeros(wd, dtype=torch.int64, device=f"cuda:{dev}")
    sd = torch.zeros(1, dtype=torch.int32, device=f"cuda:{dev}")
    stream = torch.cuda.ExternalStream(tab.stream_ptr, device=f"cuda:{dev}")

    def replay(lo, hi):
        for i in range(lo, hi):
            if seq[i][0]:
                work.copy_from(tab.root)
            work.propagate_async(rem_dev[i], od, None, sd)

    replay(0, args.warmup)
    work.synchronize()
    clocks = Clocks(dev)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    replay(args.warmup, len(seq))
    ev1.record(stream)
    ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    barrier(world)
    ms_max = max_over_ranks(ms, world)
    value = world * n_calls / (ms_max / 1e3)
    # per-kernel times + kernel-counted bytes: replay once more with events, reading stats per call
    work.copy_from(tab.root)
    C.ct_table_profile(tab.handle, True)
    C.ct_table_profile_read(tab.handle, reset=True)
    byts = 0
    for i in range(args.warmup, len(seq)):
        if seq[i][0]:
            work.copy_from(tab.root)
        work.propagate_async(rem_dev[i], od, None, sd)
        s_ = work.stats()
        byts += 8 * (s_.update_support_words + s_.filter_support_words) + 16 * (s_.words_in + s_.update_table_writes) \
            + 4 * (s_.words_in + s_.words_out) + 32 * s_.n_filter_items
    prof = C.ct_table_profile_read(tab.handle, reset=True)
    C.ct_table_profile(tab.handle, False)
    kname = C.KERNEL_PATHS.get(tab.info.kernel_path)
    k_n, k_ms = prof["small"]
    peak, peak_src = peaks()
    t_k = k_ms / max(k_n, 1) / 1e3
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        import oracle
        oracle.lib()
        cur = root_m.copy()
        n = 0
        t1 = time.perf_counter()
        i = 0
        while time.perf_counter() - t1 < min(args.cpu_budget, 10.0) or n == 0:
            restore_, r = seq[i % len(seq)]
            if restore_:
                cur = root_m.copy()
            ok, dout, _ = oracle.gac(p.lo, p.d, p.tuples, cur & (1 - bitmap_to_member(r, p.d)))
            cur = dout if ok else root_m.copy()
            n += 1
            i += 1
        dt = time.perf_counter() - t1
        cpu = {"value": n / dt, "unit": "propagations/s", "cores": 1, "kind": "oracle",
               "sample": f"first {n} calls of the same walk (oracle/ct_oracle.c brute-force scan of the 1e4 "
                         f"tuples, single thread) in {dt:.1f} s", "host_nproc": os.cpu_count()}
    q = lambda xs, f: sorted(xs)[min(len(xs) - 1, int(f * len(xs)))]
    tab.close()
    if rank == 0:
        line = {
            "metric": "propagations/s (LIN_B-shaped knapsack table, P(2,0.5) walk, ct_propagate)",
            "value": value, "unit": "propagations/s", "n_gpus": world, "steps": n_calls, "warmup": args.warmup,
            "ms_per_step": ms_max / n_calls, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u64", "data": "synthetic (seeded knapsack configurations, workloads.knapsack_table)",
            "config": {"workload": "lin", "table": f"knapsack n={p.n}, max domain {preset['max_dom']}, "
                                                   f"t={p.t}, R={p.R} support rows, {tab.info.words} words, seed 21",
                       "step": "restore after FAIL/solved (D2D) + ct_propagate_async of a P(2,0.5) removal",
                       "kernel_path": kname, "parallelism": "1 GPU" if world == 1 else f"{world} replicas",
                       "l2": "table (supports 0.03 GB) L2-resident: latency-bound regime", "build_s": round(build_s, 3),
                       "fails": fails, "restores_solved": solved},
            "roofline": {"bound": "hbm", "achieved": byts / max(k_n, 1) / t_k / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": byts / max(k_n, 1) / t_k / 1e9 / peak, "traffic": None,
                         "kernel": "ctk::k_wide + ctk::k_wide_filter" if kname == "k_wide" else "ctk::" + str(kname),
                         "bytes_per_launch": byts / max(k_n, 1), "ms_per_launch": t_k * 1e3, "peak_source": peak_src,
                         "note": "latency-bound: a call moves ~0.1-1 MB; the number that matters is latency"},
            "e2e": {"value": n_calls / t_e2e, "unit": "propagations/s", "h2d_bytes_per_step": 8 * wd,
                    "d2h_bytes_per_step": 8 * (1 + 2 * wd), "steps": n_calls,
                    "api": "ct_propagate (host buffers; mapped I/O; CUDA graph)"},
            "latency": {"calls": len(lat), "p50_us": q(lat, 0.5), "p90_us": q(lat, 0.9), "p99_us": q(lat, 0.99)},
            "gpu_launches": 2 * n_calls if kname == "k_wide" else n_calls,
            "clocks": clk, "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ---------------------------------------------------------------- distributed
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------- our arm
def algorithmic_bytes(table_words_in, table_words_out, rows, kept_items, removed_values):
    """SURVEY §8(d) per-call model at 64-bit-word granularity (the method's own
    minimum, residue-independent): B_upd = 8 L_in (sum_x r_x + 2) (support
    words of the chosen branch's rows over the active words + currTable read
    and write), B_filt = 8 K + 8 L_out Rm (one residue probe per kept value of
    s_sup + a full scan of every removed value's row over the surviving words)."""
    return 8 * table_words_in * (rows + 2) + 8 * kept_items + 8 * table_words_out * removed_values


def nonzero_words(bits):
    return int(np.count_nonzero(bits))


def nonzero_sectors(bits):
    """32-byte DRAM sectors (4 currTable words) holding a valid tuple: a scan of a
    support row over the active words must fetch at least these sectors."""
    b = np.asarray(bits)
    pad = (-b.size) % 4
    if pad:
        b = np.concatenate([b, np.zeros(pad, b.dtype)])
    return int(np.count_nonzero(b.reshape(-1, 4).any(axis=1)))


def measure_c3(workload, args, dev, world, rank, full=True, use_gather=True):
    """One C3-family workload (c3bulk or c3b): device-timed steps, per-kernel
    times, kernel-counted and algorithmic bytes; with full=True also the e2e
    host-buffer runs.  use_gather=False forces Alg. 3's support-row scans for
    the residue misses (ct_config.use_gather).  Returns a dict (rank 0's view;
    times max over ranks)."""
    import torch
    from paper_2507_18413_b200 import CT_OK, Table
    from paper_2507_18413_b200 import ct as C
    from paper_2507_18413_b200.sharded import broadcast_nccl_id
    from workloads import member_to_bitmap, bitmap_to_member

    build, t_rows, iid = C3_FAMILY[workload]
    p = build(t_rows)
    nid = broadcast_nccl_id() if world > 1 else None
    t0 = time.perf_counter()
    tab = Table(p.lo, p.d, p.tuples, device=dev, n_shards=world, shard_rank=rank, nccl_unique_id=nid,
                use_gather=use_gather)
    build_s = time.perf_counter() - t0
    assert tab.root_status == CT_OK
    combine = None
    if world > 1:
        # tuple-range shards: the flags are OR-combined inside k_fast over NVLink
        # peer memory (ct_peer_attach) unless --combine nccl or the attach fails
        import torch.distributed as dist
        combine = "nccl"
        if getattr(args, "combine", "peer") == "peer":
            # every rank must reach every other rank's memory (peer access over
            # NVLink) before any rank attaches: decided together, attached together
            devs = [None] * world
            dist.all_gather_object(devs, dev)
            ok = all(torch.cuda.can_device_access_peer(dev, o) for o in devs if o != dev)
            oks = [None] * world
            dist.all_gather_object(oks, ok)
            if all(oks):
                from paper_2507_18413_b200.sharded import attach_peers
                attach_peers(tab.handle)
                combine = "peer"
            else:
                print("[bench] no peer access between all ranks' GPUs: NCCL all-reduce combine", file=sys.stderr)
    root_m = bitmap_to_member(tab.root_dom, p.d)
    P = 16
    pats = bulk_patterns(root_m, p.d, P) if iid else fix_patterns(root_m, p.d, P)
    wd = tab.Wd
    rem_host = np.stack([member_to_bitmap(m, p.d) for m in pats])                 # [P][Wd] uint64
    rem_dev = torch.from_numpy(rem_host.view(np.int64)).to(f"cuda:{dev}")
    out_dom = torch.zeros(wd, dtype=torch.int64, device=f"cuda:{dev}")
    out_pr = torch.zeros(wd, dtype=torch.int64, device=f"cuda:{dev}")
    status = torch.zeros(1, dtype=torch.int32, device=f"cuda:{dev}")
    work = tab.root.clone()
    stream = torch.cuda.ExternalStream(tab.stream_ptr, device=f"cuda:{dev}")
    torch.cuda.synchronize()   # the tensors above were filled on torch's stream

    def step(k):
        # one call from the root into the work state (ct_propagate_from_async:
        # the root is only read, so no restore copy per step)
        work.propagate_from_async(tab.root, rem_dev[k % P], out_dom, out_pr, status)

    # per-pattern work counters (deterministic; untimed) and the SURVEY §8(d)
    # algorithmic bytes from the call's inputs/outputs (active words before /
    # after = non-zero words of this shard's currTable; rows of the chosen
    # branches; kept / removed values of s_sup)
    L_root = nonzero_words(tab.root.read_table())
    d_np = np.asarray(p.d)
    rb = np.concatenate([[0], np.cumsum(d_np)])
    per_pat = []
    for k in range(P):
        step(k)
        s = work.stats()
        assert s.last_status == CT_OK
        dout = bitmap_to_member(out_dom.cpu().numpy().view(np.uint64), p.d)
        din = root_m & (1 - pats[k])
        rows = kept = removed = 0
        for i in range(p.n):
            di = int(din[rb[i]:rb[i + 1]].sum())
            dl = int((root_m[rb[i]:rb[i + 1]] & pats[k][rb[i]:rb[i + 1]]).sum())
            if dl:
                rows += dl if dl < di else di                   # Alg. 2 L163 branch (tie -> dom)
            if di > 1:                                          # x in s_sup
                ko = int(dout[rb[i]:rb[i + 1]].sum())
                kept += ko
                removed += di - ko
        tbits = work.read_table()
        L_out = nonzero_words(tbits)
        sec_out = nonzero_sectors(tbits)
        # the gather filter reads the cells of every valid tuple once (one
        # 32-byte sector each, the cells of a sparse valid set share none)
        n_valid = int(np.unpackbits(tbits.view(np.uint8)).sum())
        per_pat.append(dict(L_in=s.words_in, L_out=s.words_out, rows=s.n_update_rows,
                            loads=s.update_support_words, writes=s.update_table_writes,
                            scan=s.filter_support_words, miss=s.n_residue_miss,
                            gathered=s.filter_gathered_tuples, valid=n_valid,
                            alg=algorithmic_bytes(L_root, L_out, rows, kept, removed),
                            alg_sector=algorithmic_bytes(L_root, 0, rows, kept, 0) + 32 * sec_out * removed,
                            alg_gather=algorithmic_bytes(L_root, 0, rows, kept, 0) + 32 * s.filter_gathered_tuples,
                            words_in=L_root, words_out=L_out, sectors_out=sec_out,
                            removed_values=removed, kept_values=kept))
    for k in range(args.warmup):
        step(k)
    work.synchronize()

    clocks = Clocks(dev)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for k in range(args.steps):
        step(k)
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    barrier(world)
    ms_max = max_over_ranks(ms, world)
    value = args.steps / (ms_max / 1e3)
    # per-kernel device times (roofline): the same steps again with CUDA events
    # around every kernel launch, outside the timed region above
    C.ct_table_profile(tab.handle, True)
    C.ct_table_profile_read(tab.handle, reset=True)
    for k in range(args.steps):
        step(k)
    prof = C.ct_table_profile_read(tab.handle, reset=True)
    C.ct_table_profile(tab.handle, False)
    phases = work.stats().phase_ns

    dom_kernel = next((k for k in ("fused", "small") if prof.get(k, (0, 0.0))[0]), "update")
    k_n, k_ms = prof[dom_kernel]
    counted = alg = alg_sec = 0
    gathered = any(c["gathered"] for c in per_pat)
    for k in range(args.steps):
        c = per_pat[k % P]
        b = 8 * c["loads"] + 16 * c["L_in"] + 16 * c["writes"] + 4 * (c["L_in"] + c["L_out"])
        if dom_kernel in ("fused", "small"):
            b += 8 * c["scan"] + 32 * c["gathered"]
        counted += b
        # bytes of the method the call ran: Alg. 3's scans (word model), or the
        # gather filter's cells when it resolved the misses
        alg += c["alg_gather"] if c["gathered"] else c["alg"]
        alg_sec += c["alg_gather"] if c["gathered"] else c["alg_sector"]
    kernel_name = "ctk::" + C.KERNEL_PATHS.get(tab.info.kernel_path, "k_update") if dom_kernel in ("fused", "small") \
        else "ctk::k_update"
    k_ms_per_launch = k_ms / max(k_n, 1)
    k_s = k_ms_per_launch / 1e3
    peak, peak_src = peaks()
    alg_pl = alg / max(k_n, 1)
    counted_pl = counted / max(k_n, 1)
    # c3b with the scans forced has its own capture (same kernel, other path)
    traffic = ncu_traffic(workload if use_gather or workload != "c3b" else "c3b_scan", world, kernel_name)
    step_ms = ms_max / args.steps
    roofline = {"bound": "hbm", "achieved": alg_pl / k_s / 1e9, "peak": peak, "unit": "GB/s",
                "frac": alg_pl / k_s / 1e9 / peak, "traffic": traffic, "kernel": kernel_name,
                "algorithmic_bytes_per_launch": alg_pl, "ms_per_launch": k_ms_per_launch,
                "counted_bytes_per_launch": counted_pl,
                "counted_frac": counted_pl / k_s / 1e9 / peak,
                "dram_frac": (traffic / k_s / 1e9 / peak) if traffic else None,
                "sector_floor_bytes_per_launch": alg_sec / max(k_n, 1),
                "sector_floor_frac": alg_sec / max(k_n, 1) / k_s / 1e9 / peak,
                "filter_method": "gather (valid tuples' cells)" if gathered else "Alg. 3 support-row scans",
                "bytes_model": ("SURVEY §8(d) update bytes 8 L_in (sum r_x + 2) + 8 K, plus the gather filter's "
                                "32 B (one sector of cells) per valid tuple it read") if gathered else
                               ("SURVEY §8(d): 8 L_in (sum r_x + 2) + 8 K + 8 L_out Rm at 64-bit-word granularity "
                                "(L = non-zero currTable words of the call's input / output); sector_floor: the "
                                "scans at 32-byte-sector granularity (32 x sectors holding a valid tuple x Rm)"),
                "peak_source": peak_src}
    out = dict(p=p, tab=tab, work=work, root_m=root_m, pats=pats, rem_host=rem_host, value=value, combine=combine,
               ms_per_step=step_ms, build_s=build_s, roofline=roofline, clocks=clk, per_pat=per_pat,
               kernel_ms={k: (v[1] / v[0] if v[0] else None) for k, v in prof.items()},
               kernel_share=k_ms_per_launch / step_ms,
               launches=sum(v[0] for k, v in prof.items() if k != "combine"),
               phase_ns=[int(x) for x in phases])
    if full:
        out["e2e"] = measure_c3_e2e(tab, work, rem_host, P, wd, args, world)
    return out


def measure_c3_e2e(tab, work, rem_host, P, wd, args, world):
    """e2e through the public API on host buffers (H2D of the removal set and
    D2H of status + domains + pruned inside every step)."""
    import torch
    e2e_steps = max(50, min(args.steps, 400))
    host_rems = [rem_host[k % P].copy() for k in range(e2e_steps)]
    barrier(world)
    torch.cuda.synchronize()
    for k in range(5):
        work.copy_from(tab.root)
        work.propagate(host_rems[k])
    barrier(world)
    t1 = time.perf_counter()
    o_dom, o_pr = np.zeros(wd, np.uint64), np.zeros(wd, np.uint64)
    for k in range(e2e_steps):
        work.copy_from(tab.root)
        work.propagate(host_rems[k], o_dom, o_pr)
    t2 = time.perf_counter()
    e2e_sync_s = max_over_ranks(t2 - t1, world)
    # the same calls kept in flight: ct_propagate_async on pinned host buffers
    # (every step's removal copied in by a DMA, its status + domains + pruned
    # values written back to host memory by the kernel; the host checks every
    # step's status after the last one)
    h_rem = torch.from_numpy(np.stack(host_rems).view(np.int64)).pin_memory()
    h_dom = torch.zeros((e2e_steps, wd), dtype=torch.int64).pin_memory()
    h_pr = torch.zeros((e2e_steps, wd), dtype=torch.int64).pin_memory()
    h_st = torch.full((e2e_steps,), -1, dtype=torch.int32).pin_memory()
    ptrs = [(h_rem[k].data_ptr(), h_dom[k].data_ptr(), h_pr[k].data_ptr(), h_st[k].data_ptr())
            for k in range(e2e_steps)]   # raw pinned addresses: no per-call tensor marshalling
    for k in range(5):
        work.propagate_from_async(tab.root, *ptrs[k])
    work.synchronize()
    h_st.fill_(-1)
    barrier(world)
    t1 = time.perf_counter()
    for k in range(e2e_steps):
        work.propagate_from_async(tab.root, *ptrs[k])
    t_enq = time.perf_counter() - t1
    work.synchronize()
    n_ok = int((h_st >= 0).sum())
    t2 = time.perf_counter()
    if n_ok != e2e_steps:
        raise RuntimeError(f"e2e: {e2e_steps - n_ok} calls left no status")
    e2e_s = max_over_ranks(t2 - t1, world)
    return {"value": e2e_steps / e2e_s, "unit": "propagations/s", "h2d_bytes_per_step": 8 * wd,
            "d2h_bytes_per_step": 4 + 16 * wd, "steps": e2e_steps,
            "api": "ct_propagate_from_async(work, root) on pinned host buffers (removal DMA'd in, status/"
                   "domains/pruned written to host memory by the kernel), calls pipelined, every status checked "
                   "on the host",
            "host_enqueue_us_per_step": t_enq / e2e_steps * 1e6,
            "sync_call": {"value": e2e_steps / e2e_sync_s, "unit": "propagations/s",
                          "api": "ct_propagate (host buffers, pinned staging, CUDA graph, waits per call)",
                          "d2h_bytes_per_step": 8 * (1 + 2 * wd)}}


def sharded_overhead(m, args, dev):
    """N = 1: the same C3 bulk steps through the SHARDED code paths vs the
    unsharded single launch, and the Amdahl projection to 8 GPUs (SURVEY §8(e):
    the update streams 1/G of the table, the rest is taken as fixed).
      nccl: a 1-rank NCCL communicator -- k_fast without finalize,
            ncclAllReduce of the R+1 flags, k_finalize (three stream operations);
      peer: the in-kernel NVLink combine (ct_peer_attach) with one rank: the
            k_fast finalizer stores its flags into the inbox, releases, acquires
            and ORs them (one kernel; with G ranks the same code stores to G
            inboxes over NVLink)."""
    import torch
    from paper_2507_18413_b200 import Table
    from paper_2507_18413_b200 import ct as C
    p, wd = m["p"], m["tab"].Wd
    rem_dev = torch.from_numpy(m["rem_host"].view(np.int64)).to(f"cuda:{dev}")
    od = torch.zeros(wd, dtype=torch.int64, device=f"cuda:{dev}")
    sd = torch.zeros(1, dtype=torch.int32, device=f"cuda:{dev}")
    P = len(m["rem_host"])

    def measure(peer):
        tab = Table(p.lo, p.d, p.tuples, device=dev, n_shards=1, shard_rank=0,
                    nccl_unique_id=None if peer else C.ct_nccl_unique_id())
        if peer:
            C.ct_peer_attach(tab.handle, [C.ct_peer_export(tab.handle)])
        w = tab.root.clone()
        stream = torch.cuda.ExternalStream(tab.stream_ptr, device=f"cuda:{dev}")

        def run(n):
            for k in range(n):
                w.propagate_from_async(tab.root, rem_dev[k % P], od, None, sd)

        run(args.warmup)
        w.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        run(args.steps)
        ev1.record(stream)
        ev1.synchronize()
        t_sh = ev0.elapsed_time(ev1) / args.steps * 1e3               # us per step
        C.ct_table_profile(tab.handle, True)
        C.ct_table_profile_read(tab.handle, reset=True)
        run(args.steps)
        prof = C.ct_table_profile_read(tab.handle, reset=True)
        tab.close()
        return t_sh, {k: (v[1] / v[0] * 1e3 if v[0] else None) for k, v in prof.items() if v[0]}

    t_nccl, k_nccl = measure(False)
    t_peer, k_peer = measure(True)
    t1 = m["ms_per_step"] * 1e3
    ph = m["phase_ns"]                                             # k_fast: ingest, update(+barrier), ...
    t_upd = ph[1] / 1e3 if ph and ph[1] > 0 else None

    def proj(t_sh):
        if not t_upd:
            return {}
        fixed = t1 - t_upd
        return {str(g): t1 / (t_upd / g + fixed + max(0.0, t_sh - t1)) for g in (2, 4, 8)}

    return {"unsharded_us_per_step": t1, "sharded_path_us_per_step": t_nccl, "overhead_us": t_nccl - t1,
            "kernels_us_per_launch": k_nccl, "update_phase_us": t_upd,
            "amdahl_projected_speedup": proj(t_nccl),
            "peer": {"sharded_path_us_per_step": t_peer, "overhead_us": t_peer - t1,
                     "kernels_us_per_launch": k_peer, "amdahl_projected_speedup": proj(t_peer),
                     "api": "ct_peer_export / ct_peer_attach (1 rank: the table's own inbox)"},
            "note": "1 GPU: the cost a sharded call adds (nccl: 1-rank communicator; peer: in-kernel NVLink "
                    "combine with one rank); projection = T1 / (T_update/G + (T1 - T_update) + overhead), "
                    "not a measurement"}


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    wl = WORKLOADS[args.workload]
    m = measure_c3(args.workload, args, dev, world, rank, full=True, use_gather=not args.no_gather)
    p, root_m, pats = m["p"], m["root_m"], m["pats"]
    latency = filt = shov = None
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        cpu = cpu_baseline(p, root_m, pats, budget_s=args.cpu_budget, what=args.workload)
    m["tab"].close()
    if world == 1 and not args.skip_latency and args.workload == "c3bulk":
        latency = c2_latency(dev, serve=True)
        latency["launched"] = c2_latency(dev, serve=False)
    if args.workload == "c3bulk" and not args.skip_filter:
        # the filter-heavy C3b line, so the filterDomains roofline is in every default run
        f = measure_c3("c3b", args, dev, world, rank, full=False)
        filt = {"workload": "c3b", "table": WORKLOADS["c3b"]["table"], "step": WORKLOADS["c3b"]["step"],
                "value": f["value"], "unit": "propagations/s", "ms_per_step": f["ms_per_step"],
                "roofline": f["roofline"], "kernel_share_of_step": f["kernel_share"],
                "kernel_ms_per_launch": f["kernel_ms"], "workload_counters": f["per_pat"][0],
                "phase_ns": f["phase_ns"], "clocks": f["clocks"]}
        f["tab"].close()
        # the same calls with Alg. 3's full support-row scans (use_gather = 0):
        # the HBM-bound filterDomains the paper's kernels run
        f = measure_c3("c3b", args, dev, world, rank, full=False, use_gather=False)
        filt["alg3_scan"] = {"value": f["value"], "unit": "propagations/s", "ms_per_step": f["ms_per_step"],
                             "roofline": f["roofline"], "kernel_share_of_step": f["kernel_share"],
                             "workload_counters": f["per_pat"][0]}
        f["tab"].close()
    if world == 1 and args.workload == "c3bulk" and not args.skip_sharded:
        shov = sharded_overhead(m, args, dev)
    if rank == 0:
        line = {
            "metric": wl["metric"],
            "value": m["value"], "unit": "propagations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": m["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded " + ("i.i.d." if C3_FAMILY[args.workload][2] else "banded") + " table, workloads/)",
            "config": {"workload": args.workload, "table": wl["table"],
                       "step": wl["step"],
                       "patterns": 16, "parallelism": f"tuple-range shards x{world}, {m['combine']} flag combine" if world > 1 else "1 GPU",
                       "l2": ("inputs larger than L2 (1.0 GB supports streamed each step)"
                              if C3_FAMILY[args.workload][1] >= 10_000_000 else
                              "100 MB of supports: partly L2-resident across back-to-back calls -- the "
                              "CUDA-event GB/s is L2-assisted; the HBM fraction is the ncu capture's "
                              "(caches flushed between replays, profiles/)"),
                       "build_s": round(m["build_s"], 3)},
            "roofline": m["roofline"],
            "kernel_ms_per_launch": m["kernel_ms"],
            "kernel_share_of_step": m["kernel_share"],
            "e2e": m["e2e"], "gpu_launches": m["launches"], "clocks": m["clocks"], "latency": latency,
            "filter": filt, "sharded_overhead": shov,
            "cpu_baseline": cpu, "workload_counters": m["per_pat"][0],
        }
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def c2_latency(dev, serve=False):
    """p50/p90/p99 of the C call ct_propagate (sync, host buffers) on config 2:
    1000 calls of policy P(2, 0.5) after 100 warm-up calls.  The timer brackets
    only the foreign call (arguments pre-marshalled), so the number is the
    library's latency, not Python's.  device_us = the kernel's own duration
    (%globaltimer phase stamps) for the same calls.  serve=False: one CUDA-graph
    launch per call; serve=True: the state's calls are served by a persistent
    kernel polling a doorbell in mapped host memory (ct_state_serve; the
    restores after FAIL / solved stop it, so the next call restarts it)."""
    import ctypes
    from paper_2507_18413_b200 import CT_OK, Table
    from paper_2507_18413_b200 import ct as C
    from workloads import Rng, member_to_bitmap, bitmap_to_member
    from workloads.policies import walk_removal
    p = c2_problem()
    tab = Table(p.lo, p.d, p.tuples, device=dev)
    root_m = bitmap_to_member(tab.root_dom, p.d)
    st = tab.root.clone()
    if serve:
        st.serve(True)
    wd = tab.Wd
    rem = np.zeros(wd, np.uint64)
    out = np.zeros(wd, np.uint64)
    pr = np.zeros(wd, np.uint64)
    fn = C.lib().ct_propagate
    args = (st.handle, rem.ctypes.data_as(ctypes.c_void_p), out.ctypes.data_as(ctypes.c_void_p),
            pr.ctypes.data_as(ctypes.c_void_p))
    rng = Rng(2, lanes=1)
    cur = root_m.copy()
    lat, dev_us = [], []
    fails = solved = 0
    for k in range(1100):
        r = walk_removal(rng, cur, p.d)
        if r is None:
            st.copy_from(tab.root)
            cur = root_m.copy()
            solved += 1
            continue
        rem[:] = member_to_bitmap(r, p.d)
        t0 = time.perf_counter_ns()
        s = fn(*args)
        t1 = time.perf_counter_ns()
        if s < 0:
            raise RuntimeError(C.ct_last_error())
        if k >= 100:
            lat.append((t1 - t0) / 1e3)
            dev_us.append(sum(st.stats().phase_ns) / 1e3)
        if s == CT_OK:
            cur = bitmap_to_member(out, p.d)
        else:
            fails += 1
            st.copy_from(tab.root)
            cur = root_m.copy()
    tab.close()
    q = lambda xs, f: sorted(xs)[min(len(xs) - 1, int(f * len(xs)))]
    return {"config": "C2 arity 5, domain 20, 1e5 tuples; policy P(2,0.5)", "calls": len(lat),
            "p50_us": q(lat, 0.5), "p90_us": q(lat, 0.9), "p99_us": q(lat, 0.99),
            "device_p50_us": q(dev_us, 0.5), "fails": fails, "restores_solved": solved,
            "api": ("ct_propagate on a served state (ct_state_serve: persistent single-CTA kernel, doorbell and "
                    "zero-copy I/O in mapped host memory)" if serve else
                    "ct_propagate (host buffers; single-CTA kernel in a CUDA graph; zero-copy I/O)")}


def _time_oracle(p, root_m, pats, budget_s, threads):
    import oracle
    n = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < budget_s or n == 0:
        oracle.gac(p.lo, p.d, p.tuples, root_m & (1 - pats[n % len(pats)]), threads=threads)
        n += 1
    return n, time.perf_counter() - t0


def cpu_baseline(p, root_m, pats, budget_s=12.0, what="c3bulk"):
    """The oracle (oracle/ct_oracle.c, brute-force tuple scan) on the same calls,
    on every host core this process may use (oracle_gac_split) and on one core."""
    import oracle
    oracle.lib()
    cores = oracle.host_threads()
    n1, dt1 = _time_oracle(p, root_m, pats, budget_s / 3, 1)
    n, dt = _time_oracle(p, root_m, pats, budget_s * 2 / 3, cores)
    name = "C3 bulk" if what.startswith("c3bulk") else "C3b banded"
    return {"value": n / dt, "unit": "propagations/s", "cores": cores, "kind": "oracle",
            "sample": f"{n} full {name} propagations (oracle_gac_split: brute-force scan of all {p.t:.0e} tuples "
                      f"split over {cores} threads) in {dt:.1f} s",
            "single_core": {"value": n1 / dt1, "unit": "propagations/s", "cores": 1,
                            "sample": f"{n1} calls (oracle_gac, one thread) in {dt1:.1f} s"},
            "host_nproc": os.cpu_count()}


# ---------------------------------------------------------------- C4: batched independent states
def c4_patterns(p, S, count, seed=6):
    """State-independent seeded removals [count][S][Wd] (workloads.policies.batch_coin_removals):
    per state, 2 random variables, each value removed with probability 1/2.
    Values already absent are ignored by the library (include/ct.h), so the same
    pattern applies to any state; states walk down until FAIL and are restarted
    on the device (ct_batch_restore_dead)."""
    from workloads.policies import batch_coin_removals
    return batch_coin_removals(p.n, p.d, S, count, seed=seed)


def run_c4(args):
    import torch
    from paper_2507_18413_b200 import Table
    from paper_2507_18413_b200 import ct as C
    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    p = c4_problem()
    S = args.states // world + (1 if rank < args.states % world else 0)      # states split over ranks
    tab = Table(p.lo, p.d, p.tuples, device=dev)
    b = tab.batch(S)
    K = 16
    pats = c4_patterns(p, S, K, seed=6 + 1000 * rank)
    rem_dev = [torch.from_numpy(x.view(np.int64)).to(f"cuda:{dev}") for x in pats]
    out_dom = torch.zeros((S, tab.Wd), dtype=torch.int64, device=f"cuda:{dev}")
    status = torch.zeros(S, dtype=torch.int32, device=f"cuda:{dev}")
    stream = torch.cuda.ExternalStream(tab.stream_ptr, device=f"cuda:{dev}")

    def step(k):
        b.propagate_async(rem_dev[k % K], out_dom, status)
        b.restore_dead(tab.root)

    for k in range(args.warmup):
        step(k)
    tab.root.synchronize()
    b.work(reset=True)
    clocks = Clocks(dev)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for k in range(args.steps):
        step(k)
    ev1.record(stream)
    ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    work = b.work(reset=True)                     # summed over the timed steps (device counters)
    barrier(world)
    ms_max = max_over_ranks(ms, world)
    total_states = args.states
    value = total_states * args.steps / (ms_max / 1e3)
    # per-kernel device times: a second pass of the same number of steps with
    # CUDA events around every kernel (kept out of the timed region above)
    C.ct_table_profile(tab.handle, True)
    C.ct_table_profile_read(tab.handle, reset=True)
    for k in range(args.steps):
        step(k)
    prof = C.ct_table_profile_read(tab.handle, reset=True)
    C.ct_table_profile(tab.handle, False)
    b.work(reset=True)
    # e2e through the synchronous host-buffer call
    e2e_steps = max(5, min(args.steps, 20))
    host = [x.copy() for x in pats]
    outh = np.zeros((S, tab.Wd), np.uint64)
    sth = np.zeros(S, np.int32)
    barrier(world)
    t1 = time.perf_counter()
    for k in range(e2e_steps):
        C.ct_propagate_many(b.handle, host[k % K], outh, sth)
        b.restore_dead(tab.root)
    tab.root.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t1, world)
    kernel_ms = {k: (v[1] / v[0] if v[0] else None) for k, v in prof.items()}
    upd_n, upd_ms = prof["update"]
    launches = sum(v[0] for v in prof.values())
    if tab.info.batch_tile:
        # k_bcompact (and k_bsparse) share the update slot, k_bscan runs 2 passes per slot
        launches += upd_n * (2 if tab.info.batch_cells else 1) + prof["scan"][0]
    roofline = None
    if tab.info.batch_tile and upd_n:
        # dominant kernel: the tile-major update (k_bupdate + k_bcompact, one event pair).
        # HBM bytes it must move: every currTable block of every updating state read,
        # rewritten blocks written, the support tiles staged into shared memory, the
        # survivor bitmap written and read back by the compaction (index writes not counted).
        steps = args.steps
        hbm = (16 * (work["table_blocks_read"] + work["table_blocks_written"]) + work["support_bytes_staged"]
               + 2 * work["table_blocks_read"] // 8) / steps
        # SURVEY §8(d) B_upd's HBM part for a batch step: currTable read + write of
        # every updating state's ACTIVE input blocks (supports come from L2 / shared memory)
        alg = 32 * work.get("update_active_blocks_in", 0) / steps
        smem = 8 * work["update_support_words"] / steps
        t = upd_ms / upd_n / 1e3
        peak, peak_src = peaks()
        smem_peak = 148 * 128 * 1.965          # GB/s: SMs x 128 B/cycle (B300_MICROARCH.md LDS table) x max SM clock
        roofline = {"bound": "hbm", "achieved": hbm / t / 1e9, "peak": peak, "unit": "GB/s",
                    "frac": hbm / t / 1e9 / peak,
                    "traffic": ncu_traffic("c4", world, f"ctk::k_bupdate<{tab.info.batch_tile}>"),
                    "traffic_kernel": f"ctk::k_bupdate<{tab.info.batch_tile}> only (ncu)",
                    "kernel": f"ctk::k_bupdate<{tab.info.batch_tile}> + ctk::k_bcompact",
                    "bytes_per_launch": hbm, "ms_per_launch": t * 1e3, "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": alg, "algorithmic_frac": alg / t / 1e9 / peak,
                    "bytes_note": "achieved = the bytes the kernels move (every block of a dense state read, "
                                  "rewritten blocks, support tiles staged); algorithmic = SURVEY B_upd's HBM "
                                  "part, 32 bytes per active input block of an updating state",
                    "smem": {"achieved": smem / t / 1e9, "peak": smem_peak, "frac": smem / t / 1e9 / smem_peak,
                             "bytes_per_launch": smem,
                             "note": "support words OR-ed by Alg. 2, served from the shared-memory tile "
                                     "(SURVEY B_upd support term); the kernel is bound by shared-memory "
                                     "loads + issue, not by HBM"}}
    tab.close()
    if rank == 0:
        line = {
            "metric": "state-propagations/s (C4 batched ct_propagate_many, 4096 states, 1e6-tuple table)",
            "value": value, "unit": "state-propagations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded i.i.d. table, workloads/)",
            "config": {"workload": "c4", "table": "arity 6, domain 50, 1e6 tuples, seed 5", "states": total_states,
                       "states_per_rank": S, "step": "ct_propagate_many_async (2 random vars, each value removed "
                       "w.p. 1/2, per state) + ct_batch_restore_dead(root)",
                       "parallelism": f"states split over {world} GPUs, no communication",
                       "l2": "per-state currTables 512 MB > L2; supports 37.5 MB L2-resident by design"},
            "kernel_ms_per_launch": kernel_ms, "update_ms_per_launch": upd_ms / max(upd_n, 1),
            "roofline": roofline, "work_per_step": {k: v / args.steps for k, v in work.items() if k.startswith(("update", "table", "support"))},
            "e2e": {"value": total_states * e2e_steps / e2e_s, "unit": "state-propagations/s",
                    "h2d_bytes_per_step": 8 * tab.Wd * total_states,
                    "d2h_bytes_per_step": (8 * tab.Wd + 4) * total_states, "steps": e2e_steps,
                    "api": "ct_propagate_many (host buffers)"},
            "gpu_launches": launches, "clocks": clk,
        }
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ---------------------------------------------------------------- C5: DFS over a 12-table model
def run_c5(args):
    """BASELINE config 5: DFS (input_order, indomain_max, binary branching) on a
    30-var CSP of 12 tables x 1e6 tuples (arity 4-8, planted solution), every
    node propagated to the common fixpoint on the device; the whole search runs
    in one cooperative kernel (device-resident DFS; the host-driven driver's
    rate on the same tree is reported beside it).  value = DFS nodes/s over the
    first --max-nodes nodes (all
    solutions mode, so the search does not stop at the planted one).  Replicas
    only: a search is sequential; N > 1 runs N independent searches."""
    import torch
    from paper_2507_18413_b200 import Model
    from workloads.csp import csp_model
    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    m = csp_model(30, 40, 12, 1_000_000, seed=7)
    t0 = time.perf_counter()
    M = Model(m["vlo"], m["vd"], m["scopes"], m["tables"], device=dev)
    build_s = time.perf_counter() - t0
    M.search(value_order=0, max_nodes=200, max_solutions=0)           # warm-up
    barrier(world)
    clocks = Clocks(dev)
    clocks.start()
    t1 = time.perf_counter()
    st, sol, stats = M.search(value_order=0, max_nodes=args.max_nodes, max_solutions=0, driver="device")
    wall = time.perf_counter() - t1
    clk = clocks.stop()
    wall_max = max_over_ranks(wall, world)
    from paper_2507_18413_b200 import ct as C
    phases = {k: v / 1e3 / max(stats.nodes, 1) for k, v in C.ct_model_search_phases(M.handle).items()}
    # the host-driven driver on the same tree (one fixpoint launch per node), for context
    t3 = time.perf_counter()
    hst = M.search(value_order=0, max_nodes=args.max_nodes, max_solutions=0, driver="host")[2]
    wall_h = time.perf_counter() - t3
    assert (hst.nodes, hst.trace_hash) == (stats.nodes, stats.trace_hash)
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        import oracle
        from oracle.dfs import dfs as oracle_dfs
        cores = oracle.host_threads()
        n_or = 60
        t2 = time.perf_counter()
        ref = oracle_dfs(m["vlo"], m["vd"], m["scopes"], m["tables"], value_order=0, max_nodes=n_or, max_solutions=0,
                         threads=cores)
        dt = time.perf_counter() - t2
        cpu = {"value": ref["nodes"] / dt, "unit": "nodes/s", "cores": cores, "kind": "oracle",
               "sample": f"first {ref['nodes']} DFS nodes by oracle/dfs.py + oracle_fixpoint_split (C brute force, "
                         f"tuple scans over {cores} threads), {dt:.1f} s"}
        chk = M.search(value_order=0, max_nodes=n_or, max_solutions=0)[2]
        cpu["trace_matches_gpu"] = (chk.nodes, chk.trace_hash) == (ref["nodes"], ref["trace_hash"])
    wg = M.Wg
    M.close()
    if rank == 0:
        line = {
            "metric": "DFS nodes/s (C5, 12 tables x 1e6 tuples, fixpoint on device per node)",
            "gpu_launches": 1,
            "value": world * stats.nodes / wall_max, "unit": "nodes/s", "n_gpus": world, "steps": int(stats.nodes),
            "warmup": 200, "ms_per_step": wall_max / max(stats.nodes, 1) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded CSP, planted solution, workloads/csp.py)",
            "config": {"workload": "c5", "model": "30 vars d=40, 12 tables x 1e6 tuples, arity 4+(k mod 5), seed 7",
                       "search": "input_order, indomain_max, binary branching, all solutions, node budget",
                       "parallelism": "replicas" if world > 1 else "1 GPU", "build_s": round(build_s, 2)},
            "search": {"nodes": stats.nodes, "failures": stats.failures, "solutions": stats.solutions,
                       "table_calls": stats.table_calls, "jacobi_iterations": stats.iterations,
                       "max_depth": stats.max_depth, "device_ms": stats.device_ms,
                       "device_us_per_node": stats.device_ms * 1e3 / max(stats.nodes, 1),
                       "device_us_per_node_by_phase": phases,
                       "trace_hash": hex(stats.trace_hash),
                       "driver": "device-resident (k_model_search: one cooperative launch for the whole search)",
                       "host_driver_nodes_per_s": hst.nodes / wall_h},
            "e2e": {"value": stats.nodes / wall, "unit": "nodes/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0,
                    "note": "ct_model_search is the end-to-end call (host in: the model already built; out: "
                            "stats + last solution once); the search itself never leaves the GPU"},
            "clocks": clk, "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ---------------------------------------------------------------- f3: placement ablation
def record_walk(tab, p, n_calls, seed=2):
    """A policy-P(2, 0.5) walk driven by the device-resident library (synchronous
    host calls): [(restore_before, removal bitmap, status, out_dom)]."""
    from paper_2507_18413_b200 import CT_OK
    from workloads import Rng, member_to_bitmap, bitmap_to_member
    from workloads.policies import walk_removal
    root_m = bitmap_to_member(tab.root_dom, p.d)
    st = tab.root.clone()
    rng = Rng(seed, lanes=1)
    cur, restore, seq = root_m.copy(), False, []
    while len(seq) < n_calls:
        r = walk_removal(rng, cur, p.d)
        if r is None:
            cur, restore = root_m.copy(), True
            continue
        if restore:
            st.copy_from(tab.root)
        rem = member_to_bitmap(r, p.d)
        status, dom, _ = st.propagate(rem)
        seq.append((restore, rem, status, None if dom is None else dom.copy()))
        restore = status != CT_OK
        cur = bitmap_to_member(dom, p.d) if status == CT_OK else root_m.copy()
    st.close()
    return seq


def run_placement(args):
    """SURVEY §8(f) f3 / PAPER.md L320-330, L432-436, L558-561: the same recorded
    P(2, 0.5) walk replayed through the paper's serial CT (host), CT^u (device
    update), CT^f (device filter), CT^uf (both, the paper's per-call currTable /
    mask / removal-bitmap transfers) and this library's device-resident call,
    on C2 and on the LIN_B-shaped knapsack table.  Per placement: calls/s and
    the per-call split into host work, H2D, kernels and D2H (CUDA events), and
    the bytes moved.  Every replayed call's status and domains are checked
    against the recording.  1 GPU (replicas only at N > 1)."""
    import torch
    from paper_2507_18413_b200 import HostTable, Table, CT_OK
    from paper_2507_18413_b200 import ct as C
    from workloads import knapsack_table, LIN_PRESETS
    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    n_calls = max(50, args.steps)
    probs = {"c2": c2_problem(), "lin_b": knapsack_table(seed=21, **LIN_PRESETS["lin_b"])}
    out = {}
    clocks = Clocks(dev)
    clocks.start()
    for name, p in probs.items():
        tab = Table(p.lo, p.d, p.tuples, device=dev)
        seq = record_walk(tab, p, args.warmup + n_calls)
        res = {}
        # device-resident (this library): ct_propagate on host buffers; "served":
        # the same calls answered by a persistent kernel (ct_state_serve) where
        # the table's launch shape allows it (single CTA)
        for key in ("resident", "served"):
            st = tab.root.clone()
            if key == "served":
                if tab.info.kernel_path != 3:
                    st.close()
                    res[key] = {"skipped": f"launch shape {C.KERNEL_PATHS[tab.info.kernel_path]} is not servable"}
                    continue
                st.serve(True)
            od, pr = np.zeros(tab.Wd, np.uint64), np.zeros(tab.Wd, np.uint64)
            for k, (restore, rem, _, _) in enumerate(seq[:args.warmup]):
                if restore:
                    st.copy_from(tab.root)
                st.propagate(rem, od, pr)
            t0 = time.perf_counter()
            for k, (restore, rem, status, dom) in enumerate(seq[args.warmup:]):
                if restore:
                    st.copy_from(tab.root)
                s_, d_, _ = st.propagate(rem, od, pr)
            dt = time.perf_counter() - t0
            res[key] = {"calls_per_s": n_calls / dt, "us_per_call": dt / n_calls * 1e6,
                        "h2d_bytes_per_call": 8 * tab.Wd, "d2h_bytes_per_call": 8 * (1 + 2 * tab.Wd),
                        "what": ("ct_propagate on a served state: persistent single-CTA kernel, doorbell + zero-copy "
                                 "I/O in mapped host memory (restores stop the server; the next call relaunches it)"
                                 if key == "served" else
                                 "ct_propagate: state resident in HBM, removal in / status + domains out "
                                 "(mapped pinned memory, one CUDA graph)")}
            st.close()
        tab.close()
        for place in ("host", "u", "f", "uf"):
            ht = HostTable(p.lo, p.d, p.tuples, placement=place, device=dev)
            hs = ht.root.clone()
            od = np.zeros(ht.Wd, np.uint64)
            for restore, rem, _, _ in seq[:args.warmup]:
                if restore:
                    hs.copy_from(ht.root)
                hs.propagate(rem, od)
            ht.stats(reset=True)
            mism = 0
            t0 = time.perf_counter()
            for restore, rem, status, dom in seq[args.warmup:]:
                if restore:
                    hs.copy_from(ht.root)
                s_, d_, _ = hs.propagate(rem, od)
                if s_ != status or (s_ == CT_OK and not np.array_equal(d_, dom)):
                    mism += 1
            dt = time.perf_counter() - t0
            stt = ht.stats(reset=True)
            c = max(stt["calls"], 1)
            res[place] = {"calls_per_s": n_calls / dt, "us_per_call": dt / n_calls * 1e6,
                          "host_us_per_call": stt["host_ms"] / c * 1e3, "h2d_us_per_call": stt["h2d_ms"] / c * 1e3,
                          "kernel_us_per_call": stt["kernel_ms"] / c * 1e3, "d2h_us_per_call": stt["d2h_ms"] / c * 1e3,
                          "h2d_bytes_per_call": stt["h2d_bytes"] / c, "d2h_bytes_per_call": stt["d2h_bytes"] / c,
                          "kernel_launches": stt["kernel_launches"], "mismatches_vs_resident": mism}
            if stt["kernel_ms"] > 0:
                res[place]["copy_share_of_kernel"] = {"h2d": stt["h2d_ms"] / stt["kernel_ms"],
                                                      "d2h": stt["d2h_ms"] / stt["kernel_ms"]}
            ht.close()
        out[name] = {"table": f"n={p.n}, t={p.t}, R={p.R}", "calls": n_calls, "placements": res,
                     "speedup_vs_serial_ct": {k: res[k]["calls_per_s"] / res["host"]["calls_per_s"] for k in res
                                              if "calls_per_s" in res[k]}}
    clk = clocks.stop()
    if rank == 0:
        v = out["c2"]["placements"]["resident"]["calls_per_s"]
        line = {"metric": "propagations/s per CT placement (serial CT, CT^u, CT^f, CT^uf, device-resident)",
                "value": v, "unit": "propagations/s", "n_gpus": world, "steps": n_calls, "warmup": args.warmup,
                "ms_per_step": 1e3 / v, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "u64", "data": "synthetic (C2 i.i.d. table; LIN_B-shaped knapsack table), recorded P(2,0.5) walks",
                "config": {"workload": "placement", "value_is": "C2, device-resident ct_propagate (host buffers)",
                           "parallelism": "1 GPU" if world == 1 else f"{world} replicas"},
                "placement": out, "e2e": {"value": v, "unit": "propagations/s", "h2d_bytes_per_step": 8 * 5,
                                          "d2h_bytes_per_step": 8 * 11},
                "gpu_launches": None, "clocks": clk,
                "paper_context": "PAPER.md L432-436: CT^u can underperform the serial CT (transfers); L558-561: "
                                 "H2D up to 50 %, D2H up to 80 % of kernel time (RTX 4090)"}
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ---------------------------------------------------------------- f4: short and negative tables
def run_f4(args, kind):
    """f4: a C3-shaped short table (arity 8,
    domain 100, 1e7 tuples, 2 % star cells) or a negative table (arity 4,
    domain 60, 1e7 forbidden assignments drawn over the 1.3e7-point product),
    16 seeded bulk removals (half of every variable's values) from the root,
    one restore + ct_propagate_async per step, device-timed; the first pattern
    is checked against the oracle (untimed).  N > 1: independent replicas."""
    import torch
    import oracle
    from paper_2507_18413_b200 import CT_OK, CT_FAIL, Table
    from paper_2507_18413_b200 import ct as C
    from workloads import member_to_bitmap, bitmap_to_member, short_table, negative_table
    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    if kind == "short":
        p = short_table(8, 100, 10_000_000, seed=3, p_star=0.02)
        desc = "short: arity 8, domain 100, 1e7 tuples, 2 % star cells, seed 3"
    else:
        p = negative_table(4, 60, 10_000_000, seed=13)
        desc = "negative: arity 4, domain 60, 1e7 forbidden tuples i.i.d. over the 1.3e7-point product, seed 13"
    t0 = time.perf_counter()
    tab = Table(p.lo, p.d, p.tuples, device=dev, kind=kind)
    build_s = time.perf_counter() - t0
    root_m = bitmap_to_member(tab.root_dom, p.d)
    P = 16
    pats = bulk_patterns(root_m, p.d, P)
    rem_host = np.stack([member_to_bitmap(m, p.d) for m in pats])
    rem_dev = torch.from_numpy(rem_host.view(np.int64)).to(f"cuda:{dev}")
    wd = tab.Wd
    out_dom = torch.zeros(wd, dtype=torch.int64, device=f"cuda:{dev}")
    out_pr = torch.zeros(wd, dtype=torch.int64, device=f"cuda:{dev}")
    status = torch.zeros(1, dtype=torch.int32, device=f"cuda:{dev}")
    work = tab.root.clone()
    stream = torch.cuda.ExternalStream(tab.stream_ptr, device=f"cuda:{dev}")
    torch.cuda.synchronize()   # the tensors above were filled on torch's stream

    def step(k):
        work.propagate_from_async(tab.root, rem_dev[k % P], out_dom, out_pr, status)

    # parity of the first pattern (untimed)
    step(0)
    work.synchronize()
    din = root_m & (1 - pats[0])
    if kind == "short":
        ok, dout, _ = oracle.gac_short(p.lo, p.d, p.tuples, din)
    else:
        ok, dout, _ = oracle.gac_negative(p.lo, p.d, p.tuples, din)
    got = int(status.cpu()[0])
    parity = got == (CT_OK if ok else CT_FAIL) and (not ok or np.array_equal(
        bitmap_to_member(out_dom.cpu().numpy().view(np.uint64), p.d), dout))
    per_pat = []
    for k in range(P):
        step(k)
        s_ = work.stats()
        per_pat.append(dict(L_in=s_.words_in, L_out=s_.words_out, rows=s_.n_update_rows, items=s_.n_filter_items,
                            upd=s_.update_support_words, filt=s_.filter_support_words, writes=s_.update_table_writes,
                            gathered=s_.filter_gathered_tuples))
    for k in range(args.warmup):
        step(k)
    work.synchronize()
    clocks = Clocks(dev)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for k in range(args.steps):
        step(k)
    ev1.record(stream)
    ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    barrier(world)
    ms_max = max_over_ranks(ms, world)
    C.ct_table_profile(tab.handle, True)
    C.ct_table_profile_read(tab.handle, reset=True)
    for k in range(args.steps):
        step(k)
    prof = C.ct_table_profile_read(tab.handle, reset=True)
    C.ct_table_profile(tab.handle, False)
    peak, peak_src = peaks()
    if kind == "short" or C.KERNEL_PATHS.get(tab.info.kernel_path) == "k_fast":
        kname, slot = "ctk::" + C.KERNEL_PATHS.get(tab.info.kernel_path, "k_fast"), "fused"
        if not prof.get("fused", (0, 0))[0]:
            slot = "small"
        b = [8 * c["upd"] + 16 * c["L_in"] + 16 * c["writes"] + 8 * c["filt"] + 32 * c["gathered"] +
             4 * (c["L_in"] + c["L_out"]) for c in per_pat]
        model = ("counted: 8 x support words loaded (update + filter: residue scans / gathered cells for short "
                 "tables, the counting filter's rows for negative ones) + 16 B per index entry read / block "
                 "rewritten + 4 B index entries + 32 B per gathered tuple")
    else:
        kname, slot = "ctk::k_neg_count", "scan"
        b = [8 * c["filt"] + 16 * c["L_out"] for c in per_pat]
        model = ("k_neg_count: 16 B per (count row, active block) + the active currTable blocks once "
                 "(SURVEY §8(d)-style: rows counted x L_out x 16 + 16 L_out)")
    n_l, k_ms = prof.get(slot, (0, 0.0))
    k_ms_pl = k_ms / max(n_l, 1)
    bytes_pl = sum(b[k % P] for k in range(args.steps)) / max(args.steps, 1)
    roofline = {"bound": "hbm", "achieved": bytes_pl / (k_ms_pl / 1e3) / 1e9 if k_ms_pl else None, "peak": peak,
                "unit": "GB/s", "frac": (bytes_pl / (k_ms_pl / 1e3) / 1e9 / peak) if k_ms_pl else None,
                "traffic": ncu_traffic(kind, world, kname), "kernel": kname, "bytes_per_launch": bytes_pl,
                "ms_per_launch": k_ms_pl, "bytes_model": model, "peak_source": peak_src}
    value = args.steps * world / (ms_max / 1e3)
    if rank == 0:
        line = {"metric": f"propagations/s (f4 {kind} table, bulk ct_propagate from the root)", "value": value,
                "unit": "propagations/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded, workloads.%s_table)" % kind,
                "config": {"workload": kind if kind == "short" else "neg", "table": desc,
                           "step": "ct_propagate_from_async(work, root) of a bulk removal (50 % of every var)",
                           "patterns": P, "parallelism": "1 GPU" if world == 1 else f"{world} replicas",
                           "kernel_path": C.KERNEL_PATHS.get(tab.info.kernel_path), "build_s": round(build_s, 3),
                           "l2": "inputs larger than L2"},
                "roofline": roofline,
                "kernel_ms_per_launch": {k: (v[1] / v[0] if v[0] else None) for k, v in prof.items()},
                "parity_first_pattern": bool(parity), "workload_counters": per_pat[0],
                "gpu_launches": sum(v[0] for k, v in prof.items()) + args.steps, "clocks": clk,
                "e2e": None, "cpu_baseline": None}
        print(json.dumps(line))
    tab.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ---------------------------------------------------------------- reference arm (the oracle)
def run_reference(args):
    """The reference arm of this tier: the oracle (oracle/ct_oracle.c) timed as it
    stands on the box's host cores (all of them, oracle_gac_split), rank 0 only,
    on the C3 bulk calls; each step is a bounded sample of the workload."""
    world, rank, local = dist_env()
    if rank != 0:
        return
    import oracle
    from workloads import full_member
    oracle.lib()
    cores = oracle.host_threads()
    p = c3_problem()
    ok, root_m, _ = oracle.gac(p.lo, p.d, p.tuples, full_member(p.d), threads=cores)
    pats = bulk_patterns(root_m, p.d, 16)
    # if K+W full calls would exceed ~120 s, each step runs on a contiguous tuple
    # slice and the rate is scaled by t/slice (the scan is linear in t)
    t0 = time.perf_counter()
    oracle.gac(p.lo, p.d, p.tuples, root_m & (1 - pats[0]), threads=cores)
    est = time.perf_counter() - t0
    frac = min(1.0, 120.0 / max(1e-9, est * (args.steps + args.warmup)))
    ts = max(1, int(p.t * frac))
    tup = p.tuples[:ts]
    for k in range(args.warmup):
        oracle.gac(p.lo, p.d, tup, root_m & (1 - pats[k % 16]), threads=cores)
    t1 = time.perf_counter()
    for k in range(args.steps):
        oracle.gac(p.lo, p.d, tup, root_m & (1 - pats[k % 16]), threads=cores)
    dt = time.perf_counter() - t1
    value = args.steps / (dt * (p.t / ts))
    sample = (f"{args.steps} C3 bulk propagations by the CPU oracle (tuple scan split over {cores} threads) over "
              + ("all 1e7 tuples" if ts == p.t else f"the first {ts} of 1e7 tuples, time scaled by t/{ts} (linear scan)"))
    line = {"impl": "reference", "metric": WORKLOADS["c3bulk"]["metric"],
            "value": value, "unit": "propagations/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3 * (p.t / ts), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded i.i.d. table, workloads/)",
            "config": {"workload": "c3bulk", "table": "arity 8, domain 100, 1e7 tuples, seed 3"},
            "cpu_baseline": {"value": value, "unit": "propagations/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "propagations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def _free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def launch_ranks(n):
    """`bench.py --gpus N` outside a launcher: start N ranks of this same command
    under torch.distributed.run (one process per GPU, 127.0.0.1 rendezvous);
    rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="GPUs (ranks); without a launcher, bench.py starts them itself")
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3bulk",
                    choices=["c3bulk", "c3b", "c3bulk6", "c3b6", "c4", "c5", "lin", "placement", "short", "neg"])
    ap.add_argument("--max-nodes", type=int, default=10_000, help="c5: DFS node budget")
    ap.add_argument("--states", type=int, default=4096, help="c4: total independent states (split over ranks)")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-latency", action="store_true")
    ap.add_argument("--skip-filter", action="store_true", help="default line: no C3b filter sub-object")
    ap.add_argument("--skip-sharded", action="store_true", help="default line: no sharded-path overhead probe")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-gather", action="store_true", help="c3bulk/c3b: Alg. 3 scans only (ct_config.use_gather = 0)")
    ap.add_argument("--combine", default="peer", choices=["peer", "nccl"],
                    help="N > 1 shards: flag combine inside k_fast over NVLink (peer) or an NCCL all-reduce")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" not in os.environ and (args.gpus or 1) > 1:
        sys.exit(launch_ranks(args.gpus))
    if args.gpus is not None and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    args.gpus = world
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "c4":
        run_c4(args)
    elif args.workload == "c5":
        run_c5(args)
    elif args.workload == "lin":
        run_lin(args)
    elif args.workload == "placement":
        run_placement(args)
    elif args.workload in ("short", "neg"):
        run_f4(args, "short" if args.workload == "short" else "negative")
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
