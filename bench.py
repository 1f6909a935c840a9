"""Benchmark: copula fit throughput (points/s, fp64) at n=1e9 per family on
1..8 B200s — BASELINE.json metric, configs[4] (C5) workload.

One step = the full hot path for Gaussian(rho=0.5), Frank(theta=5) and
Gumbel(theta=2), each on its own n=1e9-point sample split into K=8000
contiguous subsets of 125,000: per-subset bit-exact ranks ->
Newton MPL fit -> asymptotic variance -> (N>1: NCCL all-gather of the
per-subset records) -> inverse-variance combine on device.

  value : 3e9 points / device time of one step, inputs resident in HBM
          (max over ranks; CUDA events on the library's stream)
  e2e   : the same metric through the C-ABI (pcb_fit_blocks) with HOST
          (pinned) buffers: H2D of the step's inputs and D2H of the records
          are inside the timed region

--impl reference times the reference CPU path (oracle/_ref: the reference
headers compiled in place + the SPEC restatement of fit/variance/combine) on
all host cores, on a bounded sample of the same workload; rank 0 only.
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

FAMILIES = [("gaussian", 0, 0.5), ("frank", 1, 5.0), ("gumbel", 2, 2.0)]
N_PER_FAMILY = 1_000_000_000
K_SUBSETS = 8000
BASE_SEED = 0x160905530
METRIC = "copula fit throughput (points/sec, fp64) at n=1e9, 1/2/4/8 B200, % roofline"
# SURVEY.md §8(d) frozen algorithmic FP64 instructions per point per theta candidate (F_fit)
PIPE_ROOF_PTS = {"gaussian": 6.8e10, "frank": 1.9e10, "gumbel": 1.4e10}  # SURVEY.md §8(d), per GPU
F_FIT = {"gaussian": 9, "frank": 175, "gumbel": 210}
F_VAR = {"gaussian": 24, "frank": 260, "gumbel": 350}  # per point at theta-hat (variance pass)
B_PASS = 16  # bytes per point per likelihood pass (fp64 pair)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", type=int, default=N_PER_FAMILY, help="points per family (default 1e9)")
    p.add_argument("--subsets", type=int, default=K_SUBSETS)
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg (profiling runs)")
    p.add_argument("--cpu-subsets", type=int, default=48, help="subsets per family in the CPU baseline sample")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ reference arm
def cpu_reference(args, steps, warmup, subsets_per_step):
    """Reference CPU path on a bounded sample: per step, `subsets_per_step`
    subsets of the C5 shape (125,000 points) per family, fitted by
    oracle/_ref (reference headers + SPEC driver) on all host cores."""
    from oracle.oracle import oracle_lib, ref_lib
    orc = oracle_lib()
    lib = ref_lib()
    kind = "reference" if lib is not None else "port"
    lib = lib or orc
    cores = os.cpu_count() or 1
    q = args.n // args.subsets
    data = []
    for name, fam, th in FAMILIES:
        off_full = np.arange(subsets_per_step + 1, dtype=np.uint64) * np.uint64(q)
        # the first subsets_per_step subsets of the same C5 partition (same seeds as the GPU arm)
        offs = np.arange(args.subsets + 1, dtype=np.uint64) * np.uint64(q)
        offs[-1] = args.n
        c1, c2 = orc.sample_blocks(fam, th, args.n, args.subsets, offs, 0, subsets_per_step, base_seed=BASE_SEED)
        data.append((name, fam, c1, c2, off_full))
    pts = sum(len(d[2]) for d in data)

    def one_step():
        for name, fam, c1, c2, off in data:
            recs = lib.fit_blocks(fam, c1, c2, off, workers=cores)
            lib.combine(recs)

    for _ in range(warmup):
        one_step()
    t0 = time.perf_counter()
    for _ in range(steps):
        one_step()
    dt = (time.perf_counter() - t0) / steps
    return pts, dt, kind, cores


def cpu_leg_and_parity(args, cols, gathered, first, last, q, rows, world):
    """cpu_baseline on a bounded sample + parity of the GPU records on it.
    Subsets are spread over this rank's whole range (first, middle, last ...),
    their input columns copied from the device (identical bytes)."""
    from oracle.oracle import oracle_lib, ref_lib
    lib = ref_lib()
    kind = "reference" if lib is not None else "port"
    lib = lib or oracle_lib()
    cores = os.cpu_count() or 1
    kl = last - first
    sub = max(1, min(kl, args.cpu_subsets // 3))
    picks = np.unique(np.linspace(0, kl - 1, sub).round().astype(np.int64))
    tot_pts, tot_s = 0, 0.0
    worst_t, worst_s, worst_c, mism = 0.0, 0.0, 0.0, 0
    per_family = {}
    for name, fam, th in FAMILIES:
        c1d, c2d = cols[name]
        b0 = picks * q
        n_last = rows - (kl - 1) * q
        lens = np.where(picks == kl - 1, n_last, q)
        h1 = np.concatenate([c1d[int(a):int(a + ln)].cpu().numpy() for a, ln in zip(b0, lens)])
        h2 = np.concatenate([c2d[int(a):int(a + ln)].cpu().numpy() for a, ln in zip(b0, lens)])
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
        t0 = time.perf_counter()
        recs = lib.fit_blocks(fam, h1, h2, off, workers=cores)
        tc_cpu, _, _ = lib.combine(recs)
        tot_s += time.perf_counter() - t0
        tot_pts += int(off[-1])
        arr = gathered[name].cpu().numpy().view(np.uint8).reshape(-1, 48)
        g = arr[picks + (first if world > 1 else 0)]
        gth = g[:, 0:8].copy().view(np.float64).ravel()
        gs2 = g[:, 8:16].copy().view(np.float64).ravel()
        gconv = g[:, 36:40].copy().view(np.int32).ravel()
        cth = np.array([r.theta_hat for r in recs])
        cs2 = np.array([r.sigma2 for r in recs])
        cconv = np.array([int(bool(r.converged)) for r in recs])
        mism += int(np.sum(cconv != (gconv != 0)))
        ok = cconv.astype(bool)
        rt = float(np.max(np.abs(gth[ok] - cth[ok]) / np.abs(cth[ok]))) if ok.any() else 0.0
        rs = float(np.max(np.abs(gs2[ok] - cs2[ok]) / np.abs(cs2[ok]))) if ok.any() else 0.0
        # combine of the same subsets' GPU records (fixed block order)
        w = np.where(gconv != 0, 1.0 / gs2, 0.0)
        tc_gpu = float(np.sum(w * np.where(gconv != 0, gth, 0.0)) / np.sum(w))
        rc = abs(tc_gpu - tc_cpu) / abs(tc_cpu)
        worst_t, worst_s, worst_c = max(worst_t, rt), max(worst_s, rs), max(worst_c, rc)
        per_family[name] = {"blocks": int(len(picks)), "max_rel_theta": rt, "max_rel_sigma2": rs,
                            "rel_theta_combined_of_sample": rc}
    tol = 1e-9
    parity = {"blocks_per_family": int(len(picks)), "spread": "evenly over the subset range (first..last)",
              "inputs": "device bytes copied to host", "checker": kind, "max_rel_theta": worst_t,
              "max_rel_sigma2": worst_s, "max_rel_theta_combined_of_sample": worst_c,
              "converged_mismatch": mism, "tol": tol,
              "ok": bool(worst_t <= tol and worst_s <= tol and worst_c <= tol and mism == 0),
              "per_family": per_family}
    cpu = {"value": tot_pts / tot_s, "unit": "points/s", "cores": cores, "kind": kind,
           "sample": f"{len(picks)} subsets x {q} points per family (3 families) spread over the C5 partition, "
                     f"inputs = the GPU arm's device bytes; fit by Newton on the score root (SPEC-literal Brent "
                     f"would be 4-7x slower, SURVEY.md §0)"}
    return cpu, parity


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    sub = max(1, args.cpu_subsets // 3)
    pts, dt, kind, cores = cpu_reference(args, args.steps, args.warmup, sub)
    v = pts / dt
    sample = f"{sub} subsets x {args.n // args.subsets} points per family (3 families) per step, C5 partition, seeds of the GPU arm"
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "points/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C5 (BASELINE configs[4]) bounded CPU sample", "n_per_family": args.n,
                   "subsets": args.subsets, "families": [f"{n}:{t}" for n, _, t in FAMILIES]},
        "cpu_baseline": {"value": v, "unit": "points/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        # the CPU arm times a bounded sample of the workload, not all of it
        "same_config": False,
        "bounded_sample": {"subsets_per_family": sub, "of_subsets": args.subsets, "subset_rows": args.n // args.subsets,
                           "families": len(FAMILIES), "fit_method": "safeguarded Newton on the score root (the SPEC's "
                           "Brent search would be 4-7x slower, SURVEY.md §0)",
                           "projected_full_step_s": (args.n * len(FAMILIES)) / v},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1609_05530_b200 as pcb
    from paper_1609_05530_b200 import _lib as L
    from paper_1609_05530_b200.distributed import gather_records, shard_blocks

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    ctx = pcb.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    K, n = args.subsets, args.n
    q = n // K
    first, last = shard_blocks(K, world, rank)
    row0 = first * q
    row1 = n if last == K else last * q
    rows = row1 - row0
    kl = last - first
    off = (np.arange(kl + 1, dtype=np.uint64) * np.uint64(q))
    off[-1] = rows
    offp = off.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_uint64))

    fp64_peak = ctx.fp64_peak()
    # inputs resident in HBM (generation is not timed)
    cols = {}
    for name, fam, th in FAMILIES:
        c1 = torch.empty(rows, dtype=torch.float64, device="cuda")
        c2 = torch.empty(rows, dtype=torch.float64, device="cuda")
        ctx.check(ctx.lib.pcb_sample(ctx.ptr, fam, th, n, K, first, last, BASE_SEED, c1.data_ptr(), c2.data_ptr()))
        cols[name] = (c1, c2)
    recs = {name: torch.zeros((kl, 6), dtype=torch.int64, device="cuda") for name, _, _ in FAMILIES}
    gathered = {}
    comb = {name: L.CombinedC() for name, _, _ in FAMILIES}
    stage_acc = {name: {} for name, _, _ in FAMILIES}

    def step(accumulate):
        for name, fam, th in FAMILIES:
            c1, c2 = cols[name]
            ctx.check(ctx.lib.pcb_fit_blocks(ctx.ptr, fam, 0, c1.data_ptr(), c2.data_ptr(), rows, offp, kl,
                                             recs[name].data_ptr()))
            if accumulate:
                for k, v in ctx.stage_times().items():
                    stage_acc[name][k] = stage_acc[name].get(k, 0.0) + v
            full = gather_records(recs[name], K) if world > 1 else recs[name]
            gathered[name] = full
            ctx.check(ctx.lib.pcb_combine(ctx.ptr, full.data_ptr(), K, None, __import__("ctypes").byref(comb[name])))

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        step(True)
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = ctx.launch_count() - launches0
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    total_points = n * len(FAMILIES)
    value = total_points / (ms * 1e-3)

    # roofline of the dominant kernel (the Newton likelihood pass, k_lik)
    res = {}
    for name, fam, th in FAMILIES:
        arr = gathered[name].cpu().numpy().view(np.uint8).reshape(K, 48)
        iters = arr[:, 32:36].copy().view(np.int32).ravel()
        conv = arr[:, 36:40].copy().view(np.int32).ravel()
        res[name] = {"theta_combined": comb[name].theta_combined, "blocks_used": int(comb[name].blocks_used),
                     "mean_passes": float(iters.mean()), "converged": int(conv.sum())}
    kernels = {}
    for name, fam, th in FAMILIES:
        sa = stage_acc[name]
        steps = args.steps
        kms = sa.get("lik_kernel_ms", 0.0) / steps
        nl = sa.get("lik_launches", 0.0) / steps
        wl = sa.get("warm_launches", 0.0) / steps
        passes = res[name]["mean_passes"] - wl  # fp64 passes per subset (iterations include fp32 warm-up)
        entry = {"stage_ms": {k: v / steps for k, v in sa.items()}}
        if kms > 0:
            instr = F_FIT[name] * rows * passes  # algorithmic FP64 instructions (frozen F_fit) per step
            entry["lik"] = {"ms": kms, "launches": nl, "avg_launch_ms": kms / max(nl, 1), "fp64_passes": passes,
                            "fp64_instr_per_s": instr / (kms * 1e-3),
                            "hbm_gbs": B_PASS * rows * passes / (kms * 1e-3) / 1e9}
        if wl > 0:
            wms = sa.get("warm_kernel_ms", 0.0) / steps
            entry["warm_fp32"] = {"ms": wms, "launches": wl, "hbm_gbs": 8 * rows * wl / (wms * 1e-3) / 1e9}
        kernels[name] = entry
    # ---- roofline: every kernel's share of the step, the dominant one reported
    # (algorithmic bytes / FP64 instructions per launch)
    hbm_peak = 6547.2e9  # MEASURED_PEAKS.json hbm_gbs (burst copy)
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) * 1e9
    except Exception:
        pass
    traffic_db = {}
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic_db = json.load(open(tp))
        except Exception:
            traffic_db = {}
    # L2: sectors per point per kernel and family (ncu, profiles/l2_sectors.json) against the
    # measured random-sector L2 rate (tools/l2_probe.cu, profiles/l2_probe.json): the bound of the
    # gather kernels (prepare, variance passes), reported beside the HBM roofline
    l2_db, l2_rate = {}, None
    try:
        l2_db = json.load(open(os.path.join(ROOT, "profiles", "l2_sectors.json")))
        l2_rate = float(json.load(open(os.path.join(ROOT, "profiles", "l2_probe.json")))["l2_random_sectors_per_s"])
    except Exception:
        l2_db, l2_rate = {}, None
    # measured dynamic FP64 instructions per point (ncu DFMA+DADD+DMUL, profiles/r02_fp64_pipe.json):
    # SURVEY.md §8(d) asks for the fraction by both the frozen F and the measured count
    fp64_db = {}
    try:
        fp64_db = json.load(open(os.path.join(ROOT, "profiles", "r02_fp64_pipe.json")))["kernels"]
    except Exception:
        fp64_db = {}
    # instruction issue: the rank kernel is issue / shared-memory bound, not HBM bound:
    # measured warp instructions per point (profiles/issue.json) x points / live ms against the
    # issue peak (SMs x 4 schedulers x the SM clock sampled during the timed region)
    issue_db = {}
    try:
        issue_db = json.load(open(os.path.join(ROOT, "profiles", "issue.json")))
    except Exception:
        issue_db = {}
    sm_hz = float((clk or {}).get("sm_mhz") or 1965.0) * 1e6
    issue_peak = torch.cuda.get_device_properties(local).multi_processor_count * 4 * sm_hz
    l2_sect = {}  # kernel -> sectors per step
    per_kernel = {}  # name -> [ms, launches, bytes, fp64 instr (frozen F), fp64 instr (measured per point)]
    def add(name, ms, launches, nbytes, instr, fam_name, per_launch=False, units=0.0):
        e = per_kernel.setdefault(name, [0.0, 0, 0.0, 0.0, 0.0])
        e[0] += ms
        e[1] += launches
        e[2] += nbytes
        e[3] += instr
        dyn = fp64_db.get(name, {}).get(fam_name, {}).get("fp64_instr_per_point")
        if dyn is not None and units:
            e[4] += dyn * units
        spp = l2_db.get(name, {}).get(fam_name) if isinstance(l2_db.get(name), dict) else None
        if spp is not None and ms > 0:
            l2_sect[name] = l2_sect.get(name, 0.0) + spp * rows * (launches if per_launch else 1)
    for name, fam, th in FAMILIES:
        st_ = kernels[name]["stage_ms"]
        add("k_rank_cluster", st_.get("rank", 0.0), 1, 32.0 * rows, 0.0, name)
        # prepare: read 2 packed ranks; write T (f64 pair) + its fp32 warm-up copy (Archimedean)
        add("k_prepare", st_.get("prepare", 0.0), 1, (16.0 if name == "gaussian" else 40.0) * rows, 0.0, name)
        vp = st_.get("var_point_ms", 0.0)
        # variance pass 1: read ranks + routes (+T for Gumbel); write score + two routed cross values
        add("k_var_point", vp, 1, (64.0 if name == "gumbel" else 48.0) * rows, F_VAR[name] * rows, name,
            units=rows)
        # passes 2-3: scan reads cross + local position, writes W per slot (2 x 18 B);
        # final reads route, score, W_1, W_2 (32 B)
        add("k_var_scan+final", st_.get("variance", 0.0) - vp, 2, 68.0 * rows, 0.0, name)
        if "lik" in kernels[name]:
            lk = kernels[name]["lik"]
            add("k_lik(fp64)", lk["ms"], lk["launches"], B_PASS * rows * lk["fp64_passes"],
                F_FIT[name] * rows * lk["fp64_passes"], name, per_launch=True, units=rows * lk["fp64_passes"])
        if "warm_fp32" in kernels[name]:
            wk = kernels[name]["warm_fp32"]
            add("k_lik(fp32 warm-up)", wk["ms"], wk["launches"], 8.0 * rows * wk["launches"], 0.0, name, per_launch=True)
    table = {}
    for kname, (kms, nl, nbytes, instr, dyn) in per_kernel.items():
        if kms <= 0:
            continue
        t_hbm, t_fp64 = nbytes / hbm_peak, instr / fp64_peak
        bound = "fp64" if t_fp64 > t_hbm else "hbm"
        if bound == "hbm":
            ach, peak, unit = nbytes / (kms * 1e-3) / 1e9, hbm_peak / 1e9, "GB/s"
        else:
            ach, peak, unit = instr / (kms * 1e-3) / 1e12, fp64_peak / 1e12, "T FP64-instr/s"
        table[kname] = {"ms_per_step": kms, "share": kms / ms, "launches": nl, "bound": bound, "achieved": ach,
                        "peak": peak, "unit": unit, "frac": ach / peak, "avg_launch_ms": kms / max(nl, 1)}
        if dyn > 0:
            table[kname]["fp64_measured"] = {
                "instr_per_s": dyn / (kms * 1e-3), "frac": dyn / (kms * 1e-3) / fp64_peak,
                "frac_by_frozen_F": instr / (kms * 1e-3) / fp64_peak,
                "source": "ncu DFMA+DADD+DMUL per point (profiles/r02_fp64_pipe.json) x live ms",
                "pipe_active_pct": {f: v.get("sm__pipe_fp64_cycles_active_pct") for f, v in fp64_db.get(kname, {}).items()}}
        if isinstance(issue_db.get(kname), (int, float)):
            ips = issue_db[kname] * rows * nl / (kms * 1e-3)
            table[kname]["issue"] = {"warp_instr_per_s": ips, "peak_warp_instr_per_s": issue_peak,
                                     "frac": ips / issue_peak,
                                     "source": "profiles/issue.json (ncu smsp__inst_executed per point) x live ms; "
                                               "peak = SMs x 4 schedulers x sampled SM clock"}
        if kname in l2_sect and l2_rate:
            rate = l2_sect[kname] / (kms * 1e-3)
            table[kname]["l2"] = {"sectors_per_s": rate, "peak_random_sectors_per_s": l2_rate,
                                  "frac": rate / l2_rate, "source": "profiles/l2_sectors.json x live ms"}
    dom = max(table, key=lambda k: table[k]["ms_per_step"]) if table else None
    roof = None
    if dom:
        tk = table[dom]
        roof = {"bound": tk["bound"], "kernel": dom, "achieved": tk["achieved"], "peak": tk["peak"], "unit": tk["unit"],
                "frac": tk["frac"], "share_of_step": tk["share"],
                "peak_source": ("MEASURED_PEAKS.json hbm_gbs (measured)" if tk["bound"] == "hbm"
                                else "measured live: DFMA-loop microbenchmark (pcb_measure_fp64_peak)"),
                "traffic": (traffic_db[dom] * rows if dom in traffic_db else None),
                "traffic_unit": "DRAM bytes per launch (ncu --set full, profiles/r02_ncu_full.md, per point x points)",
                "algorithmic_bytes_per_launch": per_kernel[dom][2] / max(per_kernel[dom][1], 1),
                "issue": tk.get("issue"),
                "per_kernel": table}
        # SURVEY.md §8(d) pipeline roofline per GPU (B_pipe = 96 B/pt against HBM; F_pipe with the
        # oracle's mean Newton passes against FP64): the step's floor for the C5 mix
        floor_ms = sum(n / PIPE_ROOF_PTS[name] * 1e3 for name, _, _ in FAMILIES) / world
        roof["pipeline"] = {"floor_ms_per_step": floor_ms, "frac": floor_ms / ms,
                            "pts_per_s_per_gpu": PIPE_ROOF_PTS,
                            "source": "SURVEY.md §8(d): Gaussian HBM 96 B/pt; Frank/Gumbel FP64 F_pipe (P=4/4.2)"}
    # ------------------------------------------------------------ configs[4] end to end, sampling included
    # BASELINE configs[4] defines C5's end-to-end time as sample -> rank -> fit
    # -> combine: the device sampler (copula.hpp:359-410 transforms over
    # counter-based streams) regenerates each family's columns inside the
    # timed region, then the same pipeline runs (CUDA events, max over ranks).
    sample_ms = {}
    for name, fam, th in FAMILIES:
        c1, c2 = cols[name]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(2):
            ctx.check(ctx.lib.pcb_sample(ctx.ptr, fam, th, n, K, first, last, BASE_SEED, c1.data_ptr(), c2.data_ptr()))
        e1.record(stream)
        torch.cuda.synchronize()
        sample_ms[name] = e0.elapsed_time(e1) / 2
    launches_s0 = ctx.launch_count()
    ev0.record(stream)
    for _ in range(args.steps):
        for name, fam, th in FAMILIES:
            c1, c2 = cols[name]
            ctx.check(ctx.lib.pcb_sample(ctx.ptr, fam, th, n, K, first, last, BASE_SEED, c1.data_ptr(), c2.data_ptr()))
        step(False)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms_s = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_s = float(t.item())
    e2e_sampled = {"value": total_points / (ms_s * 1e-3), "unit": "points/s", "ms_per_step": ms_s,
                   "sample_ms": sample_ms, "gpu_launches": int(ctx.launch_count() - launches_s0),
                   "definition": "BASELINE configs[4]: device sample -> rank -> fit -> variance -> "
                                 "(gather) -> combine per family, inputs generated inside the timed region "
                                 "(no host copies; the PCIe-bound host-input number is `e2e`)"}

    # ------------------------------------------------------------ cpu_baseline + parity
    # The reference CPU path (oracle/_ref) fits a spread of this rank's
    # subsets from the SAME device bytes (D2H of their input columns); the
    # GPU records of those subsets must match within 1e-9 (SPEC.md:284-301,
    # north_star), and so must the inverse-variance combine over them.
    cpu, parity = None, None
    if rank == 0 and not args.no_cpu:
        try:
            cpu, parity = cpu_leg_and_parity(args, cols, gathered, first, last, q, rows, world)
        except Exception as ex:  # never fail the GPU line on the baseline leg
            cpu = {"value": None, "unit": "points/s", "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {ex}"}

    # ------------------------------------------------------------ e2e
    e2e = None
    if not args.no_e2e:
        del cols
        torch.cuda.empty_cache()
        host = {}
        for name, fam, th in FAMILIES:
            h1 = torch.empty(rows, dtype=torch.float64, pin_memory=True)
            h2 = torch.empty(rows, dtype=torch.float64, pin_memory=True)
            ctx.check(ctx.lib.pcb_sample(ctx.ptr, fam, th, n, K, first, last, BASE_SEED, h1.data_ptr(), h2.data_ptr()))
            host[name] = (h1, h2)
        hrec = {name: np.zeros((kl, 6), np.int64) for name, _, _ in FAMILIES}

        def e2e_step():
            for name, fam, th in FAMILIES:
                h1, h2 = host[name]
                ctx.check(ctx.lib.pcb_fit_blocks(ctx.ptr, fam, 0, h1.data_ptr(), h2.data_ptr(), rows, offp, kl,
                                                 hrec[name].ctypes.data))
                if world > 1:
                    full = gather_records(torch.from_numpy(hrec[name]).cuda(), K)
                    ctx.check(ctx.lib.pcb_combine(ctx.ptr, full.data_ptr(), K, None,
                                                  __import__("ctypes").byref(comb[name])))
                else:
                    ctx.check(ctx.lib.pcb_combine(ctx.ptr, hrec[name].ctypes.data, K, None,
                                                  __import__("ctypes").byref(comb[name])))

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": total_points / dt, "unit": "points/s", "h2d_bytes_per_step": int(16 * n * len(FAMILIES)),
               "d2h_bytes_per_step": int(48 * K * len(FAMILIES)), "ms_per_step": dt * 1e3,
               "timing": "host wall clock around the synchronous C-ABI calls (max over ranks)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C5 (BASELINE configs[4]): Gaussian rho=0.5 + Frank theta=5 + Gumbel theta=2, "
                                   "n=1e9 fp64 pairs per family, K=8000 subsets of 125000, rank->fit->variance->gather->combine",
                       "n_per_family": n, "subsets": K, "subset_rows": q, "parallelism": f"dp{world} (subset shards)",
                       "l2": "inputs (16 GB per family) exceed the 126 MB L2; no flush needed"},
            "roofline": roof, "cpu_baseline": cpu, "parity": parity, "e2e": e2e, "e2e_sampled": e2e_sampled, "gpu_launches": int(launches),
            "clocks": clk, "kernels": kernels, "results": res,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    ctx.close()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
