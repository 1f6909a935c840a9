"""BASELINE.json configs[3] (C4): the accuracy/throughput sweep.

Gaussian rho in {0.2, 0.5, 0.8}, Frank theta in {2, 5, 10}, Gumbel theta in
{1.5, 2, 3}; n = 1e8 pairs per (family, theta) sampled on device; the
full-data estimate (K = 1: one global rank + fit + variance over all 1e8
rows) and the divide-and-combine estimate for K in {10, 100, 1000, 10000}
with the fp64 and the fp32 likelihood paths. One JSON line per cell:
theta_combined, |theta_combined - theta_full| (the paper's comparison,
PAPER.md:150-162), device time and points/s.

    python sweep.py [--n 100000000] [--out profiles/r01_sweep_c4.jsonl]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GRID = [(0, "gaussian", [0.2, 0.5, 0.8]), (1, "frank", [2.0, 5.0, 10.0]), (2, "gumbel", [1.5, 2.0, 3.0])]
KS = [10, 100, 1000, 10000]
BASE_SEED = 0x160905530


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_sweep_c4.jsonl"))
    args = ap.parse_args()
    import torch

    import paper_1609_05530_b200 as pcb
    from paper_1609_05530_b200 import _lib as L

    ctx = pcb.Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    n = args.n
    lines = []

    def fit(fam, c1, c2, k, prec):
        off = np.zeros(k + 1, np.uint64)
        assert L.load().pcb_partition(n, k, 0, off.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
        rec = torch.zeros((k, 6), dtype=torch.int64, device="cuda")
        comb = L.CombinedC()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        ctx.check(ctx.lib.pcb_fit_blocks(ctx.ptr, fam, prec, c1.data_ptr(), c2.data_ptr(), n,
                                         off.ctypes.data_as(C.POINTER(C.c_uint64)), k, rec.data_ptr()))
        ctx.check(ctx.lib.pcb_combine(ctx.ptr, rec.data_ptr(), k, None, C.byref(comb)))
        e1.record(stream)
        torch.cuda.synchronize()
        return comb, e0.elapsed_time(e1), ctx.stage_times()

    for fam, name, thetas in GRID:
        for th in thetas:
            c1 = torch.empty(n, dtype=torch.float64, device="cuda")
            c2 = torch.empty(n, dtype=torch.float64, device="cuda")
            # one sample per (family, theta): n rows drawn as 1,000 seeded blocks
            ctx.check(ctx.lib.pcb_sample(ctx.ptr, fam, th, n, 1000, 0, 1000, BASE_SEED, c1.data_ptr(), c2.data_ptr()))
            full, ms_full, st_full = fit(fam, c1, c2, 1, 0)
            rec = {"config": "C4", "family": name, "theta_true": th, "n": n, "K": 1, "precision": "fp64",
                   "theta": full.theta_combined, "ms": ms_full, "points_per_s": n / (ms_full * 1e-3),
                   "stage_ms": st_full}
            lines.append(rec)
            print(json.dumps(rec), flush=True)
            for k in KS:
                for prec, pname in ((0, "fp64"), (1, "fp32")):
                    comb, ms, st = fit(fam, c1, c2, k, prec)
                    rec = {"config": "C4", "family": name, "theta_true": th, "n": n, "K": k, "precision": pname,
                           # the Gaussian fit has no per-point likelihood pass (sufficient statistics)
                           "lik_arith": "fp64" if (fam == 0 or prec == 0) else "fp32 (Frank |theta|<2, Gumbel theta<1.1: fp64)",
                           "theta_combined": comb.theta_combined, "blocks_used": int(comb.blocks_used),
                           "theta_full": full.theta_combined,
                           "abs_err_vs_full": abs(comb.theta_combined - full.theta_combined),
                           "ms": ms, "points_per_s": n / (ms * 1e-3), "stage_ms": st}
                    lines.append(rec)
                    print(json.dumps(rec), flush=True)
            del c1, c2
            torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        for r in lines:
            f.write(json.dumps(r) + "\n")
    ctx.close()


if __name__ == "__main__":
    main()
