"""Parity at the headline and largest configs (VERDICT r1 "Next round" 1).

  C5 (BASELINE configs[4]): n = 1e9 pairs per family, K = 8000 subsets of
      125,000, device sample -> device rank/fit/variance of ALL 8000 blocks
      -> every block (or a spread of `--picks`) re-fitted by the CPU oracle
      on the same bytes (D2H) -> theta-hat, sigma2, loglik, converged and
      theta_combined compared (1e-9 relative).
  C4 (configs[3]) large segments: n = 1e8, K = 10 (n_m = 1e7) and K = 1
      (full data): device ranks (pcb_normalized_ranks) compared bit for bit
      with the oracle's normalized_ranks per segment, and the device fit
      records with the oracle's (pseudo_obs.hpp:44-65 on every segment size).

    python tools/parity_large.py c5 [--picks N] [--out profiles/r02_parity_c5.json]
    python tools/parity_large.py c4 [--n 100000000] [--out profiles/r02_parity_c4.json]
    python tools/parity_large.py configs [--fp32] [--out profiles/r02_parity_configs.json]
        every block of BASELINE configs[0..2] (C1 Gaussian 0.5 n=1e4 K=10, C2
        Frank 5 n=1e6 K=100, C3 Gumbel 2 n=1e8 K=1000) and of the fp64 C4 grid
        (3 families x 3 theta x K in {10, 100, 1000, 10000} at n=1e8)

The oracle is test infrastructure (oracle/): this script is a checker, run on
the GPU box; tests/test_gpu_large.py runs the same functions at bounded size.
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

BASE_SEED = 0x160905530
FAMILIES = [("gaussian", 0, 0.5), ("frank", 1, 5.0), ("gumbel", 2, 2.0)]
TOL = 1e-9


def _rel(a, b):
    return np.abs(a - b) / np.maximum(np.abs(b), 1e-300)


def _recs_np(recs):
    th = np.array([r.theta_hat for r in recs])
    s2 = np.array([r.sigma2 for r in recs])
    ll = np.array([r.loglik for r in recs])
    cv = np.array([bool(r.converged) for r in recs])
    return th, s2, ll, cv


def _device_records(ctx, fam, c1, c2, n, off, precision=0):
    """pcb_fit_blocks over device columns -> host structured records."""
    import torch
    from paper_1609_05530_b200 import _lib as L
    k = len(off) - 1
    rec = torch.zeros((k, 6), dtype=torch.int64, device=c1.device)
    offc = np.ascontiguousarray(off, np.uint64)
    ctx.check(ctx.lib.pcb_fit_blocks(ctx.ptr, fam, precision, c1.data_ptr(), c2.data_ptr(), n,
                                     offc.ctypes.data_as(C.POINTER(C.c_uint64)), k, rec.data_ptr()))
    torch.cuda.synchronize()
    arr = rec.cpu().numpy()
    out = (L.FitResultC * k).from_buffer_copy(arr.tobytes())
    return out


def _compare(dev, cpu):
    dth, ds2, dll, dcv = _recs_np(dev)
    cth, cs2, cll, ccv = _recs_np(cpu)
    ok = ccv & dcv
    r = {"blocks": int(len(cth)), "converged_mismatch": int(np.sum(dcv != ccv)),
         "converged": int(np.sum(ccv)),
         "max_rel_theta": float(_rel(dth[ok], cth[ok]).max()) if ok.any() else 0.0,
         "max_rel_sigma2": float(_rel(ds2[ok], cs2[ok]).max()) if ok.any() else 0.0,
         "max_rel_loglik": float(_rel(dll[ok], cll[ok]).max()) if ok.any() else 0.0}
    r["worst_block_theta"] = int(np.flatnonzero(ok)[np.argmax(_rel(dth[ok], cth[ok]))]) if ok.any() else -1
    return r


def c5_family(ctx, orc, fam, theta, n=1_000_000_000, K=8000, picks=None, chunk=400, workers=None, precision=0):
    """All K blocks on device; the oracle re-fits `picks` (all if None).
    precision 1: the device's fp32 likelihood path, held to 1e-5."""
    import torch
    import paper_1609_05530_b200 as pcb
    workers = workers or os.cpu_count() or 1
    q = n // K
    off = np.arange(K + 1, dtype=np.uint64) * np.uint64(q)
    off[-1] = n
    X = pcb.sample_matrix(fam, theta, n, K, base_seed=BASE_SEED, device_out=True, ctx=ctx)
    t0 = time.perf_counter()
    dev = _device_records(ctx, fam, X.col1, X.col2, n, off, precision)
    t_dev = time.perf_counter() - t0
    sel = np.arange(K) if picks is None else np.unique(np.asarray(picks, np.int64))
    cpu = []
    t_cpu = 0.0
    for s0 in range(0, len(sel), chunk):
        blk = sel[s0:s0 + chunk]
        lens = (off[blk + 1] - off[blk]).astype(np.int64)
        h1 = np.concatenate([X.col1[int(off[b]):int(off[b + 1])].cpu().numpy() for b in blk])
        h2 = np.concatenate([X.col2[int(off[b]):int(off[b + 1])].cpu().numpy() for b in blk])
        o = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
        t1 = time.perf_counter()
        cpu.extend(list(orc.fit_blocks(fam, h1, h2, o, workers=workers)))
        t_cpu += time.perf_counter() - t1
    dsel = [dev[int(b)] for b in sel]
    res = _compare(dsel, cpu)
    res["worst_block_theta"] = int(sel[res["worst_block_theta"]]) if res["worst_block_theta"] >= 0 else -1
    # theta_combined: the device combine of the device records vs the oracle
    # combine of the oracle records, over the same blocks in block order
    from paper_1609_05530_b200 import _lib as L
    arr = (L.FitResultC * len(dsel))(*dsel)
    comb = L.CombinedC()
    ctx.check(ctx.lib.pcb_combine(ctx.ptr, C.addressof(arr), len(dsel), None, C.byref(comb)))
    tc_cpu, _, used_cpu = orc.combine(cpu)
    res.update({"family": fam, "theta_true": theta, "n": n, "K": K, "blocks_checked": int(len(sel)),
                "theta_combined_device": comb.theta_combined, "theta_combined_oracle": tc_cpu,
                "rel_theta_combined": abs(comb.theta_combined - tc_cpu) / abs(tc_cpu),
                "blocks_used_device": int(comb.blocks_used), "blocks_used_oracle": int(used_cpu),
                "device_s": t_dev, "oracle_s": t_cpu, "oracle_threads": workers})
    if picks is not None:
        tall = (L.FitResultC * K)(*dev)
        ctx.check(ctx.lib.pcb_combine(ctx.ptr, C.addressof(tall), K, None, C.byref(comb)))
        res["theta_combined_device_all_blocks"] = comb.theta_combined
    tol = 1e-5 if precision else TOL
    res["precision"] = "fp32" if precision else "fp64"
    res["tol"] = tol
    res["ok"] = bool(res["converged_mismatch"] == 0 and res["max_rel_theta"] <= tol and
                     res["max_rel_sigma2"] <= tol and res["rel_theta_combined"] <= tol and
                     res["blocks_used_device"] == res["blocks_used_oracle"])
    del X
    torch.cuda.empty_cache()
    return res


def _digest(a):
    """BLAKE2b-64 of a segment's float64 bytes (per-segment rank digest)."""
    return hashlib.blake2b(np.ascontiguousarray(a, np.float64).tobytes(), digest_size=8).hexdigest()


def c4_case(ctx, orc, fam, theta, n, K, workers=None, rank_workers=None):
    """n rows sampled as 1000 seeded blocks (sweep.py layout), partitioned into
    K contiguous blocks: ranks bit for bit per segment + fit records."""
    import torch
    import paper_1609_05530_b200 as pcb
    workers = workers or os.cpu_count() or 1
    X = pcb.sample_matrix(fam, theta, n, 1000, base_seed=BASE_SEED, device_out=True, ctx=ctx)
    off = orc.partition(n, K)
    t0 = time.perf_counter()
    dev = _device_records(ctx, fam, X.col1, X.col2, n, off)
    t_dev = time.perf_counter() - t0
    U = pcb.normalized_ranks(X, off, ctx=ctx)
    h1, h2 = X.col1.cpu().numpy(), X.col2.cpu().numpy()
    u1, u2 = U.u1.cpu().numpy(), U.u2.cpu().numpy()
    del U
    segs = [(int(off[m]), int(off[m + 1])) for m in range(K)]
    jobs = [(j, a, b) for (a, b) in segs for j in (0, 1)]

    def rank_job(job):
        j, a, b = job
        ref = orc.rank_column((h1, h2)[j][a:b])
        got = (u1, u2)[j][a:b]
        return bool(np.array_equal(got, ref)), _digest(got), _digest(ref)

    t1 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=rank_workers or workers) as ex:
        rk = list(ex.map(rank_job, jobs))
    t_rank = time.perf_counter() - t1
    t1 = time.perf_counter()
    cpu = list(orc.fit_blocks(fam, h1, h2, off, workers=min(workers, K)))
    t_fit = time.perf_counter() - t1
    res = _compare(dev, cpu)
    res.update({"family": fam, "theta_true": theta, "n": n, "K": K, "segment_rows": int(n // K),
                "rank_columns_checked": len(rk), "rank_columns_identical": int(sum(r[0] for r in rk)),
                "rank_digests_device": [r[1] for r in rk], "rank_digests_oracle": [r[2] for r in rk],
                "device_s": t_dev, "oracle_rank_s": t_rank, "oracle_fit_s": t_fit})
    if K > 1:
        from paper_1609_05530_b200 import _lib as L
        arr = (L.FitResultC * K)(*dev)
        comb = L.CombinedC()
        ctx.check(ctx.lib.pcb_combine(ctx.ptr, C.addressof(arr), K, None, C.byref(comb)))
        tc_cpu, _, _ = orc.combine(cpu)
        res["rel_theta_combined"] = abs(comb.theta_combined - tc_cpu) / abs(tc_cpu)
    res["ok"] = bool(res["rank_columns_identical"] == res["rank_columns_checked"] and
                     res["converged_mismatch"] == 0 and res["max_rel_theta"] <= TOL and
                     res["max_rel_sigma2"] <= TOL and res.get("rel_theta_combined", 0.0) <= TOL)
    del X
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["c5", "c4", "configs"])
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--picks", type=int, default=None, help="C5: blocks per family spread over the range (default all)")
    ap.add_argument("--families", default="0,1,2")
    ap.add_argument("--ks", default="10,1")
    ap.add_argument("--out", default=None)
    ap.add_argument("--fp32", action="store_true", help="configs: the fp32 likelihood path (bar 1e-5)")
    args = ap.parse_args()
    import paper_1609_05530_b200 as pcb
    from oracle.oracle import oracle_lib
    orc = oracle_lib()
    ctx = pcb.Context(0)
    fams = [f for f in FAMILIES if str(f[1]) in args.families.split(",")]
    out = []
    if args.which == "c5":
        n = args.n or 1_000_000_000
        for name, fam, th in fams:
            picks = None if args.picks is None else np.linspace(0, 7999, args.picks).round().astype(np.int64)
            r = c5_family(ctx, orc, fam, th, n=n, picks=picks)
            r["name"] = name
            print(json.dumps(r), flush=True)
            out.append(r)
    elif args.which == "configs":
        cases = [("C1", 0, 0.5, 10_000, 10), ("C2", 1, 5.0, 1_000_000, 100), ("C3", 2, 2.0, 100_000_000, 1000)]
        for fam, ths in ((0, (0.2, 0.5, 0.8)), (1, (2.0, 5.0, 10.0)), (2, (1.5, 2.0, 3.0))):
            for th in ths:
                for K in (10, 100, 1000, 10000):
                    cases.append(("C4", fam, th, 100_000_000, K))
        for cfg, fam, th, n, K in cases:
            if str(fam) not in args.families.split(","):
                continue
            r = c5_family(ctx, orc, fam, th, n=n, K=K, precision=1 if args.fp32 else 0)
            r["name"] = cfg
            print(json.dumps(r), flush=True)
            out.append(r)
    else:
        n = args.n or 100_000_000
        for name, fam, th in fams:
            for K in [int(k) for k in args.ks.split(",")]:
                r = c4_case(ctx, orc, fam, th, n, K)
                r["name"] = name
                short = {k: v for k, v in r.items() if not k.startswith("rank_digests")}
                print(json.dumps(short), flush=True)
                out.append(r)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"config": args.which, "cores": os.cpu_count(), "results": out}, f, indent=1)
    ctx.close()
    sys.exit(0 if all(r["ok"] for r in out) else 1)


if __name__ == "__main__":
    main()
