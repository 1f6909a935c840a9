"""Command-line front end (SPEC.md cli module, :405-470) over the B200 path.

    python -m paper_1609_05530_b200.cli fit FILE.csv --family gaussian
    python -m paper_1609_05530_b200.cli split-fit FILE.csv --family frank --subsets 10 [--scheme strided] [--out blocks.csv]
    python -m paper_1609_05530_b200.cli simulate --family gumbel --theta 2 --rows 50000 --subsets 10 \\
        --replicates 5 --seed 0x160905530 --out results/
    python -m paper_1609_05530_b200.cli report results/ [--out report_dir]

Exit codes: 0 success, 2 usage error, 3 data error, 4
convergence failure. Output CSVs carry a versioned schema comment line.
Figures are not produced.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import math
import os
import sys
import time

import numpy as np

SCHEMA = "# parcop-b200 csv schema v1"


class DataError(Exception):
    pass


def read_csv(path: str):
    """2-column numeric CSV, header optional (auto-detected), >= 30 rows."""
    try:
        text = open(path).read()
    except OSError as e:
        raise DataError(f"cannot read {path}: {e}")
    rows = [r for r in csv.reader(io.StringIO(text)) if r and not r[0].startswith("#")]
    if not rows:
        raise DataError("empty file")

    def numeric(r):
        try:
            [float(x) for x in r]
            return True
        except ValueError:
            return False

    if not numeric(rows[0]):
        rows = rows[1:]  # header
    if any(len(r) != 2 for r in rows):
        raise DataError("expected 2 numeric columns")
    try:
        a = np.array([[float(x) for x in r] for r in rows], np.float64)
    except ValueError:
        raise DataError("non-numeric cell")
    if len(a) < 30:
        raise DataError("need at least 30 rows")
    return np.ascontiguousarray(a[:, 0]), np.ascontiguousarray(a[:, 1])


def _family(s):
    import paper_1609_05530_b200 as pcb
    f = pcb.family_from_string(s)
    if f is None:
        raise argparse.ArgumentTypeError(f"unknown family {s!r}")
    return f


def _manifest(out_dir, command, cfg):
    from . import _lib
    with open(os.path.join(out_dir, "manifest.txt"), "w") as f:
        f.write(json.dumps({"command": command, "config": cfg, "tool": "paper_1609_05530_b200",
                            "abi": int(_lib.load().pcb_abi_version()), "seed": cfg.get("seed")},
                           sort_keys=True) + "\n")


def cmd_fit(args) -> int:
    import paper_1609_05530_b200 as pcb
    c1, c2 = read_csv(args.input)
    r = pcb.fit(args.family, pcb.normalized_ranks(pcb.DataMatrix(c1, c2)))
    print(f"theta_hat={r.theta_hat!r} se={math.sqrt(r.sigma2) if r.sigma2 > 0 else float('nan')!r} "
          f"loglik={r.loglik!r} n={r.n}")
    return 0 if r.converged else 4


def cmd_split_fit(args) -> int:
    import paper_1609_05530_b200 as pcb
    c1, c2 = read_csv(args.input)
    scheme = pcb.Scheme.Strided if args.scheme == "strided" else pcb.Scheme.Contiguous
    res = pcb.fit_parallel(args.family, pcb.DataMatrix(c1, c2), args.subsets, scheme=scheme)
    part = pcb.partition(len(c1), args.subsets, scheme)
    sizes = np.diff(np.asarray(part.offsets, np.int64))
    lines = [SCHEMA, "m,n_m,theta_hat,sigma2,converged,weight"]
    for m, (r, w) in enumerate(zip(res.per_block, res.weights)):
        lines.append(f"{m},{int(sizes[m])},{r.theta_hat!r},{r.sigma2!r},{int(r.converged)},{float(w)!r}")
    table = "\n".join(lines) + "\n"
    if args.out:
        with open(args.out, "w") as f:
            f.write(table)
    else:
        sys.stdout.write(table)
    print(f"theta_combined={res.theta_combined!r} blocks_used={res.blocks_used} "
          f"wall_clock_per_block={res.wall_clock_per_block!r}")
    return 0


def cmd_simulate(args) -> int:
    from .study import SimConfig, run_study
    cfg = SimConfig(args.family, args.theta, args.rows, args.subsets, args.replicates, args.quad_nodes,
                    int(args.seed, 0))
    rep = run_study(cfg)
    os.makedirs(args.out, exist_ok=True)
    with open(os.path.join(args.out, "summary.csv"), "w") as f:
        f.write(SCHEMA + "\n")
        f.write("family,theta_true,N,M,S,theta_full_sim,theta_combined_sim,bias,mse,rel_l1,rel_l2,"
                "mean_subset_s,mean_full_s,seed\n")
        f.write(f"{int(cfg.family)},{cfg.theta_true!r},{cfg.N},{cfg.M},{cfg.S},{rep.theta_full_sim!r},"
                f"{rep.theta_combined_sim!r},{rep.bias_hat!r},{rep.mse_hat!r},{rep.rel_l1!r},{rep.rel_l2!r},"
                f"{rep.mean_subset_seconds!r},{rep.mean_full_seconds!r},{cfg.base_seed}\n")
    with open(os.path.join(args.out, "replicates.csv"), "w") as f:
        f.write(SCHEMA + "\n")
        f.write("s,theta_full,theta_combined,full_s,subset_s\n")
        for r in rep.per_replicate:
            f.write(f"{r.s},{r.theta_full!r},{r.theta_combined!r},{r.full_seconds!r},{r.subset_seconds!r}\n")
    _manifest(args.out, "simulate", {"family": int(cfg.family), "theta": cfg.theta_true, "N": cfg.N, "M": cfg.M,
                                      "S": cfg.S, "quad_nodes": cfg.quad_nodes, "seed": cfg.base_seed,
                                      "quad_unstable": rep.quad_unstable, "time": time.time()})
    print(f"bias={rep.bias_hat!r} mse={rep.mse_hat!r} rel_l1={rep.rel_l1!r} rel_l2={rep.rel_l2!r}")
    return 0


SUMMARY_COLS = ["family", "theta_true", "N", "M", "S", "theta_full_sim", "theta_combined_sim", "bias", "mse",
                "rel_l1", "rel_l2", "mean_subset_s", "mean_full_s", "seed"]
FAMILY_NAMES = {0: "gaussian", 1: "frank", 2: "gumbel"}


def cmd_report(args) -> int:  # merge summary.csv files into Table-1 layout + metric tables
    found, rows = [], []
    for root, _, files in sorted(os.walk(args.results)):
        for fn in sorted(files):
            if fn == "summary.csv":
                found.append(os.path.join(root, fn))
    for path in found:
        try:
            lines = open(path).read().splitlines()
        except OSError as e:
            print(f"error: {path}: {e}", file=sys.stderr)
            continue
        if not lines or lines[0].strip() != SCHEMA:
            print(f"error: {path}: schema mismatch (expected '{SCHEMA}')", file=sys.stderr)
            continue
        rd = list(csv.DictReader(io.StringIO("\n".join(lines[1:]))))
        if not rd or any(c not in rd[0] for c in SUMMARY_COLS):
            print(f"error: {path}: missing columns", file=sys.stderr)
            continue
        for r in rd:
            try:
                rows.append({"family": FAMILY_NAMES.get(int(r["family"]), r["family"]), "theta": float(r["theta_true"]),
                             "N": int(r["N"]), "M": int(r["M"]), "S": int(r["S"]), "bias": float(r["bias"]),
                             "mse": float(r["mse"]), "rel_l1": float(r["rel_l1"]), "rel_l2": float(r["rel_l2"]),
                             "sub_s": float(r["mean_subset_s"]), "full_s": float(r["mean_full_s"])})
            except (KeyError, ValueError) as e:
                print(f"error: {path}: corrupt row ({e})", file=sys.stderr)
    if not rows:
        print("error: data: no results found", file=sys.stderr)
        return 3
    out = args.out or args.results
    os.makedirs(out, exist_ok=True)
    # Table 1 layout (PAPER Table 1): per (family, N) the mean per-subset seconds for each M and full-data seconds
    ms = sorted({r["M"] for r in rows})
    cells = {}
    for r in rows:
        c = cells.setdefault((r["family"], r["N"]), {"sub": {}, "full": []})
        c["sub"].setdefault(r["M"], []).append(r["sub_s"])
        c["full"].append(r["full_s"])
    order = {"gaussian": 0, "frank": 1, "gumbel": 2}
    keys = sorted(cells, key=lambda k: (order.get(k[0], 9), k[1]))
    timing = [["family", "N"] + [f"subset_s_M{m}" for m in ms] + ["full_s"]]
    for fam, n in keys:
        c = cells[(fam, n)]
        timing.append([fam, str(n)] + [repr(float(np.mean(c["sub"][m]))) if m in c["sub"] else "" for m in ms]
                      + [repr(float(np.mean(c["full"])))])
    acc = [["family", "theta_true", "N", "M", "S", "bias", "mse", "rel_l1", "rel_l2"]]
    for r in sorted(rows, key=lambda r: (order.get(r["family"], 9), r["theta"], r["N"], r["M"])):
        acc.append([r["family"], repr(r["theta"]), str(r["N"]), str(r["M"]), str(r["S"]), repr(r["bias"]),
                    repr(r["mse"]), repr(r["rel_l1"]), repr(r["rel_l2"])])
    for name, table in (("report_timing.csv", timing), ("report_accuracy.csv", acc)):
        with open(os.path.join(out, name), "w") as f:
            f.write(SCHEMA + "\n" + "\n".join(",".join(t) for t in table) + "\n")
    _manifest(out, "report", {"results": os.path.abspath(args.results), "files": found, "rows": len(rows),
                              "time": time.time()})
    for title, table in (("Computation time (seconds): mean per subset by M, full data", timing),
                         ("Accuracy of the combined estimate", acc)):
        w = [max(len(t[i]) for t in table) for i in range(len(table[0]))]
        print(title)
        for t in table:
            print("  " + "  ".join(x.rjust(w[i]) for i, x in enumerate(t)))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="parcop-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("fit")
    p.add_argument("input")
    p.add_argument("--family", type=_family, default="gaussian")
    p = sub.add_parser("split-fit")
    p.add_argument("input")
    p.add_argument("--family", type=_family, default="gaussian")
    p.add_argument("--subsets", type=int, default=10)
    p.add_argument("--scheme", choices=["contiguous", "strided"], default="contiguous")
    p.add_argument("--out", default=None)
    p = sub.add_parser("simulate")
    p.add_argument("--family", type=_family, default="gaussian")
    p.add_argument("--theta", type=float, default=0.3)
    p.add_argument("--rows", type=int, default=50000)
    p.add_argument("--subsets", type=int, default=10)
    p.add_argument("--replicates", type=int, default=50)
    p.add_argument("--quad-nodes", type=int, default=200)
    p.add_argument("--seed", default=hex(0x160905530))
    p.add_argument("--out", default="results")
    p = sub.add_parser("report")
    p.add_argument("results")
    p.add_argument("--out", default=None)
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    if args.cmd == "report":  # host-only: reads CSVs, no device needed
        return cmd_report(args)
    import paper_1609_05530_b200 as pcb
    try:
        return {"fit": cmd_fit, "split-fit": cmd_split_fit, "simulate": cmd_simulate}[args.cmd](args)
    except DataError as e:
        print(f"error: data: {e}", file=sys.stderr)
        return 3
    except (ValueError, pcb.DomainError) as e:
        print(f"error: usage: {e}", file=sys.stderr)
        return 2
    except pcb.ConvergenceError as e:
        print(f"error: convergence: {e}", file=sys.stderr)
        return 4


if __name__ == "__main__":
    sys.exit(main())
