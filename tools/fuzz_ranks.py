"""Randomised rank parity: segment sizes around the cluster thresholds,
mixtures of marginals (uniform, normal, heavy tails, subnormals, huge
magnitudes, signed zeros, tie runs of every length), both rank paths and the
quantile relaunch. Every case is compared bit for bit with the oracle.

    python tools/fuzz_ranks.py [seconds] [seed]
"""
import os
import sys
import time

import numpy as np
from scipy.special import ndtri

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05530_b200 as pcb  # noqa: E402
from oracle.oracle import oracle_lib  # noqa: E402


def column(g, n):
    kind = g.integers(0, 9)
    u = g.random(n)
    if kind == 0:
        x = u
    elif kind == 1:
        x = ndtri(np.clip(u, 1e-300, 1 - 1e-16))
    elif kind == 2:
        x = np.tan(np.pi * (u - 0.5))
    elif kind == 3:
        x = np.exp(g.uniform(1, 8) * ndtri(np.clip(u, 1e-300, 1 - 1e-16)))
    elif kind == 4:  # rounded: tie runs of a controllable length
        x = np.round(ndtri(np.clip(u, 1e-12, 1 - 1e-12)), int(g.integers(0, 5)))
    elif kind == 5:  # mixture with a big constant run
        x = g.standard_normal(n)
        x[g.random(n) < g.uniform(0, 0.2)] = g.choice([0.0, -0.0, 1.5])
    elif kind == 6:  # magnitudes from subnormal to 1e308, both signs
        x = g.choice([-1.0, 1.0], n) * 10.0 ** g.uniform(-320, 308, n)
    elif kind == 7:  # sorted / reverse-sorted input
        x = np.sort(g.standard_normal(n))
        if g.random() < 0.5:
            x = x[::-1].copy()
    else:  # few distinct values
        x = g.integers(0, int(g.integers(1, 50)), n).astype(np.float64)
    return np.ascontiguousarray(x, np.float64), kind


def run(secs, seed, ctx=None, orc=None):
    """Random cases for `secs` seconds; raises AssertionError on the first mismatch."""
    g = np.random.default_rng(seed)
    orc = orc or oracle_lib()
    ctx = ctx or pcb.Context(0)
    t0, cases, paths = time.time(), 0, np.zeros(4, np.int64)
    while time.time() - t0 < secs:
        k = int(g.integers(1, 6))
        sizes = g.choice([g.integers(2, 3000), g.integers(3000, 60000), g.integers(60000, 140000),
                          g.integers(140000, 260000)], k)
        sizes = np.maximum(np.asarray(sizes, np.int64), 2)
        n = int(sizes.sum())
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64)
        c1, k1 = column(g, n)
        c2, k2 = column(g, n)
        U = pcb.normalized_ranks(pcb.DataMatrix(c1, c2), off, ctx=ctx)
        rp = ctx.rank_paths()
        paths += [rp["cluster"], rp["global"], rp["constant"], rp["invalid"]]
        for col, u, kind in ((c1, U.u1, k1), (c2, U.u2, k2)):
            want = np.concatenate([orc.rank_column(col[int(off[m]):int(off[m + 1])]) for m in range(k)])
            if not np.array_equal(u, want):
                bad = np.nonzero(u != want)[0]
                os.makedirs("gpurun_out", exist_ok=True)
                np.savez("gpurun_out/fuzz_fail.npz", c1=c1, c2=c2, off=off)
                print(f"MISMATCH case {cases} kind {kind} sizes {sizes.tolist()} first bad row {bad[0]} "
                      f"({len(bad)} rows)", flush=True)
                raise AssertionError("fuzz mismatch (inputs saved under gpurun_out/)")
        cases += 1
    return (f"fuzz ok: {cases} cases in {time.time() - t0:.0f} s; block columns by path "
            f"cluster {paths[0]} global {paths[1]} constant {paths[2]} invalid {paths[3]}")


if __name__ == "__main__":
    os.makedirs("gpurun_out", exist_ok=True)
    print(run(float(sys.argv[1]) if len(sys.argv) > 1 else 60.0, int(sys.argv[2]) if len(sys.argv) > 2 else 1))
