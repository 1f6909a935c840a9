"""Randomised pipeline parity (ranks -> fit -> variance -> combine) against
the oracle: random family and parameter, random block sizes (30 rows to
260k), random monotone marginal transforms of a device-sampled copula (so
the cluster, quantile-relaunch and global rank paths all feed the fit), fp64
records within 1e-9 relative and the combine within 1e-9; one case in four
runs the fp32 likelihood path (bar 1e-5; its Frank |theta| < 2 and Gumbel
theta < 1.1 passes run in fp64 arithmetic).

    python tools/fuzz_fit.py [seconds] [seed]
"""
import os
import sys
import time

import numpy as np
from scipy.special import ndtri

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05530_b200 as pcb  # noqa: E402
from oracle.oracle import oracle_lib  # noqa: E402
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_oracle import frank_cond_tol  # noqa: E402

TRANSFORMS = [lambda u: u, lambda u: ndtri(u), lambda u: np.tan(np.pi * (u - 0.5)), lambda u: -np.log1p(-u),
              lambda u: np.exp(4.0 * ndtri(u))]


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def run(secs, seed, ctx=None, orc=None):
    """Random cases for `secs` seconds; raises AssertionError on the first mismatch."""
    g = np.random.default_rng(seed)
    orc = orc or oracle_lib()
    ctx = ctx or pcb.Context(0)
    t0, cases, worst, worst32 = time.time(), 0, 0.0, 0.0
    while time.time() - t0 < secs:
        fam = int(g.integers(0, 3))
        theta = [g.uniform(-0.95, 0.95), g.choice([-1, 1]) * g.uniform(0.3, 20), g.uniform(1.0, 6.0)][fam]
        k = int(g.integers(1, 7))
        sizes = np.asarray(g.choice([g.integers(30, 2000), g.integers(2000, 50000), g.integers(100000, 140000),
                                     g.integers(140000, 260000)], k), np.int64)
        n = int(sizes.sum())
        X = pcb.sample_matrix(fam, float(theta), n, 1, base_seed=int(g.integers(1, 2**62)), ctx=ctx)
        f1, f2 = TRANSFORMS[g.integers(0, 5)], TRANSFORMS[g.integers(0, 5)]
        c1, c2 = np.ascontiguousarray(f1(np.asarray(X.col1))), np.ascontiguousarray(f2(np.asarray(X.col2)))
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64)
        fp32 = g.random() < 0.25
        prec = pcb.Precision.fp32 if fp32 else pcb.Precision.fp64
        got = pcb.fit_blocks(fam, pcb.DataMatrix(c1, c2), off, precision=prec, ctx=ctx)
        want = orc.fit_blocks(fam, c1, c2, off)
        for m, (a, b) in enumerate(zip(got, want)):
            ok = bool(a.converged) == bool(b.converged)
            if ok and b.converged:
                # Frank near theta = 0: the reference formulas lose ~eps/theta^2
                # (tests/test_oracle.py::frank_cond_tol, tests/golden/make_frank_near_zero.py)
                tol = frank_cond_tol(b.theta_hat) if fam == 1 else 1e-9
                e = max(rel(a.theta_hat, b.theta_hat), rel(a.sigma2, b.sigma2))
                if fp32:
                    tol = max(tol, 1e-5)
                    worst32 = max(worst32, e)
                else:
                    worst = max(worst, e * 1e-9 / tol)
                ok = e <= tol
            if not ok:
                os.makedirs("gpurun_out", exist_ok=True)
                np.savez("gpurun_out/fuzz_fit_fail.npz", c1=c1, c2=c2, off=off, fam=fam, theta=theta)
                print(f"MISMATCH case {cases} fam {fam} theta {theta} fp32 {fp32} block {m} size {sizes[m]}: "
                      f"{(a.theta_hat, a.sigma2, a.converged)} vs {(b.theta_hat, b.sigma2, b.converged)}", flush=True)
                raise AssertionError("fuzz mismatch (inputs saved under gpurun_out/)")
        cases += 1
    return (f"fuzz fit ok: {cases} cases in {time.time() - t0:.0f} s; worst fp64 rel error {worst:.2e} (in units of the "
            f"bar x 1e-9), worst fp32-path rel error {worst32:.2e} (bar 1e-5)")


if __name__ == "__main__":
    os.makedirs("gpurun_out", exist_ok=True)
    print(run(float(sys.argv[1]) if len(sys.argv) > 1 else 60.0, int(sys.argv[2]) if len(sys.argv) > 2 else 1))
