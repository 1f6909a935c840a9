"""sim_study on the B200 pipeline: the paper's simulation
study — per replicate, one sample, the full-data MPL fit (M = 1) and the
divide-and-combine fit (Eq. 16) on the SAME sample (paired design), then
bias (Eq. 17 - Eq. 18), paired MSE, and the relative L1/L2 distances of
Eq. 19-20 on device (tensor Gauss-Legendre, `pcb_rel_error`).

Everything device-side goes through the C-ABI (libparcop_b200.so); this
module is host bookkeeping only.

Seeds: replicate s of a cell draws its sample from
    seed_s = mix_seed(base_seed, {family, N, M, s})        (rng.hpp:24-29)
used as the base seed of the counter-based sampler (`sample_matrix`), so
cells are independent and individually re-runnable.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from .parcop import (BASE_SEED, Context, _check_theta, default_context, fit, fit_parallel, normalized_ranks,
                     sample_matrix)

_M64 = (1 << 64) - 1


def splitmix64(z: int) -> int:  # rng.hpp:15-20
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def mix_seed(base: int, parts: Sequence[int]) -> int:  # rng.hpp:24-29
    h = splitmix64(base & _M64)
    for p in parts:
        h = splitmix64(h ^ (int(p) & _M64))
    return h


@dataclass
class SimConfig:
    family: int
    theta_true: float
    N: int
    M: int
    S: int = 50
    quad_nodes: int = 200
    base_seed: int = BASE_SEED
    workers: int = 1  # kept for interface parity; the device runs every block at once

    def validate(self):
        if self.N // max(self.M, 1) < 30 or self.M < 1:
            raise ValueError("SimConfig: need N/M >= 30")
        if self.S < 1:
            raise ValueError("SimConfig: need S >= 1")
        if self.quad_nodes < 64:
            raise ValueError("SimConfig: need quad_nodes >= 64")
        _check_theta(int(self.family), self.theta_true)


@dataclass
class ReplicateRow:
    s: int
    seed: int
    theta_full: float
    theta_combined: float
    full_seconds: float
    subset_seconds: float  # mean per subset (fit_parallel wall / M)


@dataclass
class SimReport:
    theta_combined_sim: float
    theta_full_sim: float
    bias_hat: float
    mse_hat: float
    rel_l1: float
    rel_l2: float
    mean_subset_seconds: float
    mean_full_seconds: float
    rel_l1_doubled: float = float("nan")  # node-doubling diagnostic
    rel_l2_doubled: float = float("nan")
    quad_unstable: bool = False
    per_replicate: List[ReplicateRow] = field(default_factory=list)


def rel_error(family, theta_a: float, theta_b: float, quad_nodes: int = 200, ctx: Context = None):
    """(rel_l1, rel_l2) of SPEC.md:362-374 on device."""
    ctx = ctx or default_context()
    l1, l2 = C.c_double(), C.c_double()
    ctx.check(ctx.lib.pcb_rel_error(ctx.ptr, int(family), float(theta_a), float(theta_b), int(quad_nodes),
                                    C.byref(l1), C.byref(l2)))
    return l1.value, l2.value


def rel_l1(family, theta_a, theta_b, quad_nodes=200, ctx: Context = None) -> float:
    return rel_error(family, theta_a, theta_b, quad_nodes, ctx)[0]


def rel_l2(family, theta_a, theta_b, quad_nodes=200, ctx: Context = None) -> float:
    return rel_error(family, theta_a, theta_b, quad_nodes, ctx)[1]


def est_bias(rows: Sequence[ReplicateRow]) -> float:  # SPEC.md:348-353, Eq. 17 mean minus Eq. 18 mean
    if not rows:
        raise ValueError("est_bias: empty input")
    return sum(r.theta_combined for r in rows) / len(rows) - sum(r.theta_full for r in rows) / len(rows)


def est_mse(rows: Sequence[ReplicateRow]) -> float:  # SPEC.md:354-361, paired squared differences
    if not rows:
        raise ValueError("est_mse: empty input")
    return sum((r.theta_combined - r.theta_full) ** 2 for r in rows) / len(rows)


def replicate_seed(cfg: SimConfig, s: int) -> int:
    return mix_seed(cfg.base_seed, (int(cfg.family), cfg.N, cfg.M, s))


def run_replicate(cfg: SimConfig, s: int, ctx: Context = None) -> ReplicateRow:
    ctx = ctx or default_context()
    seed = replicate_seed(cfg, s)
    X = sample_matrix(cfg.family, cfg.theta_true, cfg.N, 1, base_seed=seed, ctx=ctx)
    t0 = time.perf_counter()
    full = fit(cfg.family, normalized_ranks(X, ctx=ctx), ctx=ctx)
    t1 = time.perf_counter()
    comb = fit_parallel(cfg.family, X, cfg.M, ctx=ctx)
    t2 = time.perf_counter()
    if not full.converged:
        raise RuntimeError(f"run_study: full-data fit did not converge (replicate {s})")
    return ReplicateRow(s, seed, full.theta_hat, comb.theta_combined, t1 - t0, (t2 - t1) / cfg.M)


def run_study(cfg: SimConfig, ctx: Context = None) -> SimReport:
    cfg.validate()
    ctx = ctx or default_context()
    rows = [run_replicate(cfg, s, ctx) for s in range(cfg.S)]
    tc = sum(r.theta_combined for r in rows) / len(rows)  # Eq. 17
    tf = sum(r.theta_full for r in rows) / len(rows)  # Eq. 18
    l1, l2 = rel_error(cfg.family, tf, tc, cfg.quad_nodes, ctx)
    l1d, l2d = rel_error(cfg.family, tf, tc, 2 * cfg.quad_nodes, ctx)
    unstable = any(abs(b - a) > 0.1 * abs(a) for a, b in ((l1, l1d), (l2, l2d)) if a > 0.0)
    return SimReport(tc, tf, est_bias(rows), est_mse(rows), l1, l2,
                     sum(r.subset_seconds for r in rows) / len(rows), sum(r.full_seconds for r in rows) / len(rows),
                     l1d, l2d, unstable, rows)
