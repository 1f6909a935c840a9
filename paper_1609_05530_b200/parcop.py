"""Python mirror of the reference's `parcop::` interface for the hot path.

Same names, argument meaning and error behaviour as the reference headers
(/root/reference/proj/include/parcop) and the SPEC contracts of its absent
estimator / partition-combine modules:

    normalized_ranks      pseudo_obs.hpp:71-77
    validate_data         pseudo_obs.hpp:30-37 (folded into the rank kernel)
    pseudo_loglik
    fit / FitResult
    asymptotic_variance
    partition / Partition SPEC.md:263-267, 275-283
    combine
    fit_parallel
    sample_matrix         copula.hpp:413-423 (device counter-based streams)

Exceptions: ValueError  == std::invalid_argument,
            DomainError == std::domain_error (a ValueError subclass),
            ConvergenceError for combine / fit_parallel with no converged block.

Inputs may be numpy arrays (host) or CUDA torch tensors (device, used in
place). Every computation runs in libparcop_b200.so on the GPU; there is no
CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L


class CopulaFamily(IntEnum):  # copula.hpp:25
    Gaussian = 0
    Frank = 1
    Gumbel = 2


class Scheme(IntEnum):
    Contiguous = 0
    Strided = 1


class Precision(IntEnum):
    fp64 = 0
    fp32 = 1


class DomainError(ValueError):
    """std::domain_error."""


class ConvergenceError(RuntimeError):
    """No converged block to combine."""


class CudaError(RuntimeError):
    """Device / runtime failure (no sm_100 device, launch error, ...)."""


BASE_SEED = 0x160905530


def family_from_string(s: str) -> Optional[CopulaFamily]:  # copula.hpp:36-43
    t = s.lower()
    if t in ("gaussian", "normal"):
        return CopulaFamily.Gaussian
    if t == "frank":
        return CopulaFamily.Frank
    if t == "gumbel":
        return CopulaFamily.Gumbel
    return None


@dataclass
class DataMatrix:  # pseudo_obs.hpp:15-20
    col1: object
    col2: object

    def rows(self) -> int:
        return int(len(self.col1))


@dataclass
class PseudoSample:  # pseudo_obs.hpp:23-28
    u1: object
    u2: object

    def rows(self) -> int:
        return int(len(self.u1))


@dataclass
class FitResult:
    theta_hat: float
    sigma2: float
    n: int
    loglik: float
    iterations: int
    converged: bool
    status: int = 0


@dataclass
class Partition:  # SPEC.md:263-267 (offsets into the scheme's row order)
    offsets: np.ndarray
    scheme: Scheme

    @property
    def blocks(self) -> int:
        return len(self.offsets) - 1


@dataclass
class CombinedResult:
    theta_combined: float
    per_block: List[FitResult]
    weights: np.ndarray
    wall_clock_per_block: float
    blocks_used: int
    stage_ms: dict = field(default_factory=dict)


# ----------------------------------------------------------------- context
def _raise(ctx_ptr, rc):
    lib = L.load()
    msg = lib.pcb_last_error(ctx_ptr)
    msg = msg.decode() if msg else ""
    if rc == L.PCB_E_INVALID:
        raise ValueError(msg)
    if rc == L.PCB_E_DOMAIN:
        raise DomainError(msg)
    if rc == L.PCB_E_CONVERGENCE:
        raise ConvergenceError(msg)
    raise CudaError(msg or f"pcb error {rc}")


class Context:
    """One pcb_context (device buffers, stream, cached workspace).

    `devices` (a list) opens a multi-device context (pcb_create_multi):
    fit_blocks / fit_parallel shard their blocks over all of them and gather
    the records by peer copies; everything else runs on the first device."""

    def __init__(self, device: int = 0, devices: Optional[Sequence[int]] = None):
        self.lib = L.load()
        devs = list(devices) if devices is not None else [int(device)]
        arr = (C.c_int * len(devs))(*devs)
        self.ptr = self.lib.pcb_create_multi(arr, len(devs))
        if not self.ptr:
            raise CudaError(self.lib.pcb_last_error(None).decode())
        self.device = devs[0]
        self.devices = devs

    def close(self):
        if getattr(self, "ptr", None):
            self.lib.pcb_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc):
        if rc != L.PCB_OK:
            _raise(self.ptr, rc)

    def set_stream(self, stream_handle: int):
        self.check(self.lib.pcb_set_stream(self.ptr, C.c_void_p(stream_handle)))

    def launch_count(self) -> int:
        return int(self.lib.pcb_launch_count(self.ptr))

    def stage_times(self) -> dict:
        buf = (C.c_double * 12)()
        k = self.lib.pcb_stage_times(self.ptr, buf, 12)
        names = ["rank", "prepare", "newton", "variance", "finalize", "lik_kernel_ms", "lik_launches",
                 "warm_kernel_ms", "warm_launches", "var_point_ms"]
        return {names[i]: float(buf[i]) for i in range(k)}

    def rank_paths(self) -> dict:
        """Block columns of the last rank stage by path (cluster / global / constant / invalid)."""
        buf = (C.c_uint64 * 4)()
        self.check(self.lib.pcb_rank_paths(self.ptr, buf))
        return dict(zip(("cluster", "global", "constant", "invalid"), (int(v) for v in buf)))

    def trim(self):
        self.check(self.lib.pcb_trim(self.ptr))

    def fp64_peak(self) -> float:
        v = C.c_double()
        self.check(self.lib.pcb_measure_fp64_peak(self.ptr, C.byref(v)))
        return v.value


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


# ----------------------------------------------------------------- buffers
def _ptr(a):
    """(pointer, keepalive) for a numpy array or a CUDA torch tensor."""
    if isinstance(a, np.ndarray):
        a = np.ascontiguousarray(a)
        return a.ctypes.data, a
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            a = a.contiguous()
        return a.data_ptr(), a
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return arr.ctypes.data, arr


def _f64(a):
    if isinstance(a, np.ndarray) or not hasattr(a, "data_ptr"):
        return np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    import torch
    return a.to(torch.float64).contiguous()


def _like(a, n):
    if hasattr(a, "data_ptr") and not isinstance(a, np.ndarray):
        import torch
        return torch.empty(n, dtype=torch.float64, device=a.device)
    return np.empty(n, np.float64)


def _offsets(n_rows, segments):
    if segments is None:
        off = np.array([0, n_rows], np.uint64)
    else:
        off = np.ascontiguousarray(np.asarray(segments, dtype=np.uint64))
    return off, off.ctypes.data_as(C.POINTER(C.c_uint64)), len(off) - 1


def _results(arr) -> List[FitResult]:
    return [FitResult(r.theta_hat, r.sigma2, int(r.n), r.loglik, int(r.iterations), bool(r.converged), int(r.status))
            for r in arr]


# ------------------------------------------------------------- pseudo_obs
def validate_data(X: DataMatrix) -> None:  # pseudo_obs.hpp:30-37
    if len(X.col1) != len(X.col2):
        raise ValueError("data matrix: columns differ in length")
    if X.rows() < 2:
        raise ValueError("data matrix: need at least 2 rows")


def normalized_ranks(X: DataMatrix, segments: Optional[Sequence[int]] = None, ctx: Context = None) -> PseudoSample:
    """pseudo_obs.hpp:71-77; `segments` (offsets) ranks each block locally."""
    validate_data(X)
    ctx = ctx or default_context()
    c1, c2 = _f64(X.col1), _f64(X.col2)
    n = len(c1)
    u1, u2 = _like(c1, n), _like(c2, n)
    off, offp, k = _offsets(n, segments)
    p1, _k1 = _ptr(c1)
    p2, _k2 = _ptr(c2)
    q1, _k3 = _ptr(u1)
    q2, _k4 = _ptr(u2)
    ctx.check(ctx.lib.pcb_normalized_ranks(ctx.ptr, p1, p2, n, offp, k, q1, q2))
    return PseudoSample(u1, u2)


# ------------------------------------------------------------ estimator
def _check_theta(family, theta):  # copula.hpp:47-55
    t = float(theta)
    ok = np.isfinite(t) and ((family == 0 and -1.0 < t < 1.0) or (family == 1 and t != 0.0)
                             or (family == 2 and t >= 1.0))
    if not ok:
        raise DomainError(f"theta={t} outside the domain of the {CopulaFamily(family).name.lower()} copula")


def pseudo_loglik(family, theta, U: PseudoSample, segments=None, ctx: Context = None):
    """SPEC.md:207-215. Scalar theta -> float; per-segment thetas -> array."""
    ctx = ctx or default_context()
    u1, u2 = _f64(U.u1), _f64(U.u2)
    if len(u1) != len(u2):
        raise ValueError("pseudo sample: columns differ in length")
    n = len(u1)
    off, offp, k = _offsets(n, segments)
    th = np.broadcast_to(np.asarray(theta, np.float64), (k,)).copy()
    for t in th:
        _check_theta(int(family), t)
    out = np.empty(k, np.float64)
    p1, _a = _ptr(u1)
    p2, _b = _ptr(u2)
    ctx.check(ctx.lib.pcb_pseudo_loglik(ctx.ptr, int(family), th.ctypes.data, p1, p2, n, offp, k, out.ctypes.data))
    return float(out[0]) if segments is None else out


def fit(family, U: PseudoSample, precision=Precision.fp64, segments=None, ctx: Context = None):
    """SPEC.md:216-224 (sigma2 filled by asymptotic_variance).
    Returns one FitResult, or a list when `segments` is given."""
    ctx = ctx or default_context()
    u1, u2 = _f64(U.u1), _f64(U.u2)
    if len(u1) != len(u2):
        raise ValueError("pseudo sample: columns differ in length")
    n = len(u1)
    off, offp, k = _offsets(n, segments)
    out = (L.FitResultC * k)()
    p1, _a = _ptr(u1)
    p2, _b = _ptr(u2)
    ctx.check(ctx.lib.pcb_fit(ctx.ptr, int(family), int(precision), p1, p2, n, offp, k, C.addressof(out)))
    res = _results(out)
    return res[0] if segments is None else res


def asymptotic_variance(family, theta_hat, U: PseudoSample, segments=None, ctx: Context = None):
    """v^2/n; DomainError if I-hat <= 0."""
    ctx = ctx or default_context()
    u1, u2 = _f64(U.u1), _f64(U.u2)
    n = len(u1)
    off, offp, k = _offsets(n, segments)
    th = np.broadcast_to(np.asarray(theta_hat, np.float64), (k,)).copy()
    for t in th:
        _check_theta(int(family), t)
    out = np.empty(k, np.float64)
    p1, _a = _ptr(u1)
    p2, _b = _ptr(u2)
    ctx.check(ctx.lib.pcb_asymptotic_variance(ctx.ptr, int(family), th.ctypes.data, p1, p2, n, offp, k,
                                              out.ctypes.data))
    return float(out[0]) if segments is None else out


# ------------------------------------------------------ parallel_combine
def partition(X_or_rows, M: int, scheme=Scheme.Contiguous) -> Partition:
    """SPEC.md:275-283 (offsets; Strided offsets index the strided row order)."""
    n = X_or_rows.rows() if hasattr(X_or_rows, "rows") else int(X_or_rows)
    if M < 1:
        raise ValueError("partition: need M >= 1")
    off = np.zeros(M + 1, np.uint64)
    rc = L.load().pcb_partition(n, M, int(scheme), off.ctypes.data_as(C.POINTER(C.c_uint64)))
    if rc != L.PCB_OK:
        raise ValueError("partition: block below the 30-row floor")
    return Partition(off, Scheme(scheme))


def combine(results: Sequence[FitResult], ctx: Context = None) -> CombinedResult:
    """SPEC.md:284-292, on device."""
    k = len(results)
    if k == 0:
        raise ValueError("combine: empty input")
    ctx = ctx or default_context()
    arr = (L.FitResultC * k)()
    for i, r in enumerate(results):
        arr[i] = L.FitResultC(r.theta_hat, r.sigma2, r.loglik, r.n, r.iterations, int(r.converged),
                              int(getattr(r, "status", 0)), 0)
    w = np.zeros(k, np.float64)
    out = L.CombinedC()
    ctx.check(ctx.lib.pcb_combine(ctx.ptr, C.addressof(arr), k, w.ctypes.data, C.byref(out)))
    return CombinedResult(out.theta_combined, list(results), w, 0.0, int(out.blocks_used))


def fit_blocks(family, X: DataMatrix, segments, precision=Precision.fp64, ctx: Context = None) -> List[FitResult]:
    """One shard of fit_parallel: per block ranks -> fit -> variance."""
    ctx = ctx or default_context()
    c1, c2 = _f64(X.col1), _f64(X.col2)
    n = len(c1)
    off, offp, k = _offsets(n, segments)
    out = (L.FitResultC * k)()
    p1, _a = _ptr(c1)
    p2, _b = _ptr(c2)
    ctx.check(ctx.lib.pcb_fit_blocks(ctx.ptr, int(family), int(precision), p1, p2, n, offp, k, C.addressof(out)))
    return _results(out)


def fit_parallel(family, X: DataMatrix, M: int, workers: Optional[int] = None, scheme=Scheme.Contiguous,
                 precision=Precision.fp64, ctx: Context = None) -> CombinedResult:
    """SPEC.md:293-301. `workers` is accepted for signature compatibility:
    blocks run on the GPU's SMs (the result is identical for any value)."""
    validate_data(X)
    if M < 1:
        raise ValueError("partition: need M >= 1")
    ctx = ctx or default_context()
    c1, c2 = _f64(X.col1), _f64(X.col2)
    n = len(c1)
    per = (L.FitResultC * M)()
    w = np.zeros(M, np.float64)
    out = L.CombinedC()
    p1, _a = _ptr(c1)
    p2, _b = _ptr(c2)
    ctx.check(ctx.lib.pcb_fit_parallel(ctx.ptr, int(family), int(precision), p1, p2, n, M, int(scheme),
                                       C.addressof(per), w.ctypes.data, C.byref(out)))
    return CombinedResult(out.theta_combined, _results(per), w, out.wall_clock_per_block, int(out.blocks_used),
                          ctx.stage_times())


def sample_matrix(family, theta, n_total: int, n_blocks: int = 1, first_block: int = 0, last_block: int = None,
                  base_seed: int = BASE_SEED, device_out: bool = False, ctx: Context = None) -> DataMatrix:
    """Synthetic input on device (copula.hpp:359-423 transforms over
    counter-based splitmix64 streams)."""
    ctx = ctx or default_context()
    _check_theta(int(family), theta)
    last = n_blocks if last_block is None else last_block
    q = n_total // n_blocks
    rows = (n_total if last == n_blocks else last * q) - first_block * q
    if device_out:
        import torch
        c1 = torch.empty(rows, dtype=torch.float64, device=f"cuda:{ctx.device}")
        c2 = torch.empty(rows, dtype=torch.float64, device=f"cuda:{ctx.device}")
        p1, p2 = c1.data_ptr(), c2.data_ptr()
    else:
        c1 = np.empty(rows, np.float64)
        c2 = np.empty(rows, np.float64)
        p1, p2 = c1.ctypes.data, c2.ctypes.data
    ctx.check(ctx.lib.pcb_sample(ctx.ptr, int(family), float(theta), n_total, n_blocks, first_block, last,
                                 base_seed, p1, p2))
    return DataMatrix(c1, c2)
