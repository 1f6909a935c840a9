"""Copula CDF and dependence measures (copula.hpp:273-290,
normal.hpp:84-166) through the C-ABI: the CDF (Gaussian via the bivariate
normal CDF) and the model's Spearman rho on device, the empirical Kendall
tau of each block's first rows on device (the fit's SPEC init),
and the closed-form model Kendall tau / inverse_tau (host scalars).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from .parcop import Context, DomainError, _f64, _like, _offsets, _ptr, default_context
from . import _lib as L


def cdf(family, theta: float, u, v, ctx: Context = None) -> np.ndarray:
    """C(u, v; theta) at every point (copula.hpp:273-290)."""
    ctx = ctx or default_context()
    u, v = _f64(u), _f64(v)
    if len(u) != len(v):
        raise ValueError("cdf: u and v differ in length")
    out = _like(u, len(u))
    (pu, ku), (pv, kv), (po, ko) = _ptr(u), _ptr(v), _ptr(out)
    ctx.check(ctx.lib.pcb_cdf(ctx.ptr, int(family), float(theta), pu, pv, len(u), po))
    return out


def spearman_rho(family, theta: float, quad_nodes: int = 200, ctx: Context = None) -> float:
    """Model Spearman rho = 12 int C - 3 by the tensor Gauss-Legendre rule."""
    ctx = ctx or default_context()
    r = C.c_double()
    ctx.check(ctx.lib.pcb_spearman_rho(ctx.ptr, int(family), float(theta), int(quad_nodes), C.byref(r)))
    return r.value


def empirical_kendall_tau(u1, u2, segments: Optional[Sequence[int]] = None, m_max: int = 5000,
                          ctx: Context = None) -> np.ndarray:
    """Kendall tau of each segment's first min(n_m, m_max) rows; rank-invariant, so raw
    columns or pseudo-observations give the same value."""
    ctx = ctx or default_context()
    u1, u2 = _f64(u1), _f64(u2)
    n = len(u1)
    off, offp, k = _offsets(n, segments)
    out = np.zeros(k, np.float64)
    (p1, k1), (p2, k2) = _ptr(u1), _ptr(u2)
    ctx.check(ctx.lib.pcb_kendall_tau(ctx.ptr, p1, p2, n, offp, k, int(m_max), out.ctypes.data))
    return out


def kendall_tau(family, theta: float) -> float:
    """Model Kendall tau: Gaussian (2/pi) asin t, Gumbel 1 - 1/t, Frank 1 - 4/t (1 - D1(t))."""
    t = C.c_double()
    rc = L.load().pcb_model_kendall_tau(int(family), float(theta), C.byref(t))
    if rc == L.PCB_E_DOMAIN:
        raise DomainError("theta outside the family domain")
    if rc:
        raise ValueError("kendall_tau: bad family")
    return t.value


def inverse_tau(family, tau: float) -> float:
    """closed form (Gaussian, Gumbel), bisection to ~1e-12 (Frank)."""
    t = C.c_double()
    rc = L.load().pcb_inverse_tau(int(family), float(tau), C.byref(t))
    if rc == L.PCB_E_DOMAIN:
        raise DomainError("tau unattainable for this family")
    if rc:
        raise ValueError("inverse_tau: bad arguments")
    return t.value
