"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes bindings to the CPU oracle (liboracle.so: the SPEC/reference
restatement) and to oracle/_ref/libparcop_ref.so (the reference headers
compiled in place). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this module, and only as the
checker or the CPU baseline — never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libparcop_ref.so")

GAUSSIAN, FRANK, GUMBEL = 0, 1, 2
BASE_SEED = 0x160905530


class FitRecord(C.Structure):
    """oracle::FitRecord (mpl_driver.hpp) == SPEC.md:200-204 FitResult."""

    _fields_ = [
        ("theta_hat", C.c_double),
        ("sigma2", C.c_double),
        ("loglik", C.c_double),
        ("n", C.c_uint64),
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("status", C.c_int32),
        ("pad", C.c_int32),
    ]


_D = C.POINTER(C.c_double)
_U64 = C.POINTER(C.c_uint64)


def _dp(a):
    return a.ctypes.data_as(_D)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build(quiet=True):
    """Build liboracle.so (+ _ref when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


class Lib:
    """One of the two oracle shared libraries (prefix orc_ or ref_)."""

    def __init__(self, path, prefix):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.p = prefix
        L = self.lib
        f = lambda n: getattr(L, prefix + n)  # noqa: E731
        f("last_error").restype = C.c_char_p
        f("normalized_ranks").argtypes = [_D, _D, C.c_uint64, _D, _D]
        f("rank_column").argtypes = [_D, C.c_uint64, _D]
        f("log_pdf_vec").argtypes = [C.c_int, C.c_double, _D, _D, C.c_uint64, _D]
        f("derivs_vec").argtypes = [C.c_int, C.c_double, _D, _D, C.c_uint64, _D]
        f("pseudo_loglik").argtypes = [C.c_int, C.c_double, _D, _D, C.c_uint64, _D]
        f("fit").argtypes = [C.c_int, _D, _D, C.c_uint64, C.POINTER(FitRecord)]
        f("asymptotic_variance").argtypes = [C.c_int, C.c_double, _D, _D, C.c_uint64, C.c_int, _D]
        f("fit_blocks").argtypes = [C.c_int, _D, _D, _U64, C.c_uint64, C.c_int, C.POINTER(FitRecord)]
        f("combine").argtypes = [C.POINTER(FitRecord), C.c_uint64, _D, _D, _U64]
        f("partition").argtypes = [C.c_uint64, C.c_uint64, _U64]
        f("kendall_tau").argtypes = [_D, _D, C.c_uint64, _D]
        f("inverse_tau").argtypes = [C.c_int, C.c_double, _D]
        f("debye1").argtypes = [C.c_double, _D]
        for n in ["normalized_ranks", "rank_column", "log_pdf_vec", "derivs_vec", "pseudo_loglik", "fit",
                  "asymptotic_variance", "fit_blocks", "combine", "partition", "kendall_tau",
                  "inverse_tau", "debye1"]:
            f(n).restype = C.c_int
        if prefix == "orc_":
            L.orc_sample_blocks.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_uint64, C.c_uint64, _U64,
                                            C.c_uint64, C.c_uint64, _D, _D, C.c_int]
            L.orc_sample_blocks.restype = C.c_int
            L.orc_mix_seed4.argtypes = [C.c_uint64] * 5
            L.orc_mix_seed4.restype = C.c_uint64
            L.orc_unit_draw.argtypes = [C.c_uint64, C.c_uint64]
            L.orc_unit_draw.restype = C.c_double
            L.orc_splitmix64.argtypes = [C.c_uint64]
            L.orc_splitmix64.restype = C.c_uint64
        else:
            L.ref_sample_matrix.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_uint64, _D, _D]
            L.ref_sample_matrix.restype = C.c_int
            L.ref_mix_seed4.argtypes = [C.c_uint64] * 5
            L.ref_mix_seed4.restype = C.c_uint64
            L.ref_splitmix64.argtypes = [C.c_uint64]
            L.ref_splitmix64.restype = C.c_uint64

    def _call(self, name, *args):
        rc = getattr(self.lib, self.p + name)(*args)
        if rc != 0:
            msg = getattr(self.lib, self.p + "last_error")().decode()
            raise OracleError(rc, msg)

    # ------------------------------------------------------------------ API
    def normalized_ranks(self, c1, c2):
        c1 = np.ascontiguousarray(c1, np.float64)
        c2 = np.ascontiguousarray(c2, np.float64)
        u1 = np.empty_like(c1)
        u2 = np.empty_like(c2)
        self._call("normalized_ranks", _dp(c1), _dp(c2), len(c1), _dp(u1), _dp(u2))
        return u1, u2

    def rank_column(self, x):
        x = np.ascontiguousarray(x, np.float64)
        u = np.empty_like(x)
        self._call("rank_column", _dp(x), len(x), _dp(u))
        return u

    def log_pdf(self, fam, t, u, v):
        u = np.ascontiguousarray(np.atleast_1d(u), np.float64)
        v = np.ascontiguousarray(np.atleast_1d(v), np.float64)
        out = np.empty_like(u)
        self._call("log_pdf_vec", fam, t, _dp(u), _dp(v), len(u), _dp(out))
        return out

    def derivs(self, fam, t, u, v):
        u = np.ascontiguousarray(np.atleast_1d(u), np.float64)
        v = np.ascontiguousarray(np.atleast_1d(v), np.float64)
        out = np.empty((len(u), 4), np.float64)
        self._call("derivs_vec", fam, t, _dp(u), _dp(v), len(u), _dp(out))
        return out

    def pseudo_loglik(self, fam, t, u1, u2):
        u1 = np.ascontiguousarray(u1, np.float64)
        u2 = np.ascontiguousarray(u2, np.float64)
        out = C.c_double()
        self._call("pseudo_loglik", fam, t, _dp(u1), _dp(u2), len(u1), C.byref(out))
        return out.value

    def fit(self, fam, u1, u2):
        u1 = np.ascontiguousarray(u1, np.float64)
        u2 = np.ascontiguousarray(u2, np.float64)
        r = FitRecord()
        self._call("fit", fam, _dp(u1), _dp(u2), len(u1), C.byref(r))
        return r

    def asymptotic_variance(self, fam, t, u1, u2, naive=False):
        u1 = np.ascontiguousarray(u1, np.float64)
        u2 = np.ascontiguousarray(u2, np.float64)
        out = C.c_double()
        self._call("asymptotic_variance", fam, t, _dp(u1), _dp(u2), len(u1), int(naive), C.byref(out))
        return out.value

    def fit_blocks(self, fam, c1, c2, offsets, workers=None):
        c1 = np.ascontiguousarray(c1, np.float64)
        c2 = np.ascontiguousarray(c2, np.float64)
        off = np.ascontiguousarray(offsets, np.uint64)
        k = len(off) - 1
        out = (FitRecord * k)()
        w = workers or os.cpu_count() or 1
        self._call("fit_blocks", fam, _dp(c1), _dp(c2), off.ctypes.data_as(_U64), k, w, out)
        return out

    def combine(self, records):
        k = len(records)
        arr = (FitRecord * k)(*records) if not isinstance(records, C.Array) else records
        tc = C.c_double()
        w = np.zeros(k, np.float64)
        used = C.c_uint64()
        self._call("combine", arr, k, C.byref(tc), _dp(w), C.byref(used))
        return tc.value, w, used.value

    def partition(self, n, m):
        off = np.zeros(m + 1, np.uint64)
        self._call("partition", n, m, off.ctypes.data_as(_U64))
        return off

    def kendall_tau(self, u1, u2, m=None):
        u1 = np.ascontiguousarray(u1, np.float64)
        u2 = np.ascontiguousarray(u2, np.float64)
        out = C.c_double()
        self._call("kendall_tau", _dp(u1), _dp(u2), m or len(u1), C.byref(out))
        return out.value

    def inverse_tau(self, fam, tau):
        out = C.c_double()
        self._call("inverse_tau", fam, tau, C.byref(out))
        return out.value

    def debye1(self, x):
        out = C.c_double()
        self._call("debye1", x, C.byref(out))
        return out.value

    def cdf(self, fam, t, u, v):
        u = np.ascontiguousarray(np.atleast_1d(u), np.float64)
        v = np.ascontiguousarray(np.atleast_1d(v), np.float64)
        out = np.empty_like(u)
        self._call("cdf_vec", fam, C.c_double(t), _dp(u), _dp(v), len(u), _dp(out))
        return out

    def spearman_rho(self, fam, t, nodes=200):
        out = C.c_double()
        self._call("spearman_rho", fam, C.c_double(t), nodes, C.byref(out))
        return out.value

    def rel_error(self, fam, ta, tb, nodes=200):
        """(rel_l1, rel_l2) of SPEC.md:362-374 by the tensor Gauss-Legendre rule."""
        out = np.zeros(2, np.float64)
        self._call("rel_error", fam, C.c_double(ta), C.c_double(tb), nodes, _dp(out), None)
        return float(out[0]), float(out[1])

    # ---- generators
    def sample_blocks(self, fam, theta, n_total, k, offsets, first, last, base_seed=BASE_SEED, workers=None):
        assert self.p == "orc_"
        off = np.ascontiguousarray(offsets, np.uint64)
        rows = int(off[last] - off[first])
        c1 = np.empty(rows, np.float64)
        c2 = np.empty(rows, np.float64)
        rc = self.lib.orc_sample_blocks(fam, theta, n_total, k, base_seed, off.ctypes.data_as(_U64), first, last,
                                        _dp(c1), _dp(c2), workers or os.cpu_count() or 1)
        if rc != 0:
            raise OracleError(rc, "sample_blocks")
        return c1, c2

    def sample_matrix(self, fam, theta, n, seed):
        assert self.p == "ref_"
        c1 = np.empty(n, np.float64)
        c2 = np.empty(n, np.float64)
        self._call("sample_matrix", fam, theta, n, seed, _dp(c1), _dp(c2))
        return c1, c2


_cache = {}


def oracle_lib() -> Lib:
    if "orc" not in _cache:
        if not os.path.exists(ORACLE_SO):
            build()
        _cache["orc"] = Lib(ORACLE_SO, "orc_")
    return _cache["orc"]


def ref_lib() -> Lib | None:
    """The compiled reference, or None where it was never built."""
    if "ref" not in _cache:
        _cache["ref"] = Lib(REF_SO, "ref_") if os.path.exists(REF_SO) else None
    return _cache["ref"]
