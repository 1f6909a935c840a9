"""ctypes binding of the C-ABI in include/parcop_b200.h (libparcop_b200.so).

The shared library is built in-tree by __graft_entry__.build() (nvcc,
sm_100a only). There is deliberately no fallback: if the library is missing
or no sm_100 device is usable, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# PCB_LIB_PATH selects an alternative in-tree build (kernel experiments)
LIB_PATH = os.environ.get("PCB_LIB_PATH") or os.path.join(HERE, "libparcop_b200.so")

# Every symbol include/parcop_b200.h declares (tests check the export table).
SYMBOLS = (
    "pcb_create", "pcb_create_multi", "pcb_device_count", "pcb_destroy", "pcb_last_error", "pcb_abi_version", "pcb_set_stream", "pcb_launch_count",
    "pcb_stage_times", "pcb_rank_paths", "pcb_trim", "pcb_normalized_ranks", "pcb_pseudo_loglik", "pcb_fit",
    "pcb_asymptotic_variance", "pcb_partition", "pcb_combine", "pcb_fit_blocks", "pcb_fit_parallel", "pcb_sample",
    "pcb_measure_fp64_peak", "pcb_rel_error", "pcb_cdf", "pcb_spearman_rho", "pcb_kendall_tau",
    "pcb_model_kendall_tau", "pcb_inverse_tau",
)

PCB_OK, PCB_E_INVALID, PCB_E_DOMAIN, PCB_E_CONVERGENCE, PCB_E_CUDA = 0, 2, 3, 4, 5


class FitResultC(C.Structure):
    """pcb_fit_result (SPEC.md:200-204 FitResult)."""

    _fields_ = [
        ("theta_hat", C.c_double),
        ("sigma2", C.c_double),
        ("loglik", C.c_double),
        ("n", C.c_uint64),
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("status", C.c_int32),
        ("reserved", C.c_int32),
    ]


class CombinedC(C.Structure):
    """pcb_combined (SPEC.md:268-272 CombinedResult scalars)."""

    _fields_ = [("theta_combined", C.c_double), ("total_weight", C.c_double), ("blocks_used", C.c_uint64),
                ("wall_clock_per_block", C.c_double)]


_lib = None


def load():
    """Load libparcop_b200.so (raises if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the CUDA library is the only implementation; there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, d, u64, i = C.c_void_p, C.c_double, C.c_uint64, C.c_int
    P = C.POINTER
    sig = {
        "pcb_create": ([i], vp),
        "pcb_create_multi": ([P(i), i], vp),
        "pcb_device_count": ([vp], i),
        "pcb_destroy": ([vp], None),
        "pcb_last_error": ([vp], C.c_char_p),
        "pcb_abi_version": ([], i),
        "pcb_set_stream": ([vp, vp], i),
        "pcb_launch_count": ([vp], u64),
        "pcb_stage_times": ([vp, P(d), i], i),
        "pcb_rank_paths": ([vp, P(u64)], i),
        "pcb_trim": ([vp], i),
        "pcb_normalized_ranks": ([vp, vp, vp, u64, P(u64), u64, vp, vp], i),
        "pcb_pseudo_loglik": ([vp, i, vp, vp, vp, u64, P(u64), u64, vp], i),
        "pcb_fit": ([vp, i, i, vp, vp, u64, P(u64), u64, vp], i),
        "pcb_asymptotic_variance": ([vp, i, vp, vp, vp, u64, P(u64), u64, vp], i),
        "pcb_partition": ([u64, u64, i, P(u64)], i),
        "pcb_combine": ([vp, vp, u64, vp, P(CombinedC)], i),
        "pcb_fit_blocks": ([vp, i, i, vp, vp, u64, P(u64), u64, vp], i),
        "pcb_fit_parallel": ([vp, i, i, vp, vp, u64, u64, i, vp, vp, P(CombinedC)], i),
        "pcb_sample": ([vp, i, d, u64, u64, u64, u64, u64, vp, vp], i),
        "pcb_measure_fp64_peak": ([vp, P(d)], i),
        "pcb_rel_error": ([vp, i, d, d, i, P(d), P(d)], i),
        "pcb_cdf": ([vp, i, d, vp, vp, u64, vp], i),
        "pcb_spearman_rho": ([vp, i, d, i, P(d)], i),
        "pcb_kendall_tau": ([vp, vp, vp, u64, P(u64), u64, u64, vp], i),
        "pcb_model_kendall_tau": ([i, d, P(d)], i),
        "pcb_inverse_tau": ([i, d, P(d)], i),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L
