"""B200-native divide-and-combine copula MPL fit (arXiv:1609.05530 hot path).

The product is libparcop_b200.so (CUDA, sm_100a) behind the C-ABI in
include/parcop_b200.h; this package is its Python mirror of the reference's
`parcop::` interface (see parcop.py).
"""
from .parcop import (  # noqa: F401
    BASE_SEED, CombinedResult, Context, ConvergenceError, CopulaFamily, CudaError, DataMatrix, DomainError,
    FitResult, Partition, Precision, PseudoSample, Scheme, asymptotic_variance, combine, default_context,
    family_from_string, fit, fit_blocks, fit_parallel, normalized_ranks, partition, pseudo_loglik, sample_matrix,
    validate_data,
)
from .study import (  # noqa: F401,E402
    ReplicateRow, SimConfig, SimReport, est_bias, est_mse, mix_seed, rel_error, rel_l1, rel_l2, run_study,
)
from .dependence import cdf, empirical_kendall_tau, inverse_tau, kendall_tau, spearman_rho  # noqa: F401,E402
