"""CPU: the oracle restatement against the reference headers compiled in
place (oracle/_ref/libparcop_ref.so) on fresh random inputs: ranks
bit-identical, per-point values ulp-level, fits identical to 1e-13."""
import numpy as np
import pytest


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_ranks_bit_identical(orc, ref, seed):
    rng = np.random.default_rng(seed)
    for x in (rng.standard_normal(3000), np.round(rng.standard_normal(3000), 1), rng.integers(0, 5, 500) * 1.0,
              np.r_[0.0, -0.0, rng.uniform(-1, 1, 100)]):
        assert np.array_equal(orc.rank_column(x), ref.rank_column(x))


@pytest.mark.parametrize("fam,theta", [(0, 0.4), (0, -0.9), (1, 5.0), (1, -8.0), (1, 0.3), (2, 1.0), (2, 2.5),
                                       (2, 15.0)])
def test_point_values(orc, ref, fam, theta):
    rng = np.random.default_rng(int(abs(theta) * 10) + fam)
    u, v = rng.uniform(1e-6, 1 - 1e-6, (2, 400))
    a, b = orc.derivs(fam, theta, u, v), ref.derivs(fam, theta, u, v)
    assert np.all(np.abs(a - b) <= 1e-12 * np.maximum(np.abs(b), 1.0))
    la, lb = orc.log_pdf(fam, theta, u, v), ref.log_pdf(fam, theta, u, v)
    assert np.all(np.abs(la - lb) <= 1e-12 * np.maximum(np.abs(lb), 1.0))


@pytest.mark.parametrize("fam,theta", [(0, 0.5), (1, 5.0), (2, 2.0)])
def test_fit_blocks_identical(orc, ref, fam, theta):
    off = orc.partition(60000, 6)
    c1, c2 = orc.sample_blocks(fam, theta, 60000, 6, off, 0, 6)
    a = orc.fit_blocks(fam, c1, c2, off)
    b = ref.fit_blocks(fam, c1, c2, off)
    for x, y in zip(a, b):
        assert abs(x.theta_hat - y.theta_hat) <= 1e-13 * abs(y.theta_hat)
        assert abs(x.sigma2 - y.sigma2) <= 1e-12 * abs(y.sigma2)
