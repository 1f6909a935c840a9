"""CDF and dependence measures (SPEC.md:97-122,
copula.hpp:273-290, normal.hpp:84-166).

CPU: the oracle's restated cdf / bvn_cdf / Spearman quadrature pinned bit for
bit against the reference's own (oracle/_ref); the SPEC's worked examples for
the model Kendall tau, Spearman rho and inverse_tau (host scalars of the
product library, no device needed).
GPU: pcb_cdf and pcb_spearman_rho against the oracle; the device's empirical
Kendall tau equal to the oracle's (integer counting) on tie-free, tied and
ragged blocks.
"""
import numpy as np
import pytest

import paper_1609_05530_b200 as pcb

MODELS = [(0, 0.3), (0, -0.95), (0, 0.97), (0, 0.0), (1, 5.0), (1, -3.0), (1, 0.2), (2, 2.0), (2, 1.0), (2, 8.0)]


def _pts(n=3000, seed=1):
    g = np.random.default_rng(seed)
    u, v = g.random(n), g.random(n)
    u[:4] = [1e-14, 1.0 - 1e-14, 0.5, 1e-300]  # clamp corners (copula.hpp:88-92)
    v[:4] = [0.5, 1e-14, 1.0 - 1e-14, 0.25]
    return u, v


@pytest.mark.parametrize("fam,t", MODELS)
def test_oracle_cdf_matches_reference(orc, ref, fam, t):
    u, v = _pts()
    assert np.array_equal(orc.cdf(fam, t, u, v), ref.cdf(fam, t, u, v))


def test_oracle_spearman_matches_reference(orc, ref):
    for fam, t in [(0, 0.3), (1, 5.0), (2, 5.0), (1, -2.0)]:
        assert orc.spearman_rho(fam, t, 64) == ref.spearman_rho(fam, t, 64)


def test_spec_dependence_examples(orc):  # SPEC.md:101-121 (PAPER §2.5 pairs)
    assert round(pcb.kendall_tau(0, 0.3), 2) == 0.19
    assert round(pcb.kendall_tau(1, 5.0), 2) == 0.46
    assert pcb.kendall_tau(2, 5.0) == pytest.approx(0.80, abs=1e-15)
    assert round(orc.spearman_rho(0, 0.3, 200), 2) == 0.29
    assert round(orc.spearman_rho(1, 5.0, 200), 2) == 0.64
    assert round(orc.spearman_rho(2, 5.0, 200), 2) == 0.94
    assert pcb.inverse_tau(2, 0.8) == pytest.approx(5.0, rel=1e-15)
    assert pcb.inverse_tau(0, 0.0) == 0.0
    assert pcb.inverse_tau(1, 0.46) == pytest.approx(5.0, abs=0.1)
    for fam, t in [(0, 0.6), (1, -4.0), (1, 12.0), (2, 3.3)]:  # kendall_tau(inverse_tau(tau)) = tau to 1e-8
        assert pcb.kendall_tau(fam, pcb.inverse_tau(fam, pcb.kendall_tau(fam, t))) == \
            pytest.approx(pcb.kendall_tau(fam, t), abs=1e-8)
        assert pcb.inverse_tau(fam, pcb.kendall_tau(fam, t)) == pytest.approx(t, rel=1e-8)
    with pytest.raises(pcb.DomainError):
        pcb.inverse_tau(2, -0.2)  # unattainable
    with pytest.raises(pcb.DomainError):
        pcb.kendall_tau(2, 0.5)


def test_oracle_kendall_spec_pairs(orc):  # inverse_tau of the oracle = the product's host scalar
    for fam, tau in [(0, 0.19), (1, 0.46), (1, -0.3), (2, 0.8)]:
        assert orc.inverse_tau(fam, tau) == pytest.approx(pcb.inverse_tau(fam, tau), rel=1e-8)


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("fam,t", MODELS)
def test_device_cdf_parity(ctx, orc, fam, t):
    u, v = _pts(20000, 3)
    d, o = pcb.cdf(fam, t, u, v, ctx=ctx), orc.cdf(fam, t, u, v)
    assert np.all(np.abs(d - o) <= 1e-12 + 1e-9 * np.abs(o))
    assert np.all((d >= 0.0) & (d <= 1.0))


@pytest.mark.gpu
def test_device_spearman_parity(ctx, orc):
    for fam, t in [(0, 0.3), (0, -0.8), (1, 5.0), (1, -2.0), (2, 5.0), (2, 1.0)]:
        assert pcb.spearman_rho(fam, t, 64, ctx=ctx) == pytest.approx(orc.spearman_rho(fam, t, 64), abs=1e-11)
    assert round(pcb.spearman_rho(2, 5.0, 200, ctx=ctx), 2) == 0.94


@pytest.mark.gpu
def test_device_empirical_kendall_equals_oracle(ctx, orc):
    X = pcb.sample_matrix(1, 5.0, 30000, 1, ctx=ctx)
    c1, c2 = np.asarray(X.col1), np.asarray(X.col2)
    c1[100:400] = 0.25  # ties in u1
    c2[300:700] = 0.75  # ties in u2
    off = [0, 6000, 13001, 30000]
    tau = pcb.empirical_kendall_tau(c1, c2, off, m_max=5000, ctx=ctx)
    for k in range(3):
        a, b = off[k], off[k + 1]
        m = min(5000, b - a)
        assert tau[k] == orc.kendall_tau(c1[a:b], c2[a:b], m)
    # rank invariance: raw columns and their pseudo-observations agree
    U = pcb.normalized_ranks(pcb.DataMatrix(c1, c2), off, ctx=ctx)
    assert np.array_equal(pcb.empirical_kendall_tau(U.u1, U.u2, off, ctx=ctx), tau)


@pytest.mark.gpu
@pytest.mark.parametrize("fam,theta", [(1, 5.0), (1, -3.0), (2, 2.0)])
def test_tau_init_same_root(ctx, orc, monkeypatch, fam, theta):
    """PCB_INIT=tau (the SPEC's start) reaches the same theta-hat as the default start."""
    X = pcb.sample_matrix(fam, theta, 60000, 6, ctx=ctx)
    off = [0, 10000, 20000, 30000, 40000, 50000, 60000]
    a = pcb.fit_blocks(fam, X, off, ctx=ctx)
    monkeypatch.setenv("PCB_INIT", "tau")
    b = pcb.fit_blocks(fam, X, off, ctx=ctx)
    want = orc.fit_blocks(fam, np.asarray(X.col1), np.asarray(X.col2), np.asarray(off, np.uint64))
    for x, y, w in zip(a, b, want):
        assert x.converged and y.converged
        assert abs(y.theta_hat - w.theta_hat) <= 1e-9 * abs(w.theta_hat)
        assert abs(y.sigma2 - w.sigma2) <= 1e-9 * abs(w.sigma2)
        assert abs(x.theta_hat - y.theta_hat) <= 1e-9 * abs(w.theta_hat)
