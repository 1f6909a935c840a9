"""CPU: the oracle (oracle/liboracle.so) pinned against the committed golden
fixtures made by the compiled reference (tests/golden/make_golden.py) and
against the SPEC's own known answers and test oracles (SPEC.md §4 table in
SURVEY.md): rank examples, combine/partition examples, finite-difference
derivative oracles, the brute-force grid-argmax optimizer oracle, the O(n^2)
variance definition, and the structural invariants."""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


# ------------------------------------------------------------ golden pins
def test_points_match_reference(orc):
    pts = json.load(open(os.path.join(GOLD, "points.json")))
    worst = 0.0
    for p in pts:
        lp = orc.log_pdf(p["family"], p["theta"], p["u"], p["v"])[0]
        d = orc.derivs(p["family"], p["theta"], p["u"], p["v"])[0]
        for got, key in zip([lp, *d], ["log_pdf", "score", "hess", "cross1", "cross2"]):
            want = p[key]
            err = abs(got - want) / max(abs(want), 1.0)
            worst = max(worst, err)
            assert err <= 1e-12, (p, key, got, want)


def test_ranks_match_reference_vectors(orc):
    cases = json.load(open(os.path.join(GOLD, "ranks_small.json")))
    for name, c in cases.items():
        got = orc.rank_column(np.array(c["x"], np.float64))
        assert np.array_equal(got, np.array(c["u"])), name


def test_c1_fixture_matches_reference(orc):
    data = np.load(os.path.join(GOLD, "c1_gaussian_rho05_n1e4.npz"))
    meta = json.load(open(os.path.join(GOLD, "c1_expected.json")))
    off = orc.partition(10000, 10)
    recs = orc.fit_blocks(0, data["col1"], data["col2"], off)
    for r, w in zip(recs, meta["per_block"]):
        assert r.converged
        assert rel(r.theta_hat, w["theta_hat"]) <= 1e-12
        assert rel(r.sigma2, w["sigma2"]) <= 1e-12
        assert rel(r.loglik, w["loglik"]) <= 1e-12
    tc, _, used = orc.combine(recs)
    assert used == 10 and rel(tc, meta["theta_combined"]) <= 1e-12


# ---------------------------------------------------- SPEC known answers
def test_spec_rank_examples(orc):
    assert np.array_equal(orc.rank_column([3.1, 1.2, 7.5]), [0.5, 0.25, 0.75])
    assert np.array_equal(orc.rank_column([1.0, 1.0, 2.0]), [0.375, 0.375, 0.75])
    x = np.random.default_rng(0).standard_normal(200)
    assert np.array_equal(orc.rank_column(x), orc.rank_column(np.exp(x)))  # monotone invariance
    u = orc.rank_column(x)
    assert np.array_equal(orc.rank_column(u), u)  # idempotence without ties


def test_spec_combine_examples(orc):
    from oracle.oracle import FitRecord
    mk = lambda t, s: FitRecord(t, s, 0.0, 100, 3, 1, 0, 0)  # noqa: E731
    assert orc.combine([mk(0.3, 1.0), mk(0.3, 2.0), mk(0.3, 9.0)])[0] == 0.3  # exact (anchored Eq. 15)
    assert orc.combine([mk(1.99112997922569, 2.0584161e-4)])[0] == 1.99112997922569  # M = 1
    assert orc.combine([mk(0.2, 2.0), mk(0.4, 2.0)])[0] == pytest.approx(0.3, rel=1e-15)
    assert orc.combine([mk(0.2, 1.0), mk(0.4, 4.0)])[0] == pytest.approx(0.24, rel=1e-15)
    bad = FitRecord(0.9, 1.0, 0.0, 100, 3, 0, 1, 0)
    tc, w, used = orc.combine([mk(0.2, 1.0), bad])
    assert used == 1 and tc == 0.2 and w[1] == 0.0


def test_spec_partition_examples(orc):
    assert list(orc.partition(200000, 100)[:3]) == [0, 2000, 4000]
    with pytest.raises(Exception):
        orc.partition(10, 3)  # below the 30-row floor
    off = orc.partition(100, 3)
    assert list(np.diff(off)) == [33, 33, 34]


def test_spec_score_gaussian_zero(orc):
    assert orc.derivs(0, 0.0, 0.5, 0.5)[0, 0] == 0.0


@pytest.mark.parametrize("fam,theta", [(0, 0.3), (0, -0.7), (1, 5.0), (1, -3.0), (2, 2.0), (2, 5.0)])
def test_fd_derivative_oracles(orc, fam, theta):
    rng = np.random.default_rng(fam * 10 + int(abs(theta)))
    uv = rng.uniform(0.05, 0.95, (50, 2))
    h = 1e-5
    d = orc.derivs(fam, theta, uv[:, 0], uv[:, 1])
    lp = lambda t: orc.log_pdf(fam, t, uv[:, 0], uv[:, 1])  # noqa: E731
    sc = lambda t: orc.derivs(fam, t, uv[:, 0], uv[:, 1])[:, 0]  # noqa: E731
    fd_s = (lp(theta + h) - lp(theta - h)) / (2 * h)
    fd_h = (sc(theta + h) - sc(theta - h)) / (2 * h)
    assert np.all(np.abs(d[:, 0] - fd_s) <= 1e-4 * np.maximum(np.abs(d[:, 0]), 1e-2))
    assert np.all(np.abs(d[:, 1] - fd_h) <= 1e-3 * np.maximum(np.abs(d[:, 1]), 1e-2))
    hu = 1e-6
    c1 = (orc.derivs(fam, theta, uv[:, 0] + hu, uv[:, 1])[:, 0] - orc.derivs(fam, theta, uv[:, 0] - hu, uv[:, 1])[:, 0]) / (2 * hu)
    c2 = (orc.derivs(fam, theta, uv[:, 0], uv[:, 1] + hu)[:, 0] - orc.derivs(fam, theta, uv[:, 0], uv[:, 1] - hu)[:, 0]) / (2 * hu)
    assert np.all(np.abs(d[:, 2] - c1) <= 1e-3 * np.maximum(np.abs(d[:, 2]), 1e-1))
    assert np.all(np.abs(d[:, 3] - c2) <= 1e-3 * np.maximum(np.abs(d[:, 3]), 1e-1))


@pytest.mark.parametrize("fam,theta", [(0, 0.5), (1, 5.0), (2, 2.0)])
def test_grid_argmax_optimizer_oracle(orc, fam, theta):
    n = 2000
    for s in range(4):
        off = np.array([0, n], np.uint64)
        c1, c2 = orc.sample_blocks(fam, theta, n, 1, off, 0, 1, base_seed=1000 + s)
        u1, u2 = orc.normalized_ranks(c1, c2)
        r = orc.fit(fam, u1, u2)
        assert r.converged
        lo, hi = {0: (-0.999, 0.999), 1: (0.5, 15.0), 2: (1.0, 6.0)}[fam]
        grid = np.arange(lo, hi, 1e-3)
        if fam == 1:
            grid = grid[np.abs(grid) > 1e-6]
        ll = np.array([orc.pseudo_loglik(fam, t, u1, u2) for t in grid])
        assert abs(grid[np.argmax(ll)] - r.theta_hat) <= 2e-3


@pytest.mark.parametrize("fam,theta", [(0, 0.5), (1, 5.0), (2, 2.0), (1, -2.0)])
def test_variance_suffix_equals_naive(orc, fam, theta):  # SPEC.md:228 vs 246
    n = 1500
    off = np.array([0, n], np.uint64)
    c1, c2 = orc.sample_blocks(fam, theta, n, 1, off, 0, 1, base_seed=77)
    c1 = np.round(c1, 3)  # exercise ties in the W-term
    u1, u2 = orc.normalized_ranks(c1, c2)
    r = orc.fit(fam, u1, u2)
    a = orc.asymptotic_variance(fam, r.theta_hat, u1, u2)
    b = orc.asymptotic_variance(fam, r.theta_hat, u1, u2, naive=True)
    assert rel(a, b) <= 1e-12
    assert rel(a, r.sigma2) <= 1e-15


def test_variance_halves_when_n_doubles(orc):
    ratios = []
    for s in range(10):
        off = np.array([0, 8000], np.uint64)
        c1, c2 = orc.sample_blocks(0, 0.3, 8000, 1, off, 0, 1, base_seed=500 + s)
        r_half = orc.fit_blocks(0, c1[:4000], c2[:4000], [0, 4000])[0]
        r_full = orc.fit_blocks(0, c1, c2, [0, 8000])[0]
        ratios.append(r_full.sigma2 / r_half.sigma2)
    assert 0.4 <= np.mean(ratios) <= 0.6


# the Monte Carlo variance oracle, the only external
# calibration of the variance formula (the reference ships no variance code):
# over i.i.d. replicates at n = 5000, the mean reported sigma2 lies within 20%
# of the empirical variance of theta-hat. The SPEC says 200 replicates; the
# sampling error of a variance over 200 replicates is ~10% (one seed gave
# 1.26 for Frank), so this runs 1000 (error ~4.5%: the 20% bar is > 4 SE) —
# a stronger form of the same oracle. The SPEC names Gaussian 0.3 and Frank
# 5; Gumbel 2 is held to the same bar. Replicate m is block m of one seeded
# draw (independent per-block streams).
MC_CASES = [(0, 0.3), (1, 5.0), (2, 2.0)]


@pytest.mark.parametrize("fam,theta", MC_CASES)
def test_monte_carlo_variance_oracle(orc, fam, theta):
    reps, n = 1000, 5000
    off = np.arange(reps + 1, dtype=np.uint64) * np.uint64(n)
    c1, c2 = orc.sample_blocks(fam, theta, reps * n, reps, off, 0, reps, base_seed=0x5EC231)
    recs = orc.fit_blocks(fam, c1, c2, off)
    th = np.array([r.theta_hat for r in recs])
    s2 = np.array([r.sigma2 for r in recs])
    assert all(r.converged for r in recs)
    ratio = s2.mean() / th.var(ddof=1)
    assert 0.8 <= ratio <= 1.2, ratio
    assert abs(th.mean() - theta) <= 3.0 * np.sqrt(s2.mean() / reps)  # consistency


def test_invariants(orc):
    off = np.array([0, 3000], np.uint64)
    c1, c2 = orc.sample_blocks(0, 0.6, 3000, 1, off, 0, 1, base_seed=9)
    a = orc.fit_blocks(0, c1, c2, [0, 3000])[0]
    b = orc.fit_blocks(0, np.exp(5 * c1), np.log(c2), [0, 3000])[0]
    assert a.theta_hat == b.theta_hat and a.sigma2 == b.sigma2
    neg = orc.fit_blocks(0, -c1, c2, [0, 3000])[0]
    assert abs(abs(neg.theta_hat) - abs(a.theta_hat)) < 1e-6 and neg.theta_hat < 0
    # workers-invariance
    off = orc.partition(30000, 10)
    d1, d2 = orc.sample_blocks(2, 2.0, 30000, 10, off, 0, 10)
    r1 = orc.fit_blocks(2, d1, d2, off, workers=1)
    r8 = orc.fit_blocks(2, d1, d2, off, workers=8)
    assert [x.theta_hat for x in r1] == [x.theta_hat for x in r8]
    # M = 1 identity
    full = orc.fit_blocks(2, d1, d2, [0, 30000])[0]
    tc, _, _ = orc.combine([full])
    assert tc == full.theta_hat


def test_gumbel_independence_boundary(orc):
    off = np.array([0, 5000], np.uint64)
    hits = 0
    for s in range(6):
        c1, c2 = orc.sample_blocks(2, 1.0, 5000, 1, off, 0, 1, base_seed=300 + s)
        r = orc.fit_blocks(2, c1, c2, [0, 5000])[0]
        assert r.converged and 1.0 <= r.theta_hat < 1.05
        hits += r.theta_hat == 1.0
    assert hits >= 1


def test_counter_stream_is_splitmix(orc):
    # draw d of a stream = output d+1 of SplitMix64 seeded with seed
    seed = 12345
    state = seed
    for d in range(5):
        state = (state + 0x9E3779B97F4A7C15) & (2**64 - 1)
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        z ^= z >> 31
        assert orc.lib.orc_unit_draw(seed, d) == ((z >> 11) + 0.5) * 2.0**-53


def frank_cond_tol(theta_hat, base=1e-9, theta_c=0.03):
    """Parity tolerance for Frank estimates near 0: the reference's formulas
    (copula.hpp:147-172) cancel terms of size 1/t and 1/t^2, so any fp64
    evaluation carries ~eps/t^2 relative error below |t| ~ theta_c
    (tests/golden/make_frank_near_zero.py measures it against 60 digits)."""
    return base * max(1.0, (theta_c / max(abs(theta_hat), 1e-300)) ** 2)


def test_frank_near_zero_against_high_precision(orc):
    """A 240-row Frank block with estimate ~1e-3: the oracle (and, in
    test_gpu_parity, the device) against a 60-digit evaluation of the same
    estimator. Both fp64 evaluations sit ~1e-9 (theta) / ~1e-8 (sigma2) from
    the truth here, which bounds how closely they can agree."""
    inp = json.load(open(os.path.join(GOLD, "frank_near_zero_input.json")))
    hp = json.load(open(os.path.join(GOLD, "frank_near_zero_expected.json")))
    c1, c2 = np.asarray(inp["c1"]), np.asarray(inp["c2"])
    (rec,) = orc.fit_blocks(1, c1, c2, np.array([0, len(c1)], np.uint64))
    assert rec.converged
    assert rel(rec.theta_hat, hp["theta_hat"]) <= 3e-9, (rec.theta_hat, hp["theta_hat"])
    assert rel(rec.sigma2, hp["sigma2"]) <= 2e-8, (rec.sigma2, hp["sigma2"])
    assert rel(rec.theta_hat, hp["theta_hat"]) <= frank_cond_tol(hp["theta_hat"])
