"""Device-vs-oracle parity through the C-ABI (libparcop_b200.so) on a B200.

Bars (BASELINE.json north_star): ranks bit-identical; theta-hat, sigma2,
loglik and theta_combined within 1e-9 relative (fp64 path) or 1e-5 (fp32
likelihood path) of the CPU oracle on the same bytes.
"""
import numpy as np
import pytest
from scipy.special import ndtri

import paper_1609_05530_b200 as pcb

pytestmark = pytest.mark.gpu

TOL64 = 1e-9
TOL32 = 1e-5
FAMS = [(0, 0.5), (1, 5.0), (2, 2.0)]
SWEEP = [(0, 0.2), (0, 0.8), (0, -0.5), (1, 2.0), (1, 10.0), (1, -4.0), (2, 1.5), (2, 3.0)]


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def oracle_ranks(orc, col, off):
    return np.concatenate([orc.rank_column(col[int(off[m]):int(off[m + 1])]) for m in range(len(off) - 1)])


def check_records(got, want, tol):
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert bool(g.converged) == bool(w.converged), (g, w.converged)
        if not w.converged:
            continue
        assert rel(g.theta_hat, w.theta_hat) <= tol, (g.theta_hat, w.theta_hat)
        assert rel(g.sigma2, w.sigma2) <= max(tol, 1e-9), (g.sigma2, w.sigma2)
        if tol <= 1e-9:
            assert rel(g.loglik, w.loglik) <= 1e-9 or abs(g.loglik - w.loglik) < 1e-9, (g.loglik, w.loglik)


# ----------------------------------------------------------------- ranks
@pytest.mark.parametrize("n,k", [(10000, 10), (100000, 10), (30000, 7), (2, 1), (4097, 1)])
def test_ranks_bit_exact_random(ctx, orc, n, k):
    rng = np.random.default_rng(n + k)
    c1 = rng.standard_normal(n)
    c2 = rng.exponential(size=n) * 1e3
    off = np.linspace(0, n, k + 1).astype(np.uint64)
    U = pcb.normalized_ranks(pcb.DataMatrix(c1, c2), off, ctx=ctx)
    assert np.array_equal(U.u1, oracle_ranks(orc, c1, off))
    assert np.array_equal(U.u2, oracle_ranks(orc, c2, off))


def test_ranks_match_compiled_reference(ctx, ref):
    rng = np.random.default_rng(7)
    c1 = np.round(rng.standard_normal(5000), 2)  # many ties
    c2 = rng.uniform(size=5000)
    U = pcb.normalized_ranks(pcb.DataMatrix(c1, c2), ctx=ctx)
    r1, r2 = ref.normalized_ranks(c1, c2)
    assert np.array_equal(U.u1, r1) and np.array_equal(U.u2, r2)


ADVERSARIAL = {
    "spec_example": ([3.1, 1.2, 7.5], [1.0, 1.0, 2.0]),
    "signed_zero": ([0.0, -0.0, 1.0, -1.0], [-0.0, 0.0, -0.0, 0.0]),
    "constant": (np.full(5000, 3.0), np.full(5000, -2.0)),
    "few_values": (np.arange(20000) % 7 * 1.0, np.arange(20000) % 3 * 1.0),
    "big_tie_runs": (np.repeat([1.0, 2.0, 3.0], 3000), np.tile([5.0, 4.0], 4500)),
    "geometric": (2.0 ** np.arange(-500, 500, 1.0), -(2.0 ** np.arange(-500, 500, 1.0))),
    "huge_range": (np.array([-1e308, 1e308, 0.0, 5e-324, -5e-324, 1.0] * 50), np.linspace(-1, 1, 300)),
    "one_outlier": (np.r_[np.zeros(9999) + 0.5, 1e300], np.r_[np.linspace(0, 1, 5000), np.full(5000, 0.25)]),
    "clustered": (np.r_[np.random.default_rng(3).uniform(0, 1e-9, 8000), np.random.default_rng(4).uniform(5, 6, 8)],
                  np.random.default_rng(5).standard_cauchy(8008)),
}


@pytest.mark.parametrize("name", sorted(ADVERSARIAL))
def test_ranks_adversarial(ctx, orc, name):
    c1, c2 = (np.asarray(a, np.float64) for a in ADVERSARIAL[name])
    U = pcb.normalized_ranks(pcb.DataMatrix(c1, c2), ctx=ctx)
    w1, w2 = orc.normalized_ranks(c1, c2)
    assert np.array_equal(U.u1, w1), name
    assert np.array_equal(U.u2, w2), name


def test_ranks_ragged_segments(ctx, orc):
    rng = np.random.default_rng(11)
    sizes = [2, 3, 31, 4096, 4097, 8191, 100, 17000, 2]
    off = np.r_[0, np.cumsum(sizes)].astype(np.uint64)
    n = int(off[-1])
    c1 = np.round(rng.standard_normal(n), 1)
    c2 = rng.uniform(size=n)
    U = pcb.normalized_ranks(pcb.DataMatrix(c1, c2), off, ctx=ctx)
    assert np.array_equal(U.u1, oracle_ranks(orc, c1, off))
    assert np.array_equal(U.u2, oracle_ranks(orc, c2, off))


def test_ranks_nonfinite_raises(ctx):
    with pytest.raises(pcb.DomainError):
        pcb.normalized_ranks(pcb.DataMatrix([1.0, np.nan, 2.0], [1.0, 2.0, 3.0]), ctx=ctx)
    with pytest.raises(pcb.DomainError):
        pcb.normalized_ranks(pcb.DataMatrix([1.0, 2.0, 3.0], [np.inf, 2.0, 3.0]), ctx=ctx)
    with pytest.raises(ValueError):
        pcb.normalized_ranks(pcb.DataMatrix([1.0], [1.0]), ctx=ctx)


# ------------------------------------------------------------- fit path
@pytest.mark.parametrize("fam,theta", FAMS + SWEEP)
def test_fit_blocks_parity(ctx, orc, fam, theta):
    n, k = 40000, 8
    X = pcb.sample_matrix(fam, theta, n, k, ctx=ctx)
    off = orc.partition(n, k)
    got = pcb.fit_blocks(fam, X, off, ctx=ctx)
    want = orc.fit_blocks(fam, X.col1, X.col2, off)
    check_records(got, want, TOL64)
    res = pcb.fit_parallel(fam, X, k, ctx=ctx)
    tc, w, used = orc.combine(want)
    assert res.blocks_used == used
    assert rel(res.theta_combined, tc) <= TOL64
    assert np.allclose(res.weights, w, rtol=1e-9, atol=0)


@pytest.mark.parametrize("fam,theta", FAMS + [(1, -4.0), (2, 3.0)])
def test_fit_fp32_parity(ctx, orc, fam, theta):
    n, k = 40000, 4
    X = pcb.sample_matrix(fam, theta, n, k, ctx=ctx)
    off = orc.partition(n, k)
    got = pcb.fit_blocks(fam, X, off, precision=pcb.Precision.fp32, ctx=ctx)
    want = orc.fit_blocks(fam, X.col1, X.col2, off)
    check_records(got, want, TOL32)


# fp32 likelihood path at edge parameters (the cases tools/fp32_edges.py
# found outside the bar before Frank blocks with |theta| < 2 ran their
# decision passes in fp64 arithmetic; fit.cu kFrank32Exact): Frank near 0 and
# around the switch, Gumbel just above the boundary theta = 1. Bar: 1e-5.
FP32_EDGES = [(1, t) for t in (-0.3, -0.05, 0.05, 0.3, 1.0, 1.9, 2.1, 25.0, -30.0)] + \
             [(2, t) for t in (1.001, 1.003, 1.006, 1.01, 1.05)] + [(0, 0.0), (0, 0.97), (0, -0.97)]


@pytest.mark.parametrize("fam,theta", FP32_EDGES)
def test_fit_fp32_edge_parameters(ctx, orc, fam, theta):
    rng = np.random.default_rng(abs(hash((fam, theta))) % 2**32)
    for _ in range(3):
        n = int(rng.integers(2000, 200000))
        k = int(rng.integers(1, 5))
        X = pcb.sample_matrix(fam, theta, n, k, base_seed=int(rng.integers(1, 2**62)), ctx=ctx)
        off = orc.partition(n, k)
        got = pcb.fit_blocks(fam, X, off, precision=pcb.Precision.fp32, ctx=ctx)
        want = orc.fit_blocks(fam, X.col1, X.col2, off)
        check_records(got, want, TOL32)


@pytest.mark.parametrize("fam,theta", FAMS)
def test_fit_from_pseudo_sample(ctx, orc, fam, theta):
    n = 5000
    X = pcb.sample_matrix(fam, theta, n, 1, ctx=ctx)
    u1, u2 = orc.normalized_ranks(X.col1, X.col2)
    g = pcb.fit(fam, pcb.PseudoSample(u1, u2), ctx=ctx)
    w = orc.fit(fam, u1, u2)
    check_records([g], [w], TOL64)
    s2 = pcb.asymptotic_variance(fam, w.theta_hat, pcb.PseudoSample(u1, u2), ctx=ctx)
    assert rel(s2, orc.asymptotic_variance(fam, w.theta_hat, u1, u2)) <= TOL64
    ll = pcb.pseudo_loglik(fam, w.theta_hat, pcb.PseudoSample(u1, u2), ctx=ctx)
    assert rel(ll, orc.pseudo_loglik(fam, w.theta_hat, u1, u2)) <= 1e-11


def test_fit_with_ties_uses_tie_run_suffix(ctx, orc):
    rng = np.random.default_rng(21)
    n = 6000
    z = rng.standard_normal(n)
    c1 = np.round(z, 1)
    c2 = np.round(0.6 * z + 0.8 * rng.standard_normal(n), 1)
    u1, u2 = orc.normalized_ranks(c1, c2)
    for fam in (0, 1, 2):
        g = pcb.fit(fam, pcb.PseudoSample(u1, u2), ctx=ctx)
        w = orc.fit(fam, u1, u2)
        check_records([g], [w], TOL64)
        naive = orc.asymptotic_variance(fam, w.theta_hat, u1, u2, naive=True)
        assert rel(g.sigma2, naive) <= 1e-9


def test_pseudo_loglik_segments(ctx, orc):
    X = pcb.sample_matrix(1, 5.0, 9000, 3, ctx=ctx)
    off = orc.partition(9000, 3)
    U = pcb.normalized_ranks(X, off, ctx=ctx)
    th = np.array([4.0, 5.0, -2.0])
    got = pcb.pseudo_loglik(1, th, U, segments=off, ctx=ctx)
    for m in range(3):
        a, b = int(off[m]), int(off[m + 1])
        assert rel(got[m], orc.pseudo_loglik(1, th[m], U.u1[a:b], U.u2[a:b])) <= 1e-11


def test_domain_errors(ctx):
    U = pcb.PseudoSample(np.array([0.2, 0.5, 0.7]), np.array([0.3, 0.6, 0.1]))
    with pytest.raises(pcb.DomainError):
        pcb.pseudo_loglik(0, 1.0, U, ctx=ctx)
    with pytest.raises(pcb.DomainError):
        pcb.pseudo_loglik(2, 0.9, U, ctx=ctx)
    with pytest.raises(pcb.DomainError):
        pcb.pseudo_loglik(1, 0.0, U, ctx=ctx)
    with pytest.raises(pcb.DomainError):
        pcb.fit(0, pcb.PseudoSample(np.array([0.2, 1.0] * 20), np.array([0.3, 0.5] * 20)), ctx=ctx)


def test_small_block_not_converged_not_error(ctx):
    X = pcb.sample_matrix(0, 0.5, 100, 1, ctx=ctx)
    g = pcb.fit_blocks(0, X, [0, 20, 100], ctx=ctx)
    assert not g[0].converged and g[0].status == 4
    assert g[1].converged


# ---------------------------------------------------- determinism / G split
def test_bitwise_determinism_and_gpu_split(ctx):
    n, k = 200000, 16
    fam = 2
    X = pcb.sample_matrix(fam, 2.0, n, k, ctx=ctx)
    off = pcb.partition(n, k).offsets
    a = pcb.fit_blocks(fam, X, off, ctx=ctx)
    b = pcb.fit_blocks(fam, X, off, ctx=ctx)
    assert [r.theta_hat for r in a] == [r.theta_hat for r in b]
    assert [r.sigma2 for r in a] == [r.sigma2 for r in b]
    # the same blocks fitted as two "GPU shards" (contiguous block ranges), then combined
    h = int(off[k // 2])
    s0 = pcb.fit_blocks(fam, pcb.DataMatrix(X.col1[:h], X.col2[:h]), off[:k // 2 + 1], ctx=ctx)
    s1 = pcb.fit_blocks(fam, pcb.DataMatrix(X.col1[h:], X.col2[h:]), off[k // 2:] - off[k // 2], ctx=ctx)
    assert [r.theta_hat for r in s0 + s1] == [r.theta_hat for r in a]
    assert pcb.combine(s0 + s1, ctx=ctx).theta_combined == pcb.combine(a, ctx=ctx).theta_combined


def test_sampler_shards_identical(ctx):
    full = pcb.sample_matrix(1, 5.0, 10000, 10, ctx=ctx)
    part = pcb.sample_matrix(1, 5.0, 10000, 10, first_block=3, last_block=7, ctx=ctx)
    assert np.array_equal(full.col1[3000:7000], part.col1)
    assert np.array_equal(full.col2[3000:7000], part.col2)


def test_sampler_integer_stream_matches_oracle(ctx, orc):
    # Frank u = the raw uniform draw: bit-identical to the oracle's counter-based stream
    n, k = 4000, 4
    X = pcb.sample_matrix(1, 5.0, n, k, ctx=ctx)
    off = orc.partition(n, k)
    c1, c2 = orc.sample_blocks(1, 5.0, n, k, off, 0, k)
    assert np.array_equal(X.col1, np.clip(c1, 1e-15, 1 - 1e-15))
    assert np.allclose(X.col2, c2, rtol=1e-13, atol=0)
    for fam, th in ((0, 0.5), (2, 2.0)):
        X = pcb.sample_matrix(fam, th, n, k, ctx=ctx)
        c1, c2 = orc.sample_blocks(fam, th, n, k, off, 0, k)
        assert np.allclose(X.col1, c1, rtol=1e-12, atol=1e-300)


def test_strided_scheme(ctx, orc):
    n, k = 10007, 5
    X = pcb.sample_matrix(0, 0.5, n, 1, ctx=ctx)
    res = pcb.fit_parallel(0, X, k, scheme=pcb.Scheme.Strided, ctx=ctx)
    p = pcb.partition(n, k, pcb.Scheme.Strided)
    recs = []
    for m in range(k):
        rows = np.arange(m, n, k)
        assert len(rows) == int(p.offsets[m + 1] - p.offsets[m])
        recs.append(orc.fit_blocks(0, X.col1[rows], X.col2[rows], [0, len(rows)])[0])
    check_records(res.per_block, recs, TOL64)


def test_combine_spec_examples_on_device(ctx):  # SPEC.md:290-292, exact where the SPEC is exact
    from paper_1609_05530_b200.parcop import FitResult
    mk = lambda t, s: FitResult(t, s, 100, 0.0, 3, True)  # noqa: E731
    assert pcb.combine([mk(0.3, 1.0), mk(0.3, 2.0), mk(0.3, 9.0)], ctx=ctx).theta_combined == 0.3
    assert pcb.combine([mk(1.99112997922569, 2.0584161e-4)], ctx=ctx).theta_combined == 1.99112997922569
    assert pcb.combine([mk(0.2, 1.0), mk(0.4, 4.0)], ctx=ctx).theta_combined == pytest.approx(0.24, rel=1e-15)
    bad = FitResult(9.0, 1.0, 100, 0.0, 50, False)
    r = pcb.combine([bad, mk(0.2, 2.0), mk(0.4, 2.0)], ctx=ctx)
    assert r.blocks_used == 2 and r.theta_combined == pytest.approx(0.3, rel=1e-15)


def test_m1_equals_full_fit(ctx):
    X = pcb.sample_matrix(2, 2.0, 20000, 1, ctx=ctx)
    res = pcb.fit_parallel(2, X, 1, ctx=ctx)
    full = pcb.fit(2, pcb.normalized_ranks(X, ctx=ctx), ctx=ctx)
    assert res.theta_combined == full.theta_hat


def test_c1_golden_fixture(ctx):
    """configs[0] on the reference's own sampler bytes (tests/golden)."""
    import json
    import os
    d = os.path.join(os.path.dirname(__file__), "golden")
    data = np.load(os.path.join(d, "c1_gaussian_rho05_n1e4.npz"))
    meta = json.load(open(os.path.join(d, "c1_expected.json")))
    X = pcb.DataMatrix(data["col1"], data["col2"])
    res = pcb.fit_parallel(0, X, 10, ctx=ctx)
    for g, w in zip(res.per_block, meta["per_block"]):
        assert rel(g.theta_hat, w["theta_hat"]) <= TOL64
        assert rel(g.sigma2, w["sigma2"]) <= TOL64
    assert rel(res.theta_combined, meta["theta_combined"]) <= TOL64
    U = pcb.normalized_ranks(X, pcb.partition(10000, 10).offsets, ctx=ctx)
    import hashlib
    assert hashlib.sha256(U.u1.tobytes() + U.u2.tobytes()).hexdigest() == meta["ranks_sha256"]


# ------------------------------------------- cluster vs global code paths
@pytest.fixture
def env(monkeypatch):
    return monkeypatch


@pytest.mark.parametrize("n,k", [(300000, 1), (250000, 2), (125000, 1)])
def test_rank_large_and_cluster_segments(ctx, orc, n, k):
    rng = np.random.default_rng(n + 7)
    c1 = rng.uniform(size=n)
    c2 = np.round(rng.standard_normal(n), 2)  # heavy ties spanning cluster slices
    off = np.linspace(0, n, k + 1).astype(np.uint64)
    U = pcb.normalized_ranks(pcb.DataMatrix(c1, c2), off, ctx=ctx)
    assert np.array_equal(U.u1, oracle_ranks(orc, c1, off))
    assert np.array_equal(U.u2, oracle_ranks(orc, c2, off))


SKEWED = {
    "normal": lambda u: ndtri(u),
    "exponential": lambda u: -np.log1p(-u),
    "cauchy": lambda u: np.tan(np.pi * (u - 0.5)),
    "lognormal": lambda u: np.exp(3.0 * ndtri(u)),
    "narrow-offset": lambda u: 1000.0 + 1e-3 * ndtri(u),
    "mixed-sign-pareto": lambda u: np.sign(u - 0.5) * (np.abs(2.0 * u - 1.0) + 1e-12) ** -1.5,
}


@pytest.mark.parametrize("name", list(SKEWED))
def test_rank_skewed_marginals_stay_on_cluster_path(ctx, orc, name):
    """Raw (non-uniform) marginals overflow the value-linear owner split; the
    cluster kernel re-splits by exact quantile knots instead of handing the
    block to the global path. Ranks stay bit-exact."""
    rng = np.random.default_rng(hash(name) % 2**32)
    n, k = 500000, 4  # 125k-row blocks: 9-CTA clusters in tail mode
    f = SKEWED[name]
    c1, c2 = f(rng.uniform(size=n)), f(rng.uniform(size=n))
    off = np.linspace(0, n, k + 1).astype(np.uint64)
    U = pcb.normalized_ranks(pcb.DataMatrix(c1, c2), off, ctx=ctx)
    assert np.array_equal(U.u1, oracle_ranks(orc, c1, off))
    assert np.array_equal(U.u2, oracle_ranks(orc, c2, off))
    assert ctx.rank_paths() == {"cluster": 2 * k, "global": 0, "constant": 0, "invalid": 0}


@pytest.mark.parametrize("fam,theta,name", [(1, 5.0, "normal"), (2, 2.0, "cauchy"), (0, 0.5, "lognormal")])
def test_fit_on_skewed_raw_marginals(ctx, orc, fam, theta, name):
    """Raw columns with skewed marginals (quantile-split ranks in slot space)
    through the whole pipeline: theta-hat, sigma2 and the combine against the
    oracle on the same bytes."""
    n, k = 1_000_000, 8  # 125k-row blocks
    X = pcb.sample_matrix(fam, theta, n, k, ctx=ctx)
    f = SKEWED[name]
    c1, c2 = f(np.asarray(X.col1)), f(np.asarray(X.col2))
    off = orc.partition(n, k)
    got = pcb.fit_blocks(fam, pcb.DataMatrix(c1, c2), off, ctx=ctx)
    assert ctx.rank_paths()["global"] == 0
    want = orc.fit_blocks(fam, c1, c2, off)
    check_records(got, want, TOL64)


def test_rank_extreme_magnitudes_bit_exact(ctx, orc):
    """Quantile-knot positions over keys spanning subnormals, signed zeros and
    +-1e308 (halved-value interpolation, underflowed interval widths)."""
    rng = np.random.default_rng(99)
    n, k = 250000, 2
    q = n // 8
    tiny = rng.choice([-1.0, 1.0], q) * 5e-324 * rng.integers(1, 1 << 40, q)  # subnormals, few ties
    parts = [rng.standard_normal(n - 2 * q - 64), rng.choice([-1.0, 1.0], q) * 10.0 ** rng.uniform(200, 308, q),
             tiny, np.where(rng.random(64) < 0.5, -0.0, 0.0)]
    c1 = np.concatenate(parts)
    rng.shuffle(c1)
    c2 = c1[::-1].copy()
    off = np.linspace(0, n, k + 1).astype(np.uint64)
    U = pcb.normalized_ranks(pcb.DataMatrix(c1, c2), off, ctx=ctx)
    assert np.array_equal(U.u1, oracle_ranks(orc, c1, off))
    assert np.array_equal(U.u2, oracle_ranks(orc, c2, off))
    assert ctx.rank_paths()["cluster"] == 2 * k  # the quantile-knot split handled it


def test_rank_forced_global_path_identical(ctx, env):
    rng = np.random.default_rng(5)
    n = 100000
    X = pcb.DataMatrix(rng.uniform(size=n), np.round(rng.uniform(size=n), 3))
    off = np.linspace(0, n, 5).astype(np.uint64)
    a = pcb.normalized_ranks(X, off, ctx=ctx)
    env.setenv("PCB_RANK_GLOBAL", "1")
    b = pcb.normalized_ranks(X, off, ctx=ctx)
    assert np.array_equal(a.u1, b.u1) and np.array_equal(a.u2, b.u2)


def test_rank_lean_variant_identical(ctx, orc, env):
    """The opt-in two-CTAs-per-SM rank kernel (PCB_RANK_LEAN=1) ranks bit-identically and feeds the same fit."""
    rng = np.random.default_rng(11)
    n = 250000
    X = pcb.DataMatrix(rng.uniform(size=n), np.round(rng.standard_normal(n), 3))
    off = np.linspace(0, n, 3).astype(np.uint64)
    a = pcb.normalized_ranks(X, off, ctx=ctx)
    env.setenv("PCB_RANK_LEAN", "1")
    b = pcb.normalized_ranks(X, off, ctx=ctx)
    assert np.array_equal(a.u1, b.u1) and np.array_equal(a.u2, b.u2)
    assert np.array_equal(b.u2, oracle_ranks(orc, X.col2, off))
    Y = pcb.sample_matrix(2, 2.0, 125000, 1, ctx=ctx)
    r = pcb.fit_blocks(2, Y, [0, 125000], ctx=ctx)[0]
    w = orc.fit_blocks(2, np.asarray(Y.col1), np.asarray(Y.col2), np.array([0, 125000], np.uint64))[0]
    assert abs(r.theta_hat - w.theta_hat) <= 1e-9 * w.theta_hat and abs(r.sigma2 - w.sigma2) <= 1e-9 * w.sigma2


@pytest.mark.parametrize("var", ["PCB_RANK_FK", "PCB_RANK_FK2"])
def test_rank_fine_key_variants_identical(ctx, orc, env, var):
    """The fine-key rank kernels (32-bit keys over DSMEM, full keys in the
    side array for equal fine keys; FK2: two CTAs per SM) rank bit-identically
    on continuous, tie-heavy, signed-zero and skewed columns, and feed the same fit."""
    rng = np.random.default_rng(17)
    n = 375000
    z = rng.standard_normal(n)
    c2 = np.round(rng.uniform(size=n), 3)
    c2[::97] = -0.0
    c2[1::97] = 0.0
    X = pcb.DataMatrix(rng.uniform(size=n), c2)
    off = np.linspace(0, n, 4).astype(np.uint64)
    a = pcb.normalized_ranks(X, off, ctx=ctx)
    S = pcb.DataMatrix(z, np.exp(2.0 * z))  # skewed: overflowing owners take the quantile relaunch
    sa = pcb.normalized_ranks(S, off, ctx=ctx)
    env.setenv(var, "1")
    b = pcb.normalized_ranks(X, off, ctx=ctx)
    sb = pcb.normalized_ranks(S, off, ctx=ctx)
    assert np.array_equal(a.u1, b.u1) and np.array_equal(a.u2, b.u2)
    assert np.array_equal(sa.u1, sb.u1) and np.array_equal(sa.u2, sb.u2)
    assert np.array_equal(b.u2, oracle_ranks(orc, X.col2, off))
    Y = pcb.sample_matrix(1, 5.0, 250000, 2, ctx=ctx)
    r = pcb.fit_blocks(1, Y, [0, 125000, 250000], ctx=ctx)
    w = orc.fit_blocks(1, np.asarray(Y.col1), np.asarray(Y.col2), np.array([0, 125000, 250000], np.uint64))
    check_records(r, w, TOL64)


@pytest.mark.parametrize("fam,theta", FAMS)
def test_variance_cluster_vs_global(ctx, orc, env, fam, theta):
    n, k = 60000, 3
    X = pcb.sample_matrix(fam, theta, n, k, ctx=ctx)
    X = pcb.DataMatrix(X.col1, np.round(X.col2, 4))  # ties in column 2
    off = orc.partition(n, k)
    a = pcb.fit_blocks(fam, X, off, ctx=ctx)
    env.setenv("PCB_VAR_GLOBAL", "1")
    b = pcb.fit_blocks(fam, X, off, ctx=ctx)
    want = orc.fit_blocks(fam, X.col1, X.col2, off)
    check_records(a, want, TOL64)
    check_records(b, want, TOL64)


def test_variance_large_segment_global(ctx, orc):
    n = 320000
    X = pcb.sample_matrix(2, 3.0, n, 1, ctx=ctx)
    got = pcb.fit_blocks(2, X, [0, n], ctx=ctx)
    want = orc.fit_blocks(2, X.col1, X.col2, [0, n])
    check_records(got, want, TOL64)


def test_host_streaming_identical(ctx, env):
    """Host-resident columns are streamed group by group (H2D overlapping
    compute); every block's record must equal the device-resident call's."""
    n, k = 64000, 16
    X = pcb.sample_matrix(2, 2.0, n, k, ctx=ctx)
    off = pcb.partition(n, k).offsets
    env.setenv("PCB_STREAM_ROWS", "9000")  # groups of 2 blocks
    host = pcb.fit_blocks(2, X, off, ctx=ctx)
    import torch
    dev = pcb.DataMatrix(torch.from_numpy(X.col1).cuda(), torch.from_numpy(X.col2).cuda())
    devr = pcb.fit_blocks(2, dev, off, ctx=ctx)
    assert [(r.theta_hat, r.sigma2, r.loglik) for r in host] == [(r.theta_hat, r.sigma2, r.loglik) for r in devr]
    res = pcb.fit_parallel(2, X, k, ctx=ctx)
    assert res.theta_combined == pcb.combine(devr, ctx=ctx).theta_combined


# --------------------------------------------------- BASELINE configs as parity cases
def test_config_c2_full_parity(ctx, orc):
    """configs[1] (C2): Frank theta=5, n=1e6, K=100 subsets of 1e4 — every block against the oracle."""
    n, k = 1_000_000, 100
    X = pcb.sample_matrix(1, 5.0, n, k, ctx=ctx)
    res = pcb.fit_parallel(1, X, k, ctx=ctx)
    off = orc.partition(n, k)
    want = orc.fit_blocks(1, X.col1, X.col2, off)
    check_records(res.per_block, want, TOL64)
    tc, w, used = orc.combine(want)
    assert res.blocks_used == used == k and rel(res.theta_combined, tc) <= TOL64
    assert abs(res.theta_combined - 5.0) < 0.05


def test_config_c3_sampled_parity_and_invariants(ctx, orc):
    """configs[2] (C3): Gumbel theta=2, n=1e8, K=1000 subsets of 1e5 on device; eight blocks against the
    oracle on the same bytes, SPEC.md:304-308 invariants over all of them."""
    import torch
    n, k = 100_000_000, 1000
    X = pcb.sample_matrix(2, 2.0, n, k, device_out=True, ctx=ctx)
    res = pcb.fit_parallel(2, X, k, ctx=ctx)
    assert res.blocks_used == k and all(r.converged for r in res.per_block)
    q = n // k
    for m in (0, 1, 137, 500, 501, 777, 998, 999):
        c1 = X.col1[m * q:(m + 1) * q].cpu().numpy()
        c2 = X.col2[m * q:(m + 1) * q].cpu().numpy()
        w = orc.fit_blocks(2, c1, c2, np.array([0, q], np.uint64))[0]
        check_records([res.per_block[m]], [w], TOL64)
    th = np.array([r.theta_hat for r in res.per_block])
    assert th.min() <= res.theta_combined <= th.max()  # convexity
    assert abs(res.theta_combined - 2.0) < 0.01
    scaled = [pcb.FitResult(r.theta_hat, 3.0 * r.sigma2, r.n, r.loglik, r.iterations, r.converged)
              for r in res.per_block]
    assert rel(pcb.combine(scaled, ctx=ctx).theta_combined, res.theta_combined) <= 1e-13  # weight-scale invariance
    del X
    torch.cuda.empty_cache()


EXTREME = [(0, 0.99), (0, -0.99), (0, 0.0), (1, 35.0), (1, -30.0), (1, 0.05), (2, 1.0), (2, 15.0)]


@pytest.mark.parametrize("fam,theta", EXTREME)
def test_fit_extreme_parameters(ctx, orc, fam, theta):
    n, k = 30000, 3
    X = pcb.sample_matrix(fam, theta, n, k, ctx=ctx)
    off = orc.partition(n, k)
    got = pcb.fit_blocks(fam, X, off, ctx=ctx)
    want = orc.fit_blocks(fam, X.col1, X.col2, off)
    check_records(got, want, TOL64)


def test_frank_near_zero_conditioning(ctx, orc):
    """Frank estimate ~1e-3 on 240 rows (a fuzz case): both the device and the
    oracle against a 60-digit evaluation (tests/golden/make_frank_near_zero.py),
    and device vs oracle within the conditioning-scaled bar of
    tests/test_oracle.py::frank_cond_tol (1e-9 x (0.03/|theta|)^2 below |theta| = 0.03)."""
    import json
    import os

    from test_oracle import frank_cond_tol

    gold = os.path.join(os.path.dirname(__file__), "golden")
    inp = json.load(open(os.path.join(gold, "frank_near_zero_input.json")))
    hp = json.load(open(os.path.join(gold, "frank_near_zero_expected.json")))
    c1, c2 = np.asarray(inp["c1"]), np.asarray(inp["c2"])
    off = np.array([0, len(c1)], np.uint64)
    (g,) = pcb.fit_blocks(1, pcb.DataMatrix(c1, c2), off, ctx=ctx)
    (w,) = orc.fit_blocks(1, c1, c2, off)
    assert g.converged and w.converged
    assert rel(g.theta_hat, hp["theta_hat"]) <= 5e-9, (g.theta_hat, hp["theta_hat"])
    assert rel(g.sigma2, hp["sigma2"]) <= 5e-8, (g.sigma2, hp["sigma2"])
    tol = frank_cond_tol(w.theta_hat)
    assert rel(g.theta_hat, w.theta_hat) <= tol and rel(g.sigma2, w.sigma2) <= tol


@pytest.mark.parametrize("theta,seed", [(1.003, 11), (1.006, 12), (1.01, 13), (1.006, 14)])
def test_gumbel_near_boundary(ctx, orc, theta, seed):
    """Gumbel estimates just above the independence boundary theta = 1: the
    score is strongly curved there and sigma2 amplifies any error of
    theta-hat ~100x, so the fp64 stop must account for the residual the last
    Newton step leaves (fit.cu newton_update); found by tools/fuzz_fit.py."""
    n = 120000
    X = pcb.sample_matrix(2, theta, n, 1, base_seed=0x160905530 + seed, ctx=ctx)
    off = np.array([0, n], np.uint64)
    (g,) = pcb.fit_blocks(2, X, off, ctx=ctx)
    (w,) = orc.fit_blocks(2, np.asarray(X.col1), np.asarray(X.col2), off)
    check_records([g], [w], TOL64)


# the Monte Carlo variance oracle on the device path
# (tests/test_oracle.py runs it on the oracle): 1000 i.i.d. replicates of
# n = 5000 (the SPEC's 200 carry ~10% sampling error), mean device sigma2
# within 20% of the empirical variance of the device theta-hats; and the
# 1/n scaling: sigma2 at 2n over sigma2 at n averages in [0.4, 0.6].
@pytest.mark.parametrize("fam,theta", [(0, 0.3), (1, 5.0), (2, 2.0)])
def test_monte_carlo_variance_oracle_device(ctx, fam, theta):
    reps, n = 1000, 5000
    X = pcb.sample_matrix(fam, theta, reps * n, reps, base_seed=0x5EC231, ctx=ctx)
    off = pcb.partition(reps * n, reps).offsets
    recs = pcb.fit_blocks(fam, X, off, ctx=ctx)
    th = np.array([r.theta_hat for r in recs])
    s2 = np.array([r.sigma2 for r in recs])
    assert all(r.converged for r in recs)
    assert 0.8 <= s2.mean() / th.var(ddof=1) <= 1.2
    half = pcb.fit_blocks(fam, X, np.sort(np.concatenate([off, off[:-1] + n // 2])), ctx=ctx)
    s2h = np.array([r.sigma2 for r in half]).reshape(reps, 2).mean(axis=1)
    assert 0.4 <= np.mean(s2 / s2h) <= 0.6
