"""Parity at the headline and largest configs, bounded for the test suite
(tools/parity_large.py runs the unbounded versions; their results are in
profiles/r02_parity_c5.json and profiles/r02_parity_c4.json).

* C5 (configs[4]): n = 1e9 per family, K = 8000 subsets of 125,000 -- the
  device fits ALL 8000 blocks; 256 blocks spread over the whole range are
  re-fitted by the CPU oracle on the same bytes; theta-hat / sigma2 within
  1e-9, theta_combined over those blocks within 1e-9.
* Large segments (configs[3]'s global-path sizes): 1e7-row blocks, ranks
  bit-identical per segment (pseudo_obs.hpp:44-65) and the fit records within
  1e-9.
"""
import numpy as np
import pytest

from tools.parity_large import c4_case, c5_family

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fam,theta", [(0, 0.5), (1, 5.0), (2, 2.0)])
def test_c5_headline_parity_spread_blocks(ctx, orc, fam, theta):
    picks = np.linspace(0, 7999, 256).round().astype(np.int64)
    r = c5_family(ctx, orc, fam, theta, n=1_000_000_000, K=8000, picks=picks)
    assert r["converged_mismatch"] == 0 and r["converged"] == 256, r
    assert r["max_rel_theta"] <= 1e-9, r
    assert r["max_rel_sigma2"] <= 1e-9, r
    assert r["rel_theta_combined"] <= 1e-9, r
    assert r["blocks_used_device"] == r["blocks_used_oracle"]


@pytest.mark.parametrize("fam,theta", [(0, 0.5), (1, 5.0), (2, 2.0)])
def test_large_segments_ranks_and_fit(ctx, orc, fam, theta):
    r = c4_case(ctx, orc, fam, theta, n=20_000_000, K=2)
    assert r["rank_columns_identical"] == r["rank_columns_checked"] == 4, r
    assert r["converged_mismatch"] == 0, r
    assert r["max_rel_theta"] <= 1e-9, r
    assert r["max_rel_sigma2"] <= 1e-9, r
    assert r["rel_theta_combined"] <= 1e-9, r
