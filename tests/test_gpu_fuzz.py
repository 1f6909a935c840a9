"""Short randomised parity runs (tools/fuzz_ranks.py, tools/fuzz_fit.py):
random segment sizes around the cluster thresholds and random marginals
(tie runs, signed zeros, subnormals to 1e308, sorted input, heavy tails)
through every rank path, compared with the oracle — ranks bit for bit, fit
records within 1e-9. Longer runs: `python tools/fuzz_ranks.py 240`."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

pytestmark = pytest.mark.gpu


def test_fuzz_ranks(ctx, orc):
    import fuzz_ranks
    print(fuzz_ranks.run(12.0, 20261020, ctx=ctx, orc=orc))


def test_fuzz_fit(ctx, orc):
    import fuzz_fit
    print(fuzz_fit.run(12.0, 20261021, ctx=ctx, orc=orc))
