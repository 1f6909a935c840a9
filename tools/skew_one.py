"""One rank call on skewed (normal-marginal) blocks: the cluster kernel's
quantile-knot path, for ncu captures."""
import os
import sys

import numpy as np
from scipy.special import ndtri

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05530_b200 as pcb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
dist = sys.argv[2] if len(sys.argv) > 2 else "normal"
g = np.random.default_rng(1)
f = {"normal": ndtri, "uniform": lambda u: u}[dist]
x, y = f(g.random(n)), f(g.random(n))
ctx = pcb.Context(0)
off = np.linspace(0, n, n // 125000 + 1).astype(np.uint64)
U = pcb.normalized_ranks(pcb.DataMatrix(x, y), off, ctx=ctx)
print(dist, ctx.rank_paths())
