"""Parity of skewed-marginal fits against the oracle on a few blocks (ties created by
the transforms' rounding are legitimate, so each transform is checked on its own bytes)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05530_b200 as pcb  # noqa: E402
from oracle.oracle import oracle_lib  # noqa: E402

orc = oracle_lib()
n, K = 1_000_000, 8
ctx = pcb.Context(0)
X = pcb.sample_matrix(1, 5.0, n, K, ctx=ctx)
u1, u2 = torch.from_numpy(np.asarray(X.col1)), torch.from_numpy(np.asarray(X.col2))
off = orc.partition(n, K)
for name, f in {"normal": torch.special.ndtri, "exponential": lambda u: -torch.log1p(-u),
                "cauchy": lambda u: torch.tan(np.pi * (u - 0.5)), "lognormal": lambda u: torch.exp(3 * torch.special.ndtri(u))}.items():
    c1, c2 = f(u1).numpy().copy(), f(u2).numpy().copy()
    got = pcb.fit_blocks(1, pcb.DataMatrix(c1, c2), off, ctx=ctx)
    want = orc.fit_blocks(1, c1, c2, off)
    worst = max(abs(g.theta_hat - w.theta_hat) / abs(w.theta_hat) for g, w in zip(got, want))
    ties = sum(len(c) - len(np.unique(c)) for c in (c1, c2))
    print(f"{name:12s} worst rel err vs oracle {worst:.2e}  ties created {ties}")
