"""Rank stage of large blocks (the global multi-level path): n rows, K
segments of uniform keys (optionally rounded to D decimals: tie-heavy),
ranked three times; prints the wall time of each call and a digest of the
ranks. python tools/global_rank_probe.py [n] [K] [D]"""
import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05530_b200 as pcb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1
D = int(sys.argv[3]) if len(sys.argv) > 3 else -1
g = np.random.default_rng(1)
c1, c2 = g.random(n), g.random(n)
if D >= 0:
    c2 = np.round(c2, D)
import torch  # noqa: E402
ctx = pcb.Context(0)
off = np.linspace(0, n, K + 1).astype(np.uint64)
Xd = pcb.DataMatrix(torch.from_numpy(c1).cuda(), torch.from_numpy(c2).cuda())
for i in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    U = pcb.normalized_ranks(Xd, off, ctx=ctx)
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t)
    h = hashlib.sha256(np.asarray(U.u1.cpu() if hasattr(U.u1, "cpu") else U.u1).tobytes()
                       + np.asarray(U.u2.cpu() if hasattr(U.u2, "cpu") else U.u2).tobytes()).hexdigest()[:12]
    print(f"n={n} K={K} D={D} ranks {ms:.1f} ms paths {ctx.rank_paths()} digest {h}", flush=True)
