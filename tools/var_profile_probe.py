import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_1609_05530_b200 as pcb
ctx = pcb.Context(0)
n, K = 200_000_000, 1600
for fam, th in ((0, 0.5), (1, 5.0)):
    X = pcb.sample_matrix(fam, th, n, K, device_out=True, ctx=ctx)
    for i in range(2):
        r = pcb.fit_parallel(fam, X, K, ctx=ctx)
    print(fam, ctx.stage_times(), flush=True)
