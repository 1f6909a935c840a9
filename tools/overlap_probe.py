"""Probe: do two library contexts on one GPU (two host threads, two streams)
overlap the three C5 families usefully? Prints ms per step for the serial
order and for a 2-way split, device-synchronised wall clock."""
import ctypes as C
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05530_b200 as pcb  # noqa: E402

N, K = 1_000_000_000, 8000
FAMS = [("gaussian", 0, 0.5), ("frank", 1, 5.0), ("gumbel", 2, 2.0)]
q = N // K
off = (np.arange(K + 1, dtype=np.uint64) * np.uint64(q))
offp = off.ctypes.data_as(C.POINTER(C.c_uint64))
ctxs = [pcb.Context(0), pcb.Context(0)]
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
for c, s in zip(ctxs, streams):
    c.set_stream(s.cuda_stream)
cols = {}
for name, fam, th in FAMS:
    c1 = torch.empty(N, dtype=torch.float64, device="cuda")
    c2 = torch.empty(N, dtype=torch.float64, device="cuda")
    ctxs[0].check(ctxs[0].lib.pcb_sample(ctxs[0].ptr, fam, th, N, K, 0, K, pcb.BASE_SEED, c1.data_ptr(), c2.data_ptr()))
    cols[name] = (c1, c2, fam)
recs = {name: torch.zeros((K, 6), dtype=torch.int64, device="cuda") for name, _, _ in FAMS}
torch.cuda.synchronize()


def run(ci, names):
    c = ctxs[ci]
    for nm in names:
        c1, c2, fam = cols[nm]
        c.check(c.lib.pcb_fit_blocks(c.ptr, fam, 0, c1.data_ptr(), c2.data_ptr(), N, offp, K, recs[nm].data_ptr()))


def timed(plan, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        ths = [threading.Thread(target=run, args=(i, names)) for i, names in enumerate(plan)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t) * 1e3)
    return best


timed([["gaussian", "frank", "gumbel"]], 2)  # warm-up both workspaces
timed([["gaussian", "gumbel"], ["frank"]], 2)
print("serial          ms/step", round(timed([["gaussian", "frank", "gumbel"]]), 1))
print("2-way (G+U | F) ms/step", round(timed([["gaussian", "gumbel"], ["frank"]]), 1))
print("2-way (G+F | U) ms/step", round(timed([["gaussian", "frank"], ["gumbel"]]), 1))
print("mem used GB", round(torch.cuda.mem_get_info()[1] / 1e9 - torch.cuda.mem_get_info()[0] / 1e9, 1))
