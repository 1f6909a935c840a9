"""Full-data (K = 1) fit at n = 1e8 on device: timing probe for the global rank path."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05530_b200 as pcb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
ctx = pcb.Context(0)
s = torch.cuda.current_stream()
ctx.set_stream(s.cuda_stream)
c1 = torch.empty(n, dtype=torch.float64, device="cuda")
c2 = torch.empty(n, dtype=torch.float64, device="cuda")
ctx.check(ctx.lib.pcb_sample(ctx.ptr, 1, 5.0, n, 1000, 0, 1000, pcb.BASE_SEED, c1.data_ptr(), c2.data_ptr()))
off = np.array([0, n], np.uint64)
rec = torch.zeros((1, 6), dtype=torch.int64, device="cuda")
for it in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    ctx.check(ctx.lib.pcb_fit_blocks(ctx.ptr, 1, 0, c1.data_ptr(), c2.data_ptr(), n,
                                     off.ctypes.data_as(C.POINTER(C.c_uint64)), 1, rec.data_ptr()))
    e1.record(s)
    torch.cuda.synchronize()
    print("K=1 fit ms", round(e0.elapsed_time(e1), 2), {k: round(v, 2) for k, v in ctx.stage_times().items()})
