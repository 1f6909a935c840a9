"""torchrun worker for tests/test_gpu_nccl.py: the per-process multi-GPU leg
of bench.py (NCCL process group, contiguous block shard, device records
all-gathered over NCCL, combine in block order, max-over-ranks timing
all-reduce) on however many GPUs the launcher gives it. Prints one line per
rank; rank 0 also checks theta_combined against one process fitting every
block."""
import ctypes
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1609_05530_b200 as pcb  # noqa: E402
from paper_1609_05530_b200 import _lib as L  # noqa: E402
from paper_1609_05530_b200.distributed import gather_records, shard_blocks  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
assert dist.get_backend() == "nccl"
ctx = pcb.Context(local)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
n, K, seed = 4_000_000, 32, 0x160905530
q = n // K
for fam, th in ((0, 0.5), (1, 5.0), (2, 2.0)):
    first, last = shard_blocks(K, world, rank)
    rows = (last - first) * q
    kl = last - first
    c1 = torch.empty(rows, dtype=torch.float64, device="cuda")
    c2 = torch.empty(rows, dtype=torch.float64, device="cuda")
    ctx.check(ctx.lib.pcb_sample(ctx.ptr, fam, th, n, K, first, last, seed, c1.data_ptr(), c2.data_ptr()))
    off = np.arange(kl + 1, dtype=np.uint64) * np.uint64(q)
    recs = torch.zeros((kl, 6), dtype=torch.int64, device="cuda")
    ctx.check(ctx.lib.pcb_fit_blocks(ctx.ptr, fam, 0, c1.data_ptr(), c2.data_ptr(), rows,
                                     off.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), kl, recs.data_ptr()))
    full = gather_records(recs, K)  # NCCL all_gather of the 48-byte records
    comb = L.CombinedC()
    ctx.check(ctx.lib.pcb_combine(ctx.ptr, full.data_ptr(), K, None, ctypes.byref(comb)))
    t = torch.tensor([float(rank)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # the bench's max-over-ranks timing reduction
    assert t.item() == world - 1
    if rank == 0:
        X = pcb.sample_matrix(fam, th, n, K, ctx=ctx)
        ref = pcb.fit_parallel(fam, X, K, ctx=ctx)
        assert comb.theta_combined == ref.theta_combined, (fam, comb.theta_combined, ref.theta_combined)
        assert int(comb.blocks_used) == ref.blocks_used
    print(f"NCCL_OK rank={rank} world={world} family={fam} theta_combined={comb.theta_combined!r}", flush=True)
dist.barrier()
dist.destroy_process_group()
ctx.close()
