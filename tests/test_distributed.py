"""CPU, world_size 2 over gloo: the multi-GPU host logic (contiguous block
shards, the record all-gather, combine in block order) reproduces the
single-process result bitwise. Per-shard fits are the oracle's records here
(no GPU in this container); the device path is the same code with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1609_05530_b200.distributed import gather_records, shard_blocks

N, K = 24000, 10


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import oracle_lib
    orc = oracle_lib()
    off = orc.partition(N, K)
    first, last = shard_blocks(K, world, rank)
    # each rank draws and fits ONLY its own blocks (same per-block seeds as one process)
    c1, c2 = orc.sample_blocks(2, 2.0, N, K, off, first, last)
    loc_off = off[first:last + 1] - off[first]
    recs = orc.fit_blocks(2, c1, c2, loc_off, workers=2)
    raw = np.frombuffer(bytes(recs), dtype=np.int64).reshape(last - first, 6).copy()
    full = gather_records(torch.from_numpy(raw), K)
    q.put((rank, full.numpy().tobytes()))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_blocks_cover():
    for k in (1, 7, 8000):
        for w in (1, 2, 3, 8):
            spans = [shard_blocks(k, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == k
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_world2_gather_and_combine_bitwise():
    from oracle.oracle import FitRecord, oracle_lib
    orc = oracle_lib()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert outs[0] == outs[1]  # every rank holds the same gathered records
    gathered = (FitRecord * K).from_buffer_copy(outs[0])
    off = orc.partition(N, K)
    c1, c2 = orc.sample_blocks(2, 2.0, N, K, off, 0, K)
    single = orc.fit_blocks(2, c1, c2, off)
    assert bytes(gathered) == bytes(single)
    assert orc.combine(gathered)[0] == orc.combine(single)[0]
