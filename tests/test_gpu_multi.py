"""Multi-device contexts (pcb_create_multi):
fit_blocks / fit_parallel shard the blocks over the context's devices with
no communication, gather the 48-byte records by peer copies and combine in
block order, so every record and theta_combined is bitwise identical for any
device list. gpurun grants one GPU, so the "devices" are
the same GPU listed 2 and 3 times (independent contexts, streams and host
threads); the code path is the one a multi-GPU box takes (peer copies become
NVLink transfers)."""
import numpy as np
import pytest

import paper_1609_05530_b200 as pcb

pytestmark = pytest.mark.gpu


def recs(rs):
    return [(r.theta_hat, r.sigma2, r.loglik, r.iterations, r.converged, r.status) for r in rs]


@pytest.mark.parametrize("fam,theta", [(0, 0.5), (1, 5.0), (2, 2.0)])
def test_multi_device_context_bitwise(ctx, fam, theta):
    import torch
    n, k = 2_000_000, 37
    X = pcb.sample_matrix(fam, theta, n, k, ctx=ctx)  # host (pageable numpy)
    off = pcb.partition(n, k).offsets
    one = pcb.fit_blocks(fam, X, off, ctx=ctx)
    res1 = pcb.fit_parallel(fam, X, k, ctx=ctx)
    Xd = pcb.DataMatrix(torch.from_numpy(X.col1).cuda(), torch.from_numpy(X.col2).cuda())
    for devs in ([0, 0], [0, 0, 0]):
        m = pcb.Context(devices=devs)
        assert m.lib.pcb_device_count(m.ptr) == len(devs)
        assert recs(pcb.fit_blocks(fam, X, off, ctx=m)) == recs(one)      # host columns, per-device streaming
        assert recs(pcb.fit_blocks(fam, Xd, off, ctx=m)) == recs(one)     # device columns on device 0
        r = pcb.fit_parallel(fam, X, k, ctx=m)
        assert r.theta_combined == res1.theta_combined and r.blocks_used == res1.blocks_used
        assert np.array_equal(r.weights, res1.weights)
        assert r.wall_clock_per_block > 0.0
        rs = pcb.fit_parallel(fam, X, k, scheme=pcb.Scheme.Strided, ctx=m)
        assert rs.theta_combined == pcb.fit_parallel(fam, X, k, scheme=pcb.Scheme.Strided, ctx=ctx).theta_combined
        m.close()


def test_multi_device_more_devices_than_blocks(ctx):
    X = pcb.sample_matrix(1, 5.0, 3000, 2, ctx=ctx)
    m = pcb.Context(devices=[0, 0, 0])
    a = pcb.fit_parallel(1, X, 2, ctx=m)
    b = pcb.fit_parallel(1, X, 2, ctx=ctx)
    assert a.theta_combined == b.theta_combined and recs(a.per_block) == recs(b.per_block)
    m.close()


def test_pageable_host_streaming_groups_identical(ctx, monkeypatch):
    """Pageable numpy columns streamed in many groups by the staging thread
    (and split over two contexts) give the device-resident records."""
    import torch
    n, k = 640000, 40
    X = pcb.sample_matrix(2, 2.0, n, k, ctx=ctx)
    off = pcb.partition(n, k).offsets
    dev = pcb.fit_blocks(2, pcb.DataMatrix(torch.from_numpy(X.col1).cuda(), torch.from_numpy(X.col2).cuda()), off,
                         ctx=ctx)
    monkeypatch.setenv("PCB_STREAM_ROWS", "50000")  # ~3 blocks per group, >10 groups
    assert recs(pcb.fit_blocks(2, X, off, ctx=ctx)) == recs(dev)
    m = pcb.Context(devices=[0, 0])
    assert recs(pcb.fit_blocks(2, X, off, ctx=m)) == recs(dev)
    m.close()
