"""CPU, world_size 2 over gloo: batch sharding + gradient allreduce reproduce the
full-batch gradients (the N>1 path of bench.py, minus the GPU kernels — each rank's
per-shard gradients come from the oracle here)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import pyoracle as po
    from paper_1606_04884_b200.dp import GradBucket, allreduce_async, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = 5
        g = po.geom(N, 3, 9, 9, 4, 3, 3, 1, 1, 1, 1)
        x = po.uniform((N, 3, 9, 9), 1)
        gy = po.uniform((N, 4, 9, 9), 2)
        lo, hi = shard_range(N, rank, world)
        gs = po.geom(hi - lo, 3, 9, 9, 4, 3, 3, 1, 1, 1, 1)
        gw, gb = po.conv_backward_weight(gs, x[lo:hi], gy[lo:hi])
        bucket = GradBucket([gw.shape, gb.shape], "cpu")
        bucket.views[0].copy_(torch.from_numpy(gw))
        bucket.views[1].copy_(torch.from_numpy(gb))
        allreduce_async(bucket)
        if rank == 0:
            rgw, rgb = po.conv_backward_weight(g, x, gy)
            q.put((bucket.views[0].numpy().copy(), bucket.views[1].numpy().copy(), rgw, rgb))
    finally:
        dist.destroy_process_group()


def test_shard_ranges_partition_the_batch():
    from paper_1606_04884_b200.dp import shard_range
    for n in (1, 5, 8, 128, 129):
        for w in (1, 2, 3, 8):
            got = [shard_range(n, r, w) for r in range(w)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(h - l for l, h in got) - min(h - l for l, h in got) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_dp_allreduce_equals_full_batch_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gw, gb, rgw, rgb = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    np.testing.assert_allclose(gw, rgw, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(gb, rgb, rtol=1e-5, atol=1e-5)
