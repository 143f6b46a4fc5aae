"""GPU data parallelism (north_star: "shards the minibatch ..., allreducing
gradWeight/gradBias with NCCL, and nothing else is sharded") on one B200:

  * G in {2, 4, 8} ranks emulated in one process: the fixed global batch of the AlexNet /
    VGG-A stacks is split with dp.shard_range, every shard runs the real kernels through
    the bench path (finput + combined backward), the per-rank gradient buckets are summed.
    With TF32-exact inputs the shard outputs concatenate, and the bucket sum equals, the
    full-batch device result BITWISE (integer partial sums are exact in any order).
  * two real processes on cuda:0 over gloo running bench.Workload.step — the bench's own
    DP code (per-layer GradBucket, allreduce_async) around the real kernels: the
    all-reduced buckets equal the full-batch gradients bitwise.
"""
import os
import socket
import sys

import pytest

from bench import WORKLOADS

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _pt():
    import paper_1606_04884_b200 as pt
    return pt


def _exact(shape, seed, a):
    pt = _pt()
    return pt.fill_uniform(torch.empty(shape, device="cuda"), seed, -a - 0.5, a + 0.5).round_().clamp_(-a, a)


def _layer_inputs(l, seed):
    pt = _pt()
    _, N, C, H, W, K, kH, kW, pH, pW, sH, sW = l
    G = pt.ConvGeometry(N, C, H, W, K, kH, kW, pH, pW, sH, sW)
    return G, (_exact(G.input_shape(), seed + 1, 8), _exact(G.weight_shape(), seed + 2, 1),
               _exact((K,), seed + 3, 4), _exact(G.output_shape(), seed + 4, 8))


def _bench_path(G, x, w, b, gy):
    pt = _pt()
    nb = pt.finput_bytes(G)
    fin = torch.empty(nb, dtype=torch.uint8, device="cuda") if nb else None
    y = pt.conv_forward(G, x, w, b, finput=fin)
    gx, gw, gb = pt.conv_backward(G, x, gy, w, finput=fin)
    return y, gx, gw, gb


@pytest.mark.parametrize("ranks", [2, 4, 8])
@pytest.mark.parametrize("wl", ["alexnet", "vgga", "convnet"])
def test_emulated_ranks_equal_full_batch(wl, ranks):
    from paper_1606_04884_b200.dp import GradBucket, shard_range
    for i, l in enumerate(WORKLOADS[wl]):
        G, (x, w, b, gy) = _layer_inputs(l, 0xD0 + 10 * i)
        y, gx, gw, gb = _bench_path(G, x, w, b, gy)
        bucket = GradBucket([gw.shape, gb.shape], "cuda")  # the allreduce(sum) result
        ys, gxs = [], []
        for r in range(ranks):
            lo, hi = shard_range(G.batch, r, ranks)
            Gr = G.with_batch(hi - lo)
            yr, gxr, gwr, gbr = _bench_path(Gr, x[lo:hi].contiguous(), w, b, gy[lo:hi].contiguous())
            ys.append(yr)
            gxs.append(gxr)
            bucket.views[0].add_(gwr)
            bucket.views[1].add_(gbr)
        torch.cuda.synchronize()
        tag = f"{wl}/{l[0]} G={ranks}"
        assert torch.equal(torch.cat(ys), y), f"{tag}: sharded outputs differ from the full batch"
        assert torch.equal(torch.cat(gxs), gx), f"{tag}: sharded gradInput differs"
        assert torch.equal(bucket.views[0], gw), f"{tag}: summed gradWeight differs"
        assert torch.equal(bucket.views[1], gb), f"{tag}: summed gradBias differs"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    import torch
    import torch.distributed as dist
    import bench
    import paper_1606_04884_b200 as pt
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        glayers = bench.WORKLOADS["alexnet"]
        local = bench.local_layers(glayers, rank, world)
        wl = bench.Workload(pt, torch, local, torch.device("cuda", 0), rank, "tf32")
        full = []
        for i, (gl, s) in enumerate(zip(glayers, wl.st)):
            G, (x, w, b, gy) = _layer_inputs(gl, 0xE0 + 10 * i)  # same on every rank
            lo, hi = bench_shard(gl[1], rank, world)
            for k, t in (("x", x[lo:hi]), ("gy", gy[lo:hi]), ("w", w), ("b", b)):
                s[k].copy_(t)
            full.append(_bench_path(G, x, w, b, gy))
        wl.step(comm=None)  # the bench's step: graph-free launches + per-layer allreduce
        torch.cuda.synchronize()
        ok = []
        for (y, gx, gw, gb), s in zip(full, wl.st):
            lo, hi = bench_shard(y.shape[0], rank, world)
            ok.append(bool(torch.equal(s["y"], y[lo:hi]) and torch.equal(s["gx"], gx[lo:hi])
                           and torch.equal(s["gw"], gw) and torch.equal(s["gb"], gb)))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def bench_shard(n, rank, world):
    from paper_1606_04884_b200.dp import shard_range
    return shard_range(n, rank, world)


def test_gloo_two_processes_bench_step():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r, ok in res.items():
        assert all(ok), f"rank {r}: layers {ok} (y / gradInput slice, all-reduced gradients)"
