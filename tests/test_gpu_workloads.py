"""GPU parity on EVERY layer bench.py times (convnet-benchmarks L1-L5, AlexNet c1-c5,
Overfeat-fast c1-c5, VGG-A c1-c8 — the shapes are imported from bench.WORKLOADS, so the
tests and the bench cannot drift apart), through exactly the path the bench times:
updateOutput keeping Torch's finput, then the combined updateGradInput + accGradParameters
call reusing it, captured once as a CUDA graph and replayed.

  * full batch, TF32-exact integer inputs (helpers.exact_inputs): every element of y,
    gradInput, gradWeight and gradBias equals the CPU oracle BITWISE — the index mapping
    of whichever tcgen05 engine the layer takes is proven exactly, at the real shape and
    batch; the graph replay equals the eager launches bitwise;
  * a 2-image slice with real-valued inputs: elementwise TF32 bounds (helpers.tf32_bounds)
    and the normwise 1e-3 bound, through the bench path and the separate passes.
"""
import numpy as np
import pytest

import pyoracle as po
from bench import WORKLOADS
from engine_check import check_geometry
from helpers import check_exact, with_batch

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

BENCH_LAYERS = [(wl, l) for wl in ("convnet", "alexnet", "overfeat", "vgga") for l in WORKLOADS[wl]]
IDS = [f"{wl}-{l[0]}" for wl, l in BENCH_LAYERS]


def _pt():
    import paper_1606_04884_b200 as pt
    return pt


def _geoms(l):
    _, N, C, H, W, K, kH, kW, pH, pW, sH, sW = l
    return (_pt().ConvGeometry(N, C, H, W, K, kH, kW, pH, pW, sH, sW),
            po.geom(N, C, H, W, K, kH, kW, pH, pW, sH, sW))


def _exact_device_inputs(G, seed):
    """Integers in [-8, 8] (x, gy), {-1, 0, 1} (w), [-4, 4] (b), generated on the device."""
    pt = _pt()
    t = lambda shape, s, a: pt.fill_uniform(torch.empty(shape, device="cuda"), s, -a - 0.5,  # noqa: E731
                                            a + 0.5).round_().clamp_(-a, a)
    return (t(G.input_shape(), seed + 1, 8), t(G.weight_shape(), seed + 2, 1),
            t((G.outChannels,), seed + 3, 4), t(G.output_shape(), seed + 4, 8))


def bench_step_graph(G, x, w, b, gy):
    """The bench's per-layer step (bench.py `layer`), eager once, then captured as a CUDA
    graph on a side stream (workspace warmed on that stream first) and replayed."""
    pt = _pt()
    nb = pt.finput_bytes(G)
    fin = torch.empty(nb, dtype=torch.uint8, device="cuda") if nb else None
    outs = [torch.empty(G.output_shape(), device="cuda"), torch.empty(G.input_shape(), device="cuda"),
            torch.empty(G.weight_shape(), device="cuda"), torch.empty((G.outChannels,), device="cuda")]

    def step():
        y, gx, gw, gb = outs
        pt.conv_forward(G, x, w, b, y, finput=fin)
        pt.conv_backward(G, x, gy, w, gx, gw, gb, finput=fin)

    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        step()
    side.synchronize()
    eager = [o.clone() for o in outs]
    for o in outs:
        o.fill_(float("nan"))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        step()
    graph.replay()
    torch.cuda.synchronize()
    for name, e, o in zip(("y", "gx", "gw", "gb"), eager, outs):
        assert torch.equal(e, o), f"{name}: graph replay differs from the eager launches"
    return [o.cpu().numpy() for o in outs]


@pytest.mark.parametrize("wl,l", BENCH_LAYERS, ids=IDS)
def test_bench_layer_full_batch_exact(wl, l):
    G, g = _geoms(l)
    x, w, b, gy = _exact_device_inputs(G, 0x5EED + 17 * len(l[0]))
    y, gx, gw, gb = bench_step_graph(G, x, w, b, gy)
    hx, hw, hb, hgy = (t.cpu().numpy() for t in (x, w, b, gy))
    check_exact(y, po.conv_forward(g, hx, hw, hb), f"{wl}/{l[0]} y")
    check_exact(gx, po.conv_backward_input(g, hgy, hw), f"{wl}/{l[0]} gradInput")
    rgw, rgb = po.conv_backward_weight(g, hx, hgy)
    check_exact(gw, rgw, f"{wl}/{l[0]} gradWeight")
    check_exact(gb, rgb, f"{wl}/{l[0]} gradBias")


@pytest.mark.parametrize("wl,l", BENCH_LAYERS, ids=IDS)
def test_bench_layer_slice_tf32(wl, l):
    _, g = _geoms(l)
    fails, rels = check_geometry(with_batch(g, 2), seed=0xC0FFEE, exact=True, real=True)
    assert not fails, "\n".join(fails[:4])
    assert max(rels.values()) <= 1e-3
