"""Stream-ordering guarantees of the conv C ABI on the GPU.

* CUDA-graph capture: a whole forward + backward (updateOutput, then the combined
  updateGradInput + accGradParameters call with its internal weight-gradient stream)
  captured with torch.cuda.graph and replayed gives bitwise the eager results, also after
  the static inputs are overwritten in place. This is what a caller needs to replace a
  launch-bound inner loop by one graph launch.
* A multi-layer step (several layers' forward + backward, as bench.py's one-rank step)
  captured as ONE graph replays bitwise to the eager results.
* The in-call concurrency switch (pt_b200_set_bwd_streams) never changes results.
* Two host threads driving the library on two streams at once get their own results.
"""
import threading

import numpy as np
import pytest

from helpers import conv_inputs
import pyoracle as po

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GEOMS = [
    # (N, C, H, W, K, kH, kW, pH, pW, sH, sW)
    (4, 64, 20, 20, 64, 5, 5, 2, 2, 1, 1),    # Hankel engines, channel-rich wgrad
    (4, 3, 24, 24, 32, 5, 5, 0, 0, 1, 1),     # small-C row kernels
    (2, 32, 17, 19, 48, 3, 3, 1, 1, 2, 2),    # strided, ragged
    (2, 3, 35, 35, 64, 11, 11, 2, 2, 4, 4),   # space-to-depth (AlexNet conv1-like)
    (2, 3, 24, 24, 64, 3, 3, 1, 1, 1, 1),     # small-C row forward + plane wgrad (VGG conv1-like)
    (2, 3, 30, 30, 96, 11, 11, 0, 0, 1, 1),   # convnet L1-like
]


def _pt():
    import paper_1606_04884_b200 as pt
    return pt


def _geom(t):
    return _pt().ConvGeometry(*t)


def _og(t):
    N, C, H, W, K, kH, kW, pH, pW, sH, sW = t
    return po.Geom(N, C, H, W, K, kH, kW, pH, pW, sH, sW)


def _inputs(t, seed):
    x, w, b, gy = conv_inputs(_og(t), seed)
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (x, w, b, gy)]


def _step(G, x, w, b, gy, fin):
    pt = _pt()
    y = pt.conv_forward(G, x, w, b, finput=fin)
    gx, gw, gb = pt.conv_backward(G, x, gy, w, finput=fin)
    return y, gx, gw, gb


def _finput(G):
    n = _pt().finput_bytes(G)
    return torch.empty(max(n, 1), dtype=torch.uint8, device="cuda") if n else None


@pytest.mark.parametrize("t", GEOMS, ids=lambda t: "x".join(map(str, t)))
def test_graph_capture_replay_bitwise(t):
    G = _geom(t)
    x, w, b, gy = _inputs(t, 0x5EED)
    fin = _finput(G)
    eager = [r.clone() for r in _step(G, x, w, b, gy, fin)]

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm the per-stream workspace and plan caches
        _step(G, x, w, b, gy, fin)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()

    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        out = _step(G, x, w, b, gy, fin)
    graph.replay()
    torch.cuda.synchronize()
    for name, e, o in zip(("y", "gx", "gw", "gb"), eager, out):
        assert torch.equal(e, o), f"{name}: graph replay differs from eager"

    # new values in the captured input buffers: the replay must see them
    x2, w2, b2, gy2 = _inputs(t, 0xBEEF)
    eager2 = [r.clone() for r in _step(G, x2, w2, b2, gy2, fin)]
    for dst, src in zip((x, w, b, gy), (x2, w2, b2, gy2)):
        dst.copy_(src)
    graph.replay()
    torch.cuda.synchronize()
    for name, e, o in zip(("y", "gx", "gw", "gb"), eager2, out):
        assert torch.equal(e, o), f"{name}: replay after an input update differs"


def test_multi_layer_step_one_graph_bitwise():
    layers = []
    for i, t in enumerate(GEOMS):
        G = _geom(t)
        layers.append((G, *_inputs(t, 100 + i), _finput(G)))
    eager = [[r.clone() for r in _step(*L)] for L in layers]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # the capture stream's workspace and plans, before capture
        for L in layers:
            _step(*L)
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        outs = [_step(*L) for L in layers]
    for _ in range(2):
        graph.replay()
    torch.cuda.synchronize()
    for t, e, o in zip(GEOMS, eager, outs):
        for name, a, b in zip(("y", "gx", "gw", "gb"), e, o):
            assert torch.equal(a, b), f"{t} {name}: one-graph step differs from eager"


@pytest.mark.parametrize("t", GEOMS[:2], ids=lambda t: "x".join(map(str, t)))
def test_bwd_streams_switch_bitwise(t):
    pt = _pt()
    G = _geom(t)
    x, w, b, gy = _inputs(t, 11)
    fin = _finput(G)
    lib = pt._lib.lib()
    try:
        lib.pt_b200_set_bwd_streams(0)
        serial = [r.clone() for r in _step(G, x, w, b, gy, fin)]
        lib.pt_b200_set_bwd_streams(1)
        conc = [r.clone() for r in _step(G, x, w, b, gy, fin)]
    finally:
        lib.pt_b200_set_bwd_streams(1)
    torch.cuda.synchronize()
    for name, a, c in zip(("y", "gx", "gw", "gb"), serial, conc):
        assert torch.equal(a, c), f"{name}: concurrent backward differs from serial"


def test_two_threads_two_streams():
    t0, t1 = GEOMS[0], GEOMS[1]
    jobs = []
    for t, seed in ((t0, 1), (t1, 2)):
        G = _geom(t)
        ins = _inputs(t, seed)
        fin = _finput(G)
        ref = [r.clone() for r in _step(G, *ins, fin)]
        jobs.append((G, ins, fin, ref))
    torch.cuda.synchronize()
    errors = []

    def run(G, ins, fin, ref):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(5):
                    out = _step(G, *ins, fin)
                    s.synchronize()
                    for a, o in zip(ref, out):
                        if not torch.equal(a, o):
                            errors.append("mismatch")
        except Exception as e:  # surfaced in the main thread
            errors.append(repr(e))

    th = [threading.Thread(target=run, args=j) for j in jobs]
    for h in th:
        h.start()
    for h in th:
        h.join()
    assert not errors, errors
