"""Scratch probe: convnet step eager vs one CUDA-graph replay per step (1 GPU)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1606_04884_b200 as pt  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "convnet"
dev = torch.device("cuda", 0)
st = []
for i, l in enumerate(bench.WORKLOADS[wl]):
    name, N, C, H, W, K, kH, kW, pH, pW, sH, sW = l
    g = pt.ConvGeometry(N, C, H, W, K, kH, kW, pH, pW, sH, sW)
    x = pt.fill_uniform(torch.empty(g.input_shape(), device=dev), i + 1)
    s = 1.0 / (C * kH * kW) ** 0.5
    w = pt.fill_uniform(torch.empty(g.weight_shape(), device=dev), i + 2, -s, s)
    b = pt.fill_uniform(torch.empty((K,), device=dev), i + 3, -0.1, 0.1)
    gy = pt.fill_uniform(torch.empty(g.output_shape(), device=dev), i + 4)
    fb = pt.finput_bytes(g)
    st.append(dict(g=g, x=x, w=w, b=b, gy=gy, y=torch.empty(g.output_shape(), device=dev),
                   gx=torch.empty(g.input_shape(), device=dev), gw=torch.empty(g.weight_shape(), device=dev),
                   gb=torch.empty((K,), device=dev),
                   fin=torch.empty(fb, dtype=torch.uint8, device=dev) if fb else None))


def step():
    for s in st:
        pt.conv_forward(s["g"], s["x"], s["w"], s["b"], s["y"], finput=s["fin"])
        pt.conv_backward(s["g"], s["x"], s["gy"], s["w"], s["gx"], s["gw"], s["gb"], finput=s["fin"])


def timed(fn, k=20):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record()
    for _ in range(k):
        fn()
    h1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k, (h1 - h0) * 1e3 / k


for _ in range(3):
    step()
print(wl, "eager  gpu %.3f ms/step  host %.3f ms/step" % timed(step))
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
torch.cuda.current_stream().wait_stream(s)
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    step()
for _ in range(3):
    graph.replay()
print(wl, "graph  gpu %.3f ms/step  host %.3f ms/step" % timed(graph.replay))
print(wl, "eager  gpu %.3f ms/step  host %.3f ms/step" % timed(step))
