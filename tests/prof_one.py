"""Run one conv pass of one bench layer a few times (target for ncu captures).

  python tests/prof_one.py --workload convnet --layer L2 --pass fwd|dgrad|wgrad [--iters 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1606_04884_b200 as pt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="convnet")
ap.add_argument("--layer", default="L2")
ap.add_argument("--pass", dest="which", default="fwd")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--math", default="tf32")
a = ap.parse_args()
l = [x for x in bench.WORKLOADS[a.workload] if x[0] == a.layer][0]
g = pt.ConvGeometry(*l[1:])
x = pt.fill_uniform(torch.empty(g.input_shape(), device="cuda"), 1)
w = pt.fill_uniform(torch.empty(g.weight_shape(), device="cuda"), 2, -0.05, 0.05)
b = pt.fill_uniform(torch.empty((g.outChannels,), device="cuda"), 3)
gy = pt.fill_uniform(torch.empty(g.output_shape(), device="cuda"), 4)
y = torch.empty(g.output_shape(), device="cuda")
gx = torch.empty(g.input_shape(), device="cuda")
gw = torch.empty(g.weight_shape(), device="cuda")
gb = torch.empty((g.outChannels,), device="cuda")
for _ in range(a.iters):
    if a.which == "fwd":
        pt.conv_forward(g, x, w, b, y, math=a.math)
    elif a.which == "dgrad":
        pt.conv_backward_input(g, gy, w, gx, math=a.math)
    elif a.which == "bwd":
        pt.conv_backward(g, x, gy, w, gx, gw, gb, math=a.math)
    else:
        pt.conv_backward_weight(g, x, gy, gw, gb, math=a.math)
torch.cuda.synchronize()
print("done", g)
