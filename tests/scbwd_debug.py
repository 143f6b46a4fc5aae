"""Debug (GPU box): run one mode of the fused small-C backward on a small geometry and
compare with the oracle. usage: scbwd_debug.py dgrad|wgrad|both"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import torch  # noqa: E402

import paper_1606_04884_b200 as pt  # noqa: E402
import pyoracle as po  # noqa: E402
from helpers import exact_inputs  # noqa: E402

mode = sys.argv[1]
g = po.geom(2, 3, 20, 32, 64, 3, 3, 1, 1, 1, 1) if len(sys.argv) < 3 else po.geom(4, 3, 64, 64, 64, 3, 3, 1, 1, 1, 1)
G = pt.ConvGeometry(g.N, g.C, g.H, g.W, g.K, g.kH, g.kW, g.padH, g.padW, g.strideH, g.strideW)
x, w, b, gy = exact_inputs(g, 3)
d = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
if mode == "dgrad":
    gx = pt.conv_backward_input(G, d(gy), d(w))
    torch.cuda.synchronize()
    r = po.conv_backward_input(g, gy, w)
    print("dgrad maxdiff", np.abs(gx.cpu().numpy() - r).max())
elif mode == "wgrad":
    gw, gb = pt.conv_backward_weight(G, d(x), d(gy))
    torch.cuda.synchronize()
    rw, rb = po.conv_backward_weight(g, x, gy)
    print("wgrad maxdiff", np.abs(gw.cpu().numpy() - rw).max(), "gb", np.abs(gb.cpu().numpy() - rb).max())
else:
    gx, gw, gb = pt.conv_backward(G, d(x), d(gy), d(w))
    torch.cuda.synchronize()
    r = po.conv_backward_input(g, gy, w)
    rw, rb = po.conv_backward_weight(g, x, gy)
    print("both", np.abs(gx.cpu().numpy() - r).max(), np.abs(gw.cpu().numpy() - rw).max(),
          np.abs(gb.cpu().numpy() - rb).max())
