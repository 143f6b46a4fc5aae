"""Scratch: dgrad normwise error of one geometry vs the oracle (env switches pick engines).
  python tests/dgrad_probe.py N,C,H,W,K,kH,kW,pH,pW,sH,sW"""
import os
import sys
sys.path[:0] = [os.getcwd(), os.path.join(os.getcwd(), "oracle"), os.path.join(os.getcwd(), "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1606_04884_b200 as pt  # noqa: E402
import pyoracle as po  # noqa: E402
from helpers import conv_inputs  # noqa: E402

spec = [int(v) for v in sys.argv[1].split(",")]
g = po.geom(*spec)
G = pt.ConvGeometry(*spec)
x, w, b, gy = conv_inputs(g, 3)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
gx = pt.conv_backward_input(G, d(gy), d(w))
gx2, _, _ = pt.conv_backward(G, d(x), d(gy), d(w))
torch.cuda.synchronize()
r = po.conv_backward_input(g, gy, w)
rel = lambda a: float(np.linalg.norm(a.cpu().numpy().astype(np.float64) - r) / np.linalg.norm(r))  # noqa: E731
bad = np.abs(gx.cpu().numpy() - r) > 1e-2 * np.abs(r).max()
idx = np.argwhere(bad)
print(os.environ.get("TAGX", ""), spec, "dgrad %.2e combined %.2e" % (rel(gx), rel(gx2)), "bad", int(bad.sum()), "of", bad.size,
      "first", idx[:3].tolist())
