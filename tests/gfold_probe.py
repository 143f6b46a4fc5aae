"""GPU probe for the small-C gradCol + fold dgrad (umma_gfold.cu), not collected by pytest:
  python tests/gfold_probe.py N C H W K kH kW pH pW [reps]
runs updateGradInput reps times on seeded inputs and compares image 0 with the oracle."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, os.path.join(ROOT, "oracle"), HERE):
    sys.path.insert(0, p)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_04884_b200 as pt  # noqa: E402
import pyoracle as po  # noqa: E402
from helpers import conv_inputs, with_batch  # noqa: E402

a = [int(v) for v in sys.argv[1:10]]
reps = int(sys.argv[10]) if len(sys.argv) > 10 else 3
g = po.geom(*a, 1, 1)
G = pt.ConvGeometry(*a, 1, 1)
x, w, b, gy = conv_inputs(g, 7)
dgy, dw = torch.from_numpy(gy).cuda(), torch.from_numpy(w).cuda()
gx = torch.empty(G.input_shape(), device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for r in range(reps):
    ev[0].record()
    pt.conv_backward_input(G, dgy, dw, gx)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"rep {r}: {ev[0].elapsed_time(ev[1]):.3f} ms", flush=True)
g1 = with_batch(g, 1)
ref = po.conv_backward_input(g1, gy[:1], w)
out = gx[:1].cpu().numpy()
d = np.abs(out - ref)
print("max|d|", d.max(), "normwise", np.linalg.norm(out - ref) / np.linalg.norm(ref))
bad = np.argwhere(d > 1e-2 * (np.abs(ref).max() + 1e-6))
print("bad", len(bad), bad[:10].tolist())
