import sys, os
sys.path[:0] = [os.getcwd(), os.path.join(os.getcwd(), "oracle"), os.path.join(os.getcwd(), "tests")]
import numpy as np, torch
import paper_1606_04884_b200 as pt, pyoracle as po
from helpers import conv_inputs
spec = [int(v) for v in sys.argv[1].split(",")]
g = po.geom(*spec); G = pt.ConvGeometry(*spec)
x, w, b, gy = conv_inputs(g, 91)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
which = sys.argv[2]
if which == "fwd": y = pt.conv_forward(G, d(x), d(w), d(b))
else: gx = pt.conv_backward_input(G, d(gy), d(w))
torch.cuda.synchronize(); print("ok", spec, which)
