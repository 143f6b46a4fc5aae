"""Per-geometry parity check of the conv passes through the C ABI, used in-process by the
GPU tests and as a subprocess under engine-forcing environment switches (the switches
are read once per process):

  python tests/engine_check.py '<json list of [N,C,H,W,K,kH,kW,pH,pW,sH,sW]>' [seed]

For every geometry, through the path bench.py times (updateOutput keeping Torch's finput,
then the combined updateGradInput + accGradParameters reusing it) and through the separate
passes:
  * TF32-exact integer inputs (helpers.exact_inputs): y, gradInput, gradWeight, gradBias
    must equal the oracle BITWISE;
  * real-valued inputs (helpers.conv_inputs): elementwise TF32 bounds (helpers.tf32_bounds)
    and the normwise bound.
Prints one JSON list: per geometry the list of failure messages (empty = pass) and the
normwise errors of the real-valued run.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, os.path.join(ROOT, "oracle"), HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

import numpy as np  # noqa: E402

import pyoracle as po  # noqa: E402
from helpers import (check_exact, check_tf32, conv_inputs, exact_inputs, gstr,  # noqa: E402
                     tf32_bounds)


def _passes(pt, torch, G, x, w, b, gy, separate=True):
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    dx, dw, db, dgy = d(x), d(w), d(b), d(gy)
    nb = pt.finput_bytes(G)
    fin = torch.empty(nb, dtype=torch.uint8, device="cuda") if nb else None
    y = pt.conv_forward(G, dx, dw, db, finput=fin)
    gx, gw, gb = pt.conv_backward(G, dx, dgy, dw, finput=fin)
    out = {"fwd": y, "dgrad": gx, "wgrad": gw, "gradBias": gb}
    if separate:
        out["fwd/plain"] = pt.conv_forward(G, dx, dw, db)
        out["dgrad/plain"] = pt.conv_backward_input(G, dgy, dw)
        out["wgrad/plain"], out["gradBias/plain"] = pt.conv_backward_weight(G, dx, dgy)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def _oracle(g, x, w, b, gy):
    y = po.conv_forward(g, x, w, b)
    gx = po.conv_backward_input(g, gy, w)
    gw, gb = po.conv_backward_weight(g, x, gy)
    return {"fwd": y, "dgrad": gx, "wgrad": gw, "gradBias": gb}


def check_geometry(g, seed=0x5EED, exact=True, real=True, separate=True):
    """Returns (failures, normwise errors of the real-valued run)."""
    import torch
    import paper_1606_04884_b200 as pt
    G = pt.ConvGeometry(g.N, g.C, g.H, g.W, g.K, g.kH, g.kW, g.padH, g.padW, g.strideH,
                        g.strideW)
    fails, rels = [], {}
    if exact:
        x, w, b, gy = exact_inputs(g, seed)
        out = _passes(pt, torch, G, x, w, b, gy, separate)
        ref = _oracle(g, x, w, b, gy)
        for k, v in out.items():
            try:
                check_exact(v, ref[k.split("/")[0]], f"{gstr(g)} exact {k}")
            except AssertionError as ex:
                fails.append(str(ex))
    if real:
        x, w, b, gy = conv_inputs(g, seed)
        out = _passes(pt, torch, G, x, w, b, gy, separate)
        ref = _oracle(g, x, w, b, gy)
        tol = tf32_bounds(g, x, w, b, gy)
        for k, v in out.items():
            base = k.split("/")[0]
            try:
                rels[k] = check_tf32(v, ref[base], f"{gstr(g)} tf32 {k}", tol[base])
            except AssertionError as ex:
                fails.append(str(ex))
    return fails, rels


def main():
    specs = json.loads(sys.argv[1])
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0x5EED
    res = []
    for s in specs:
        fails, rels = check_geometry(po.geom(*s), seed)
        res.append({"geom": s, "fails": fails, "rels": rels})
    print(json.dumps(res))


if __name__ == "__main__":
    main()
