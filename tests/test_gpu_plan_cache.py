"""The per-thread TMA-descriptor (plan) cache: a second call on the same buffers encodes
nothing new and gives the same result bitwise (pt_b200_plan_cache_stats)."""
import numpy as np
import pytest

import pyoracle as po
from helpers import conv_inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("g", [po.geom(2, 64, 20, 20, 96, 5, 5, 2, 2, 1, 1),
                               po.geom(2, 3, 40, 40, 96, 11, 11, 0, 0, 1, 1),
                               po.geom(2, 3, 63, 63, 64, 11, 11, 2, 2, 4, 4)])
def test_repeat_call_hits_cache(g):
    import paper_1606_04884_b200 as pt
    x, w, b, gy = conv_inputs(g, 5)
    G = pt.ConvGeometry(g.N, g.C, g.H, g.W, g.K, g.kH, g.kW, g.padH, g.padW, g.strideH, g.strideW)
    dx, dw, db, dgy = (torch.from_numpy(a).cuda() for a in (x, w, b, gy))
    y = torch.empty(G.output_shape(), device="cuda")
    gx = torch.empty(G.input_shape(), device="cuda")
    gw = torch.empty(G.weight_shape(), device="cuda")
    gb = torch.empty((g.K,), device="cuda")

    def step():
        pt.conv_forward(G, dx, dw, db, y)
        pt.conv_backward(G, dx, dgy, dw, gx, gw, gb)
        torch.cuda.synchronize()
        return [t.cpu().numpy().copy() for t in (y, gx, gw, gb)]

    first = step()
    h0, e0 = pt.plan_cache_stats()
    second = step()
    h1, e1 = pt.plan_cache_stats()
    assert e1 == e0, "the repeated call re-encoded tensor maps"
    assert h1 > h0, "the repeated call did not use the cache"
    for a, c in zip(first, second):
        assert np.array_equal(a.view(np.uint32), c.view(np.uint32))
