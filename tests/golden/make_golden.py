#!/usr/bin/env python3
"""Generate tests/golden/*.npz from the REFERENCE ITSELF (run in the build container,
where /root/reference exists; the fixtures are committed so GPU boxes need no reference).

  im2col_ref.npz     : the reference's rendered im2col kernel (proj/templates/im2col.kt.tmpl,
                       rendered by its own template engine, compiled as C++ and executed)
                       on seeded images, for several geometries.
  apply_reduce_ref.npz : dispatch_apply / dispatch_reduce_all / dispatch_reduce_dim on
                       reference_backend() (proj/src/backend.cpp:115-161) over strided,
                       offset views built with narrow/select.

usage: python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import pyoracle as po  # noqa: E402
from ref_kernels import ref_im2col  # noqa: E402
from test_oracle import EXPRS, IM2COL_GEOMS, _view_from_ops, random_view  # noqa: E402


def gkey(g):
    return [g.N, g.C, g.H, g.W, g.K, g.kH, g.kW, g.padH, g.padW, g.strideH, g.strideW]


def main():
    assert po.ref_available(), "needs oracle/_ref (build in the container with /root/reference)"
    out = {}
    meta = []
    for i, g in enumerate(IM2COL_GEOMS):
        img = po.uniform((g.C, g.H, g.W), 5000 + i)
        out[f"img{i}"] = img
        out[f"col{i}"] = ref_im2col(g, img)
        meta.append(gkey(g))
    np.savez_compressed(os.path.join(HERE, "im2col_ref.npz"), geoms=np.array(meta, np.int64),
                        **out)

    cases = []
    arrays = {}
    rng = np.random.default_rng(2024)
    for c in range(40):
        text, arity = EXPRS[c % len(EXPRS)]
        shape, ops = random_view(rng)
        sizes, strides, off = _view_from_ops(shape, ops)
        bases = [po.uniform(shape, 900 * c + t).ravel().copy() for t in range(arity)]
        before = [b.copy() for b in bases]
        st, err = po.ref_apply(text, bases, [shape] * arity, [ops] * arity, -0.625)
        assert st == 0, err
        for t in range(arity):
            arrays[f"a{c}_in{t}"] = before[t]
        arrays[f"a{c}_out"] = bases[0]
        cases.append({"kind": "apply", "id": c, "expr": text, "arity": arity, "shape": shape,
                      "sizes": sizes, "strides": strides, "offset": off, "scalar": -0.625})
    for c in range(30):
        shape, ops = random_view(rng)
        sizes, strides, off = _view_from_ops(shape, ops)
        base = po.uniform(shape, 7000 + c).ravel().copy()
        op = c % 3
        st, v, err = po.ref_reduce_all(op, base, shape, ops)
        assert st == 0, err
        dim = int(rng.integers(0, len(sizes)))
        n_out = int(np.prod(sizes)) // sizes[dim]
        st, rd, err = po.ref_reduce_dim(op, base, shape, ops, dim, n_out)
        assert st == 0, err
        arrays[f"r{c}_in"] = base
        arrays[f"r{c}_all"] = np.array([v], np.float32)
        arrays[f"r{c}_dim"] = rd
        cases.append({"kind": "reduce", "id": c, "op": op, "shape": shape, "sizes": sizes,
                      "strides": strides, "offset": off, "dim": dim})
    np.savez_compressed(os.path.join(HERE, "apply_reduce_ref.npz"), **arrays)
    with open(os.path.join(HERE, "apply_reduce_ref.json"), "w") as f:
        json.dump(cases, f, indent=0)
    print("wrote golden fixtures:", len(IM2COL_GEOMS), "im2col,", len(cases), "apply/reduce")


if __name__ == "__main__":
    main()
