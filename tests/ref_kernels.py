"""Execute the REFERENCE's own rendered OpenCL im2col kernel on the CPU.

The reference renders proj/templates/im2col.kt.tmpl per geometry (its template engine,
via oracle/_ref/libportten_ref.so: ref_render_im2col). The text is OpenCL C 1.2; with
four macro shims (kernel/global qualifiers, get_global_id -> loop index) it compiles as
C++ and runs as-is — the reference's exact index maths, not a restatement.
Test infrastructure only.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess
import tempfile

import numpy as np

import pyoracle as po

_CACHE = os.path.join(tempfile.gettempdir(), "pt_ref_im2col")

SHIM = """
#define kernel extern "C"
#define global
static int pt_gid;
static inline int get_global_id(int) { return pt_gid; }
"""

DRIVER = """
extern "C" void run_all(const float* img, float* col, int n_items) {
    for (pt_gid = 0; pt_gid < n_items; ++pt_gid) portten_im2col(img, col);
}
"""


def compile_rendered(text: str, n_items: int) -> str:
    os.makedirs(_CACHE, exist_ok=True)
    key = hashlib.sha256(text.encode()).hexdigest()[:20]
    so = os.path.join(_CACHE, f"im2col_{key}.so")
    if not os.path.exists(so):
        src = os.path.join(_CACHE, f"im2col_{key}.cpp")
        # the kernel returns early for gid >= n_items; keep its guard verbatim
        body = text.replace("kernel void portten_im2col(", "kernel void portten_im2col(", 1)
        with open(src, "w") as f:
            f.write(SHIM + body + DRIVER)
        subprocess.run(["g++", "-O1", "-shared", "-fPIC", "-w", "-o", so, src], check=True)
    return so


def ref_im2col(g, img: np.ndarray) -> np.ndarray:
    """Run the reference's rendered im2col kernel for one image."""
    text = po.ref_render_im2col(g)
    oh, ow = po.out_hw(g)
    n_items = g.C * oh * ow
    so = compile_rendered(text, n_items)
    lib = C.CDLL(so)
    col = np.zeros((g.C * g.kH * g.kW, oh * ow), np.float32)
    img = np.ascontiguousarray(img, np.float32)
    lib.run_all(img.ctypes.data_as(C.POINTER(C.c_float)), col.ctypes.data_as(C.POINTER(C.c_float)),
                n_items)
    return col
