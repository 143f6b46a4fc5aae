"""Every tcgen05 engine, forced through its environment switch, on geometries aimed at its
edge cases: TF32-exact integer inputs must give the oracle's result BITWISE (fwd, gradInput,
gradWeight, gradBias — through the finput + combined-backward path and the separate
passes), real-valued inputs must meet the elementwise TF32 bounds. The switches are read
once per process, so each configuration runs tests/engine_check.py in a subprocess.
"""
import json
import os
import subprocess
import sys

import pytest

import pyoracle as po
from helpers import gstr

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# categories: small-C stride 1 (row forward, expanded tconv dgrad, plane wgrad), strided
# small-C (space-to-depth), channel-rich stride 1 of several kernel sizes (Hankel / im2col,
# tap groups, tap-quad wgrad), strided channel-rich, 1x1, ragged / rectangular shapes
GEOMS = [
    po.geom(2, 3, 40, 40, 96, 11, 11, 0, 0, 1, 1),       # convnet L1-like
    po.geom(2, 3, 37, 45, 64, 3, 3, 1, 1, 1, 1),         # VGG c1-like, odd extents
    po.geom(2, 3, 63, 63, 64, 11, 11, 2, 2, 4, 4),       # AlexNet c1-like (s2d)
    po.geom(2, 3, 67, 67, 96, 11, 11, 0, 0, 4, 4),       # Overfeat c1-like (s2d, pad 0)
    po.geom(2, 64, 24, 24, 128, 9, 9, 0, 0, 1, 1),       # convnet L2-like
    po.geom(2, 128, 16, 16, 128, 9, 9, 0, 0, 1, 1),      # convnet L3-like
    po.geom(2, 128, 13, 13, 384, 3, 3, 0, 0, 1, 1),      # convnet L5 (real shape)
    po.geom(2, 64, 27, 27, 192, 5, 5, 2, 2, 1, 1),       # AlexNet c2 (real shape)
    po.geom(2, 64, 30, 30, 128, 3, 3, 1, 1, 1, 1),       # VGG c2-like (<= 64 channels)
    po.geom(2, 96, 9, 11, 80, 3, 5, 1, 2, 1, 1),         # rectangular, K = 80
    po.geom(2, 32, 17, 19, 48, 3, 3, 1, 1, 2, 2),        # strided channel-rich
    po.geom(3, 64, 12, 12, 32, 1, 1, 0, 0, 1, 1),        # 1x1
    po.geom(2, 128, 17, 17, 64, 9, 9, 4, 4, 1, 1),       # large zero border (flat tiling)
    po.geom(1, 4, 21, 70, 128, 7, 7, 3, 3, 1, 1),        # C = 4, padded 7x7
    po.geom(2, 3, 38, 44, 64, 3, 3, 1, 1, 1, 1),         # VGG c1-like, fused small-C backward
    po.geom(2, 1, 20, 40, 48, 5, 5, 2, 2, 1, 1),         # fused small-C bwd, K = 48 (padded), 5x5
    po.geom(3, 2, 18, 36, 32, 3, 5, 1, 2, 1, 1),         # fused small-C bwd, rectangular, K = 32
]

CONFIGS = {
    "default": {},
    "hankel": {"PT_B200_HCONV": "1"},
    "hankel-runs2": {"PT_B200_HCONV": "1", "PT_B200_HCONV_RUNS": "2"},
    "hankel-g1": {"PT_B200_HCONV": "1", "PT_B200_HCONV_GROUP_MAX": "1"},
    "hankel-g2": {"PT_B200_HCONV": "1", "PT_B200_HCONV_GROUP_MAX": "2"},
    "hankel-g3": {"PT_B200_HCONV": "1", "PT_B200_HCONV_GROUP_MAX": "3"},
    "hankel-nopair": {"PT_B200_HCONV": "1", "PT_B200_HCONV_PAIR": "0"},
    "hankel-rows": {"PT_B200_HCONV": "1", "PT_B200_HCONV_A": "rows"},
    "im2col": {"PT_B200_HCONV": "0"},
    "hwgrad-forced": {"PT_B200_HWGRAD": "2"},
    "hwgrad-off": {"PT_B200_HWGRAD": "0"},
    "swgrad-off": {"PT_B200_SWGRAD": "0"},
    "no-rowconv": {"PT_B200_NO_ROWCONV": "1"},
    "no-s2d": {"PT_B200_NO_S2D": "1"},
    "rowdgrad-horizontal": {"PT_B200_ROWDGRAD": "0"},
    "rowconv-epi4": {"PT_B200_ROWCONV_EPI": "4"},
    "serial-bwd": {"PT_B200_BWD_STREAMS": "0"},
    "scbwd-off": {"PT_B200_SCBWD": "0"},
}


def _extra(cfg):
    """Each engine's own edge geometries on top of the common set."""
    from test_gpu_conv import HANKEL_EDGE, HWGRAD_EDGE, SMALLC_GEOMS
    if cfg.startswith("hankel"):
        return HANKEL_EDGE
    if cfg.startswith("hwgrad"):
        return HWGRAD_EDGE
    if cfg in ("swgrad-off", "no-rowconv", "rowdgrad-horizontal", "rowconv-epi4"):
        return SMALLC_GEOMS
    if cfg == "default":
        return SMALLC_EDGE
    return []


# more small-C stride-1 shapes through the default engines: odd batch, borders, C = 1 / 2 / 4,
# K not a multiple of 16, kH = 2 / 13, rows not 16-byte aligned (oW % 4 != 0), wide rows
SMALLC_EDGE = [
    po.geom(3, 3, 40, 40, 96, 11, 11, 0, 0, 1, 1),
    po.geom(1, 1, 50, 37, 40, 9, 7, 3, 2, 1, 1),
    po.geom(2, 2, 33, 100, 64, 5, 13, 2, 6, 1, 1),
    po.geom(3, 3, 19, 22, 16, 2, 3, 1, 1, 1, 1),
    po.geom(2, 3, 44, 70, 72, 13, 9, 6, 4, 1, 1),
    po.geom(5, 4, 26, 36, 24, 5, 5, 0, 4, 1, 1),
    po.geom(2, 3, 20, 302, 32, 3, 3, 1, 1, 1, 1),
]


@pytest.mark.parametrize("cfg", list(CONFIGS))
def test_engine_exact_and_tf32(cfg):
    geoms = GEOMS + _extra(cfg)
    specs = [[g.N, g.C, g.H, g.W, g.K, g.kH, g.kW, g.padH, g.padW, g.strideH, g.strideW]
             for g in geoms]
    env = dict(os.environ, **CONFIGS[cfg])
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "engine_check.py"),
                        json.dumps(specs)], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    fails = [f for e in res for f in e["fails"]]
    assert not fails, f"{cfg}: {len(fails)} failures\n" + "\n".join(fails[:6])
    worst = max(max(e["rels"].values()) for e in res)
    print(f"{cfg}: {len(geoms)} geometries exact + elementwise TF32, worst normwise {worst:.2e}; "
          + ", ".join(gstr(g) for g in geoms[:2]) + ", ...")
