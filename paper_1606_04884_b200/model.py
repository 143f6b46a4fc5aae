"""Model-stack layer: ModelSpecs of chained conv / pool-max / relu layers, their device
execution through the C ABI, and the bench harness of the reference's bench-cli module
(SPEC.md:462-520): bench_model (per-layer CSV (index,type,geometry,mean_time_s,checksum)
plus a per-layer-type summary), model_spec_load (bundled
alexnet / vgg-a or a spec file, shape-chain validated, :493-501) and bench_apply (the
per-element bandwidth sweep of the paper's Fig. 1-2, :475-483).

Spec file format: one layer per line,
    conv C H W K kH kW padH padW sH sW
    poolmax kH kW sH sW
    relu
('#' starts a comment). The first layer fixes the input C x H x W; every conv line's C H W
must equal the previous layer's output (a break is a ValidationError naming the layer).

Scale divisor (desk-scale runs): every channel count except the
image's input channels is divided by `scale`, which must divide them all (VGG-A: 7 does
not divide 64 -> error); spatial extents are kept so the pooling chain stays valid.

All compute is libpt_b200.so (conv passes, pt_b200_relu_*, pt_b200_maxpool_*,
pt_b200_reduce_all for the checksum); torch provides device memory, streams and events.
"""
from __future__ import annotations

import csv
import ctypes as C
import io
import os
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

from ._lib import ValidationError, check, lib

# convnet-benchmarks / public model definitions, conv stacks (the FC layers of VGG-A's 11
# weight layers are outside the three layer types of SPEC.md:470)
BUNDLED = {
    "alexnet": """
        # OWT AlexNet (convnet-benchmarks), 3x224x224
        conv 3 224 224 64 11 11 2 2 4 4
        relu
        poolmax 3 3 2 2
        conv 64 27 27 192 5 5 2 2 1 1
        relu
        poolmax 3 3 2 2
        conv 192 13 13 384 3 3 1 1 1 1
        relu
        conv 384 13 13 256 3 3 1 1 1 1
        relu
        conv 256 13 13 256 3 3 1 1 1 1
        relu
        poolmax 3 3 2 2
    """,
    "vgg-a": """
        # VGG model A (Simonyan & Zisserman), conv stack, 3x224x224
        conv 3 224 224 64 3 3 1 1 1 1
        relu
        poolmax 2 2 2 2
        conv 64 112 112 128 3 3 1 1 1 1
        relu
        poolmax 2 2 2 2
        conv 128 56 56 256 3 3 1 1 1 1
        relu
        conv 256 56 56 256 3 3 1 1 1 1
        relu
        poolmax 2 2 2 2
        conv 256 28 28 512 3 3 1 1 1 1
        relu
        conv 512 28 28 512 3 3 1 1 1 1
        relu
        poolmax 2 2 2 2
        conv 512 14 14 512 3 3 1 1 1 1
        relu
        conv 512 14 14 512 3 3 1 1 1 1
        relu
        poolmax 2 2 2 2
    """,
}

IMPLS = {"implicitgemm-sm100a": "tf32", "implicitgemm-3xtf32-sm100a": "3xtf32",
         "implicitgemm-fp32-sm100a": "fp32"}


@dataclass
class LayerSpec:
    kind: str                 # "conv" | "poolmax" | "relu"
    params: Tuple[int, ...]   # conv: C H W K kH kW pH pW sH sW; poolmax: kH kW sH sW


@dataclass
class ModelSpec:
    name: str
    layers: List[LayerSpec]


@dataclass
class Layer:
    """A concrete layer of a chained model at a batch size: input / output shapes."""
    index: int
    kind: str
    in_shape: Tuple[int, int, int, int]
    out_shape: Tuple[int, int, int, int]
    params: Tuple[int, ...] = ()
    geom: Optional[object] = None   # conv.ConvGeometry

    def geometry(self) -> str:
        N, Cc, H, W = self.in_shape
        if self.kind == "conv":
            return self.geom.toString()
        if self.kind == "poolmax":
            kH, kW, sH, sW = self.params
            return f"N{N} C{Cc} H{H} W{W} k{kH}x{kW} s{sH}x{sW}"
        return f"N{N} C{Cc} H{H} W{W}"


def parse_spec(text: str, name: str = "spec") -> ModelSpec:
    layers = []
    for ln, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].split()
        if not line:
            continue
        kind, args = line[0], line[1:]
        want = {"conv": 10, "poolmax": 4, "relu": 0}.get(kind)
        if want is None:
            raise ValidationError(f"model spec {name}: line {ln}: unknown layer type '{kind}'")
        if len(args) != want:
            raise ValidationError(f"model spec {name}: line {ln}: '{kind}' takes {want} integers")
        try:
            vals = tuple(int(a) for a in args)
        except ValueError:
            raise ValidationError(f"model spec {name}: line {ln}: non-integer argument") from None
        layers.append(LayerSpec(kind, vals))
    if not layers or layers[0].kind != "conv":
        raise ValidationError(f"model spec {name}: the first layer must be a conv (it fixes the input)")
    return ModelSpec(name, layers)


def model_spec_load(name_or_path: str) -> ModelSpec:
    """Bundled name (alexnet, vgg-a) or a spec file path."""
    if name_or_path in BUNDLED:
        spec = parse_spec(BUNDLED[name_or_path], name_or_path)
    elif os.path.isfile(name_or_path):
        with open(name_or_path) as f:
            spec = parse_spec(f.read(), os.path.basename(name_or_path))
    else:
        raise ValidationError(f"unknown model '{name_or_path}' (bundled: {', '.join(BUNDLED)})")
    chain(spec, 1, 1)  # validate the shape chain
    return spec


def chain(spec: ModelSpec, batch: int, scale: int = 1) -> List[Layer]:
    """Concrete layers at `batch` images and channel divisor `scale`; raises
    ValidationError at the first layer whose input does not match its predecessor."""
    from .conv import ConvGeometry
    if batch < 1 or scale < 1:
        raise ValidationError("batch and scale must be >= 1")
    img_c = spec.layers[0].params[0]

    def ch(c, i):
        if c == img_c and i == 0:
            return c
        if c % scale:
            raise ValidationError(f"model {spec.name}: scale {scale} does not divide the "
                                  f"{c} channels of layer {i}")
        return c // scale

    out: List[Layer] = []
    cur = None
    for i, l in enumerate(spec.layers):
        if l.kind == "conv":
            Cc, H, W, K, kH, kW, pH, pW, sH, sW = l.params
            shape_in = (batch, ch(Cc, i), H, W)
            if cur is not None and shape_in != cur:
                raise ValidationError(f"model {spec.name}: shape chain break at layer {i}: conv expects "
                                      f"{shape_in[1:]} but the previous layer gives {cur[1:]}")
            g = ConvGeometry(batch, shape_in[1], H, W, ch(K, i), kH, kW, pH, pW, sH, sW)
            try:
                g.validate()
            except ValidationError as ex:
                raise ValidationError(f"model {spec.name}: layer {i}: {ex}") from None
            cur = g.output_shape()
            out.append(Layer(i, "conv", shape_in, cur, l.params, g))
        elif l.kind == "poolmax":
            kH, kW, sH, sW = l.params
            N, Cc, H, W = cur
            if min(kH, kW, sH, sW) < 1 or kH > H or kW > W:
                raise ValidationError(f"model {spec.name}: shape chain break at layer {i}: "
                                      f"pool {kH}x{kW} on {H}x{W}")
            o = (N, Cc, (H - kH) // sH + 1, (W - kW) // sW + 1)
            out.append(Layer(i, "poolmax", cur, o, l.params))
            cur = o
        else:
            out.append(Layer(i, "relu", cur, cur))
    return out


class Model:
    """Device-resident instance of a chained model: weights, activations, gradients and
    Torch's finput per conv; forward / backward per layer through the C ABI."""

    def __init__(self, layers: Sequence[Layer], math: str = "tf32", seed: int = 0x5EED,
                 device=None):
        import torch
        from . import conv as cv
        self.torch, self.cv, self.math = torch, cv, math
        self.layers = list(layers)
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        e = lambda shape: torch.empty(shape, device=dev)  # noqa: E731
        self.x = cv.fill_uniform(e(self.layers[0].in_shape), seed)
        self.st: List[Dict] = []
        for l in self.layers:
            s: Dict = {"y": e(l.out_shape), "gx": e(l.in_shape)}
            if l.kind == "conv":
                g = l.geom
                a = 1.0 / (g.patchSize()) ** 0.5
                s["w"] = cv.fill_uniform(e(g.weight_shape()), seed + 31 * l.index + 1, -a, a)
                s["b"] = cv.fill_uniform(e((g.outChannels,)), seed + 31 * l.index + 2, -0.1, 0.1)
                s["gw"] = e(g.weight_shape())
                s["gb"] = e((g.outChannels,))
                nb = cv.finput_bytes(g, math)
                s["finput"] = torch.empty(nb, dtype=torch.uint8, device=dev) if nb else None
            elif l.kind == "poolmax":
                s["arg"] = torch.empty(l.out_shape, dtype=torch.int32, device=dev)
            self.st.append(s)
        self.gy = cv.fill_uniform(e(self.layers[-1].out_shape), seed + 7, -1e-3, 1e-3)

    def input_of(self, i):
        return self.x if i == 0 else self.st[i - 1]["y"]

    def grad_of(self, i):
        return self.gy if i == len(self.layers) - 1 else self.st[i + 1]["gx"]

    def forward_layer(self, i):
        l, s, x = self.layers[i], self.st[i], self.input_of(i)
        stream = self.torch.cuda.current_stream().cuda_stream
        if l.kind == "conv":
            self.cv.conv_forward(l.geom, x, s["w"], s["b"], s["y"], math=self.math, finput=s["finput"])
        elif l.kind == "relu":
            check(lib().pt_b200_relu_fwd(x.data_ptr(), s["y"].data_ptr(), x.numel(), stream))
        else:
            N, Cc, H, W = l.in_shape
            kH, kW, sH, sW = l.params
            check(lib().pt_b200_maxpool_fwd(x.data_ptr(), s["y"].data_ptr(), s["arg"].data_ptr(),
                                            N, Cc, H, W, kH, kW, sH, sW, 0, 0, stream))

    def backward_layer(self, i):
        l, s, x, gy = self.layers[i], self.st[i], self.input_of(i), self.grad_of(i)
        stream = self.torch.cuda.current_stream().cuda_stream
        if l.kind == "conv":
            self.cv.conv_backward(l.geom, x, gy, s["w"], s["gx"] if i > 0 else None, s["gw"],
                                  s["gb"], need_input_grad=i > 0, math=self.math,
                                  finput=s["finput"])
        elif l.kind == "relu":
            check(lib().pt_b200_relu_bwd(s["y"].data_ptr(), gy.data_ptr(), s["gx"].data_ptr(),
                                         gy.numel(), stream))
        else:
            N, Cc, H, W = l.in_shape
            kH, kW, sH, sW = l.params
            check(lib().pt_b200_maxpool_bwd(gy.data_ptr(), s["arg"].data_ptr(), s["gx"].data_ptr(),
                                            N, Cc, H, W, kH, kW, sH, sW, 0, 0, stream))

    def forward(self):
        for i in range(len(self.layers)):
            self.forward_layer(i)
        return self.st[-1]["y"]

    def backward(self):
        for i in reversed(range(len(self.layers))):
            self.backward_layer(i)

    def checksum(self, i) -> float:
        """Sum of layer i's forward output (pt_b200_reduce_all)."""
        from ._lib import PtView
        y = self.st[i]["y"]
        v = PtView()
        v.ndim = 1
        v.sizes[0] = y.numel()
        v.strides[0] = 1
        v.offset = 0
        out = self.torch.empty(1, device=self.dev)
        check(lib().pt_b200_reduce_all(0, y.data_ptr(), C.byref(v), out.data_ptr(),
                                       self.torch.cuda.current_stream().cuda_stream))
        return float(out.item())


def bench_model(spec: ModelSpec, scale: int = 1, batch: int = 1, backward: bool = False,
                impl: Optional[str] = None, reps: int = 5) -> Tuple[List[dict], List[dict]]:
    """Per-layer forward (or forward+backward) device time, mean over `reps` repetitions
    after one excluded warm-up; CUDA events per layer on the
    current stream. Returns (rows, summary)."""
    import torch
    if reps < 3:
        raise ValidationError("bench_model: repetitions must be >= 3")
    impl = impl or "implicitgemm-sm100a"
    if impl not in IMPLS:
        raise ValidationError(f"unknown conv implementation '{impl}' ({', '.join(IMPLS)})")
    layers = chain(spec, batch, scale)
    m = Model(layers, math=IMPLS[impl])
    n = len(layers)
    tot = [0.0] * n
    for rep in range(reps + 1):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(n)]
        bev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(n)]
        for i in range(n):
            ev[i][0].record()
            m.forward_layer(i)
            ev[i][1].record()
        if backward:
            for i in reversed(range(n)):
                bev[i][0].record()
                m.backward_layer(i)
                bev[i][1].record()
        torch.cuda.synchronize()
        if rep == 0:
            continue  # the first iteration is excluded
        for i in range(n):
            tot[i] += ev[i][0].elapsed_time(ev[i][1]) * 1e-3
            if backward:
                tot[i] += bev[i][0].elapsed_time(bev[i][1]) * 1e-3
    rows = [{"index": l.index, "type": l.kind, "geometry": l.geometry(),
             "mean_time_s": tot[i] / reps, "checksum": m.checksum(i)}
            for i, l in enumerate(layers)]
    total = sum(r["mean_time_s"] for r in rows)
    summary = []
    for kind in ("conv", "poolmax", "relu"):
        t = sum(r["mean_time_s"] for r in rows if r["type"] == kind)
        k = sum(1 for r in rows if r["type"] == kind)
        if k:
            summary.append({"type": kind, "layers": k, "total_time_s": t,
                            "fraction": t / total if total > 0 else 0.0})
    return rows, summary


def bench_apply(sizes: Sequence[int], reps: int = 5, expression: str = "x = x * s",
                scalar: float = 1.0001) -> List[dict]:
    """Per-element bandwidth sweep: `reps` back-to-back
    launches of one contiguous apply on `size` floats through pt_b200_apply, after one
    excluded warm-up launch (the "compile" iteration: the expression is compiled once, as
    the reference's kernel cache would), timed with CUDA events; bandwidth = size * 4 B * 2
    (one read + one write) / mean time per launch. Small sizes measure the launch overhead,
    large ones HBM (the two regimes of the paper's Fig. 1). A size whose allocation fails
    gives a row marked skipped."""
    import torch
    from ._lib import PtView
    from .expr import parse
    if reps < 3:
        raise ValidationError("bench_apply: repetitions must be >= 3")
    if not sizes or list(sizes) != sorted(sizes) or min(sizes) < 1:
        raise ValidationError("bench_apply: sizes must be ascending and >= 1")
    prog = parse(expression, 1)
    code = (C.c_int32 * len(prog.code))(*prog.code)
    rows = []
    for n in sizes:
        n = int(n)
        try:
            x = torch.ones(n, device="cuda")
        except RuntimeError:
            rows.append({"size": n, "reps": reps, "mean_time_s": None, "gb_per_s": None,
                         "skipped": True})
            continue
        v = (PtView * 3)()
        v[0].ndim, v[0].sizes[0], v[0].strides[0], v[0].offset = 1, n, 1, 0
        bases = (C.c_void_p * 3)(x.data_ptr(), None, None)
        st = torch.cuda.current_stream().cuda_stream
        launch = lambda: check(lib().pt_b200_apply(code, len(prog.code), 1, bases, v,  # noqa: E731
                                                   float(scalar), st))
        launch()  # excluded first iteration
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            launch()
        e1.record()
        e1.synchronize()
        mean = e0.elapsed_time(e1) * 1e-3 / reps
        rows.append({"size": n, "reps": reps, "mean_time_s": mean,
                     "gb_per_s": n * 4 * 2 / mean / 1e9})
        del x
    return rows


def to_csv(rows: List[dict], columns: Sequence[str]) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(columns)
    for r in rows:
        w.writerow(["skipped" if r.get("skipped") and r.get(c) is None else
                    (f"{r[c]:.9g}" if isinstance(r[c], float) else r[c]) for c in columns])
    return buf.getvalue()


LAYER_COLUMNS = ("index", "type", "geometry", "mean_time_s", "checksum")
SUMMARY_COLUMNS = ("type", "layers", "total_time_s", "fraction")
BANDWIDTH_COLUMNS = ("size", "reps", "mean_time_s", "gb_per_s")
