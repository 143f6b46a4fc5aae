#!/usr/bin/env python3
"""bench.py — conv fwd+bwd GFLOP/s of the sm_100a SpatialConvolutionMM path.

Metric (BASELINE.json): "conv fwd+bwd GFLOP/s (convnet-benchmarks L1-L5)". One step =
one fwd + bwd pass (updateOutput, updateGradInput, accGradParameters incl. gradBias)
of every layer of the workload over one synthetic batch; FLOPs = 3 * 2*N*K*CRS*oH*oW
per layer (fprop + dgrad + wgrad; bias work excluded).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload convnet|alexnet|...]
  python bench.py --impl reference ...   # the CPU reference path (oracle port), same metric

Multi-GPU (torchrun, one rank per GPU): strong scaling — the workload's fixed global batch
is sharded over the ranks (dp.shard_range; e.g. AlexNet 128 -> 16 images per GPU at 8),
and gradWeight/gradBias are all-reduced with NCCL per layer on a communication stream
overlapping the next layer's kernels; `value` = the global batch's FLOPs / the max-over-
ranks step time. The line also carries `alexnet.ms_per_batch` (the metric's second half:
AlexNet conv stack fwd+bwd per global batch of 128 at this N).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# (name, N, C, H, W, K, kH, kW, padH, padW, strideH, strideW)
WORKLOADS = {
    "convnet": [  # convnet-benchmarks layerwise suite (pad 0), BASELINE.json configs[1]
        ("L1", 128, 3, 128, 128, 96, 11, 11, 0, 0, 1, 1),
        ("L2", 128, 64, 64, 64, 128, 9, 9, 0, 0, 1, 1),
        ("L3", 128, 128, 32, 32, 128, 9, 9, 0, 0, 1, 1),
        ("L4", 128, 128, 16, 16, 128, 7, 7, 0, 0, 1, 1),
        ("L5", 128, 384, 13, 13, 384, 3, 3, 0, 0, 1, 1),
    ],
    "cfg1": [("cfg1", 16, 3, 32, 32, 64, 3, 3, 1, 1, 1, 1)],
    "alexnet": [  # OWT AlexNet conv stack, batch 128, 224x224 (configs[2])
        ("c1", 128, 3, 224, 224, 64, 11, 11, 2, 2, 4, 4),
        ("c2", 128, 64, 27, 27, 192, 5, 5, 2, 2, 1, 1),
        ("c3", 128, 192, 13, 13, 384, 3, 3, 1, 1, 1, 1),
        ("c4", 128, 384, 13, 13, 256, 3, 3, 1, 1, 1, 1),
        ("c5", 128, 256, 13, 13, 256, 3, 3, 1, 1, 1, 1),
    ],
    "overfeat": [  # Overfeat-fast, batch 128, 231x231 (configs[3])
        ("c1", 128, 3, 231, 231, 96, 11, 11, 0, 0, 4, 4),
        ("c2", 128, 96, 24, 24, 256, 5, 5, 0, 0, 1, 1),
        ("c3", 128, 256, 12, 12, 512, 3, 3, 1, 1, 1, 1),
        ("c4", 128, 512, 12, 12, 1024, 3, 3, 1, 1, 1, 1),
        ("c5", 128, 1024, 12, 12, 1024, 3, 3, 1, 1, 1, 1),
    ],
    "vgga": [  # VGG-A conv stack, batch 64, 224x224 (configs[4])
        ("c1", 64, 3, 224, 224, 64, 3, 3, 1, 1, 1, 1),
        ("c2", 64, 64, 112, 112, 128, 3, 3, 1, 1, 1, 1),
        ("c3", 64, 128, 56, 56, 256, 3, 3, 1, 1, 1, 1),
        ("c4", 64, 256, 56, 56, 256, 3, 3, 1, 1, 1, 1),
        ("c5", 64, 256, 28, 28, 512, 3, 3, 1, 1, 1, 1),
        ("c6", 64, 512, 28, 28, 512, 3, 3, 1, 1, 1, 1),
        ("c7", 64, 512, 14, 14, 512, 3, 3, 1, 1, 1, 1),
        ("c8", 64, 512, 14, 14, 512, 3, 3, 1, 1, 1, 1),
    ],
}
METRIC = "conv fwd+bwd GFLOP/s (convnet-benchmarks L1-L5)"


def layer_flops(l) -> float:
    _, N, C, H, W, K, kH, kW, pH, pW, sH, sW = l
    oH = (H + 2 * pH - kH) // sH + 1
    oW = (W + 2 * pW - kW) // sW + 1
    return 3.0 * 2.0 * N * K * C * kH * kW * oH * oW


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="convnet", choices=list(WORKLOADS))
    ap.add_argument("--math", default="tf32", choices=["tf32", "3xtf32", "fp32"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--emulate-ranks", type=int, default=1,
                    help="N=1 only: run rank 0's shard of a G-rank strong-scaling job (compute "
                         "of one rank, no collective) and report the projected job throughput")
    ap.add_argument("--no-alexnet", action="store_true",
                    help="skip the AlexNet ms/batch leg (the metric's second half)")
    ap.add_argument("--no-finput", action="store_true", help="re-lay x out in the weight gradient")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the step eagerly instead of replaying each layer's CUDA graph")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling DURING the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons, pw = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        top = max(sm)
        loaded = [s for s in sm if s >= 0.5 * top] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(pw) if pw else None}


# ---------------------------------------------------------------------------- peaks
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def measure_cublas_tf32(torch):
    """cuBLAS TF32 8192^3 (burst, best of 5) — the on-box TF32 dense denominator."""
    try:
        torch.backends.cuda.matmul.allow_tf32 = True
        n = 8192
        a = torch.randn(n, n, device="cuda")
        b = torch.randn(n, n, device="cuda")
        for _ in range(3):
            a @ b
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            a @ b
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b
        torch.cuda.empty_cache()
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12
    except Exception:
        return None


def ncu_traffic(workload, key):
    """dram__bytes_read.sum + dram__bytes_write.sum of this launch from the committed
    `ncu --set full` capture (profiles/ncu_traffic.json), or None when not captured."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        v = t.get(f"{workload}/{key}")
        return None if v is None else {"bytes": v["bytes"], "source": v["source"]}
    except Exception:
        return None


# ---------------------------------------------------------------------------- CPU legs
def cpu_sample_run(layers, batch, threads):
    """One fwd+bwd of every layer at `batch` images through the oracle port (im2col +
    blocked SGEMM + col2im). Returns (seconds, flops)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    t = 0.0
    fl = 0.0
    for l in layers:
        _, N, C, H, W, K, kH, kW, pH, pW, sH, sW = l
        g = po.geom(batch, C, H, W, K, kH, kW, pH, pW, sH, sW)
        oh, ow = po.out_hw(g)
        x = po.uniform((batch, C, H, W), 1)
        w = po.uniform((K, C, kH, kW), 2, -0.1, 0.1)
        b = po.uniform((K,), 3, -0.1, 0.1)
        gy = po.uniform((batch, K, oh, ow), 4)
        t0 = time.perf_counter()
        po.conv_forward(g, x, w, b, chunk=1, threads=threads)
        po.conv_backward_input(g, gy, w, threads=threads)
        po.conv_backward_weight(g, x, gy, threads=threads)
        t += time.perf_counter() - t0
        fl += layer_flops((l[0], batch) + tuple(l[2:]))
    return t, fl


def cpu_model():
    """The host CPU model (/proc/cpuinfo), recorded beside the CPU baseline's core count."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(layers, budget_s):
    threads = os.cpu_count() or 1
    t1, f1 = cpu_sample_run(layers, 1, threads)
    batch = 1
    if t1 > 0 and t1 < budget_s / 2:
        batch = max(1, min(layers[0][1], int(budget_s / t1)))
        t1, f1 = cpu_sample_run(layers, batch, threads)
    return {"value": f1 / t1 / 1e9, "unit": "GFLOP/s", "cores": threads, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{batch} image(s) per layer, fwd+bwd of every layer, oracle im2col+"
                      f"blocked SGEMM+col2im (oracle/oracle.c), {threads} OpenMP threads, "
                      f"{t1:.1f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    layers = WORKLOADS[args.workload]
    threads = os.cpu_count() or 1
    # bounded sample per step: 8 images per layer (the full batch would take many minutes;
    # one image per call under-fills the host threads: 196 vs 213 GFLOP/s on 16 cores)
    nimg = 8
    for _ in range(args.warmup):
        cpu_sample_run(layers, 1, threads)
    tt, ff = 0.0, 0.0
    for _ in range(args.steps):
        t, f = cpu_sample_run(layers, nimg, threads)
        tt += t
        ff += f
    v = ff / tt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic (counter-based uniform)",
        "config": {"workload": args.workload, "layers": [l[0] for l in layers],
                   "sample_batch_per_layer": nimg, "full_batch": layers[0][1]},
        "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"{nimg} images per layer per step, fwd+bwd, oracle port "
                                   "(im2col + blocked SGEMM + col2im); the reference ships no "
                                   "conv implementation (SURVEY.md §0)"},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU arm
def local_layers(layers, rank, world):
    """Strong scaling (north_star): the workload's FIXED global batch is
    sharded over the ranks (dp.shard_range: AlexNet 128 -> 64/32/16 per GPU, VGG-A 64 ->
    32/16/8); every rank holds the full weights; the gradients are all-reduced."""
    from paper_1606_04884_b200.dp import shard_range
    out = []
    for l in layers:
        lo, hi = shard_range(l[1], rank, world)
        out.append((l[0], hi - lo) + tuple(l[2:]))
    return out


class Workload:
    """One rank's share of a workload: per layer the device buffers, Torch's finput, the
    gradient bucket, and (after capture()) one CUDA graph of the layer's fwd + bwd."""

    def __init__(self, pt, torch, layers, dev, rank, math, use_finput=True):
        from paper_1606_04884_b200.dp import GradBucket
        self.pt, self.torch, self.math, self.dev = pt, torch, math, dev
        self.layers = layers
        self.st = []
        for i, l in enumerate(layers):
            name, N, C, H, W, K, kH, kW, pH, pW, sH, sW = l
            g = pt.ConvGeometry(N, C, H, W, K, kH, kW, pH, pW, sH, sW)
            seed = 0x5EED + 101 * i + 7919 * rank
            x = pt.fill_uniform(torch.empty(g.input_shape(), device=dev), seed + 1)
            s = 1.0 / (C * kH * kW) ** 0.5
            w = pt.fill_uniform(torch.empty(g.weight_shape(), device=dev), seed + 2, -s, s)
            b = pt.fill_uniform(torch.empty((K,), device=dev), seed + 3, -0.1, 0.1)
            gy = pt.fill_uniform(torch.empty(g.output_shape(), device=dev), seed + 4)
            bucket = GradBucket([torch.Size(g.weight_shape()), torch.Size((K,))], dev)
            fb = pt.finput_bytes(g, math) if use_finput else 0
            finput = torch.empty(fb, dtype=torch.uint8, device=dev) if fb else None
            self.st.append(dict(name=name, finput=finput, g=g, x=x, w=w, b=b, gy=gy,
                                y=torch.empty(g.output_shape(), device=dev),
                                gx=torch.empty(g.input_shape(), device=dev), bucket=bucket,
                                gw=bucket.views[0], gb=bucket.views[1]))
        self.graphs = None
        self.graph_launches = 0

    def layer(self, s):
        from paper_1606_04884_b200 import _lib as L
        pt, g = self.pt, s["g"]
        L.lib().pt_b200_profile_tag(s["name"].encode())
        # Torch's finput: the forward's relaid input is reused by accGradParameters
        pt.conv_forward(g, s["x"], s["w"], s["b"], s["y"], math=self.math, finput=s["finput"])
        pt.conv_backward(g, s["x"], s["gy"], s["w"], s["gx"], s["gw"], s["gb"], math=self.math,
                         finput=s["finput"])

    def step(self, comm=None, eager=False):
        from paper_1606_04884_b200.dp import allreduce_async
        cur = self.torch.cuda.current_stream()
        done = []
        for i, s in enumerate(self.st):
            if self.graphs is None or eager:
                self.layer(s)
            elif self.graphs[i] is not None:
                self.graphs[i].replay()
            # batch-sharded DP: one allreduce(sum) of this layer's gradW||gradB bucket on the
            # comm stream, overlapping the next layer's kernels
            done.append(allreduce_async(s["bucket"], comm))
        for ev in done:
            if ev is not None:
                cur.wait_event(ev)

    def capture(self, one_graph=False):
        """Each layer's forward + combined backward (internal streams included) captured
        once as a CUDA graph on a side stream whose workspace is warmed (allocated) first,
        so nothing allocates during capture; the allreduce stays an eager NCCL call between
        the replays, so every N runs the same kernels the same way. one_graph (one rank, no
        allreduce): all layers in one graph."""
        torch, pt = self.torch, self.pt
        cur = torch.cuda.current_stream()
        side = torch.cuda.Stream(device=self.dev)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            for s in self.st:
                self.layer(s)
        side.synchronize()
        graphs = []
        c0 = pt.launch_count()
        if one_graph:
            # one rank: no allreduce between the layers, so the whole step is one graph (the
            # same kernels; 1-2 % faster than one replay per layer, BENCH_ONE_GRAPH A/B)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=side, capture_error_mode="thread_local"):
                for s in self.st:
                    self.layer(s)
            graphs = [gr] + [None] * (len(self.st) - 1)
        else:
          for s in self.st:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=side, capture_error_mode="thread_local"):
                self.layer(s)
            graphs.append(gr)
        self.graph_launches = pt.launch_count() - c0
        self.graphs = graphs
        torch.cuda.synchronize()

    def bytes_working_set(self):
        return sum(4 * (s["x"].numel() + s["y"].numel() + s["gy"].numel() + s["gx"].numel())
                   for s in self.st)


def timed(torch, dist, world, run, steps):
    """Device time of `steps` calls of run(): barrier + synchronize on both sides, CUDA
    events on the current stream, max over ranks."""
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        run()
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1606_04884_b200 as pt
    from paper_1606_04884_b200 import _lib as L

    glayers = WORKLOADS[args.workload]
    emu = args.emulate_ranks if world == 1 else 1
    layers = local_layers(glayers, rank, world) if emu == 1 else local_layers(glayers, 0, emu)
    dev = torch.device("cuda", local)
    wl = Workload(pt, torch, layers, dev, rank, args.math, use_finput=not args.no_finput)
    st = wl.st
    comm = torch.cuda.Stream(device=dev) if world > 1 else None

    for _ in range(max(3, args.warmup)):
        wl.step(comm)
    torch.cuda.synchronize()

    peaks, peak_kind = load_peaks()
    clocks = ClockSampler(local)
    L.lib().pt_b200_profile_enable(0)
    L.lib().pt_b200_set_bwd_streams(int(os.environ.get("BENCH_BWD_STREAMS", "1")))
    graph = None
    if not args.no_graph:
        try:
            wl.capture(one_graph=world == 1 and os.environ.get("BENCH_ONE_GRAPH", "1") != "0")
            for _ in range(2):
                wl.step(comm)
            torch.cuda.synchronize()
            graph = wl.graphs
        except Exception as ex:  # pragma: no cover - eager launches instead
            print(f"bench: CUDA-graph capture failed ({ex}); timing eager launches", file=sys.stderr)
            torch.cuda.synchronize()
            wl.graphs = None
    launches0 = pt.launch_count()
    clocks.start()
    time.sleep(0.3)
    ms = timed(torch, dist, world, lambda: wl.step(comm), args.steps)
    clk = clocks.stop()
    launches = pt.launch_count() - launches0 + wl.graph_launches * args.steps * (graph is not None)
    # per-launch kernel timings: a second pass of the same steps with the backward's two
    # streams serialised — in the timed region the input- and weight-gradient kernels run
    # concurrently, so per-launch event spans there would overlap
    L.lib().pt_b200_set_bwd_streams(0)
    L.lib().pt_b200_profile_enable(1)
    L.lib().pt_b200_profile_reset()
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record()
    for _ in range(args.steps):
        wl.step(comm, eager=True)
    p1.record()
    torch.cuda.synchronize()
    ms_serial = p0.elapsed_time(p1)
    prof = {c: L.profile_read(c) for c in ("umma_conv", "umma_wgrad", "simt_conv", "layout")}
    ms_step = ms / args.steps
    flops_step = sum(layer_flops(l) for l in glayers)  # the global batch's work
    value = flops_step / (ms_step * 1e-3) / 1e9

    # roofline of the dominant kernel: the (layer, pass) tensor-core launch with the
    # largest device time inside the timed region (CUDA events on its own stream)
    per = {}
    for s_ in st:
        for cls in ("umma_conv", "umma_wgrad", "simt_conv"):
            for ps in ("fwd", "dgrad", "wgrad", "bwd"):  # bwd: the fused small-C backward
                v = L.profile_read(f"{cls}@{s_['name']}.{ps}")
                if v[1] > 0:
                    per[f"{cls}@{s_['name']}.{ps}"] = v
    # HBM-bound layout passes (NCHW<->NHWC, space-to-depth) per (layer, pass)
    lay = {}
    for s_ in st:
        for ps in ("fwd", "bwd", "dgrad", "wgrad"):
            v = L.profile_read(f"layout@{s_['name']}.{ps}")
            if v[1] > 0:
                lay[f"{s_['name']}.{ps}"] = {"ms": v[0] / args.steps, "launches": v[1] // args.steps,
                                             "gbs": v[3] / (v[0] * 1e-3) / 1e9 if v[0] > 0 else None}
    L.lib().pt_b200_profile_enable(0)
    L.lib().pt_b200_set_bwd_streams(1)
    tf32_cublas = measure_cublas_tf32(torch) if rank == 0 else None
    tf32_derived = peaks.get("bf16_tflops", 1590.0) / 2.0
    # denominator: the measured TF32 tensor-pipe ceiling of this GPU (back-to-back MMAs,
    # pt_b200_tf32_mma_peak); cuBLAS TF32 and MEASURED_PEAKS bf16/2 are reported beside it
    tf32_mma = float(L.lib().pt_b200_tf32_mma_peak()) if rank == 0 else -1.0
    peak_tf = max(tf32_mma, tf32_derived, tf32_cublas or 0.0)
    dom = max(per, key=lambda k: per[k][0])
    dms, dn, dfl, dby = per[dom]
    avg_ms = dms / dn
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    if dby > 0 and dfl / dby < peak_tf * 1e12 / (hbm_peak * 1e9):
        # below the ridge point (e.g. the fused small-C backward: 11 GFLOP over 0.9 GB): the
        # HBM roofline binds; achieved = its algorithmic bytes per launch / launch time
        roof = {"bound": "hbm", "achieved": dby / dn / (avg_ms * 1e-3) / 1e9, "peak": hbm_peak,
                "unit": "GB/s", "tensor_tflops": dfl / dn / (avg_ms * 1e-3) / 1e12}
    else:
        roof = {"bound": "tensor", "achieved": dfl / dn / (avg_ms * 1e-3) / 1e12, "peak": peak_tf,
                "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = ncu_traffic(args.workload, dom)
    roof["kernel"] = dom
    roof["avg_launch_ms"] = avg_ms
    roof["flops_per_launch"] = dfl / dn
    roof["bytes_per_launch"] = dby / dn
    roof["share_of_step"] = dms / ms_serial if ms_serial > 0 else None
    roof["step_frac"] = value / 1e3 / peak_tf
    roof["timing"] = ("per-launch CUDA events in a serialised, eagerly launched pass of the same steps "
                      f"right after the timed region ({ms_serial / args.steps:.3f} ms/step serialised vs "
                      f"{ms / args.steps:.3f} ms/step timed: backward's two streams, "
                      + ("CUDA-graph replay)" if graph is not None else "eager launches)"))
    if roof["bound"] == "hbm":
        roof["peak_source"] = f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}, copy bandwidth)"
    else:
        roof["peak_source"] = (f"max(measured TF32 MMA ceiling on this box = {tf32_mma:.1f} "
                               f"[pt_b200_tf32_mma_peak], cuBLAS TF32 8192^3 = {tf32_cublas}, "
                               f"{peak_kind} bf16 burst/2 = {tf32_derived:.1f})")
        roof["frac_vs_bf16_half"] = roof["achieved"] / tf32_derived
    roof["per_launch"] = {k: {"ms": v[0] / v[1], "tflops": v[2] / v[0] * 1e-9,
                              **({"gbs": v[3] / v[0] * 1e-6} if v[3] > 0 else {})}
                          for k, v in sorted(per.items())}

    result = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": args.math,
        "data": "synthetic (counter-based uniform, device-generated)",
        "config": {"workload": args.workload, "layers": [l[0] for l in layers],
                   "global_batch": glayers[0][1], "per_gpu_batch": layers[0][1],
                   "parallelism": f"dp{world}", "math": args.math,
                   "sharding": "fixed global batch split over the ranks (dp.shard_range); "
                               "gradWeight||gradBias all-reduced per layer (NCCL)",
                   "launch": ("eager" if graph is None else
                              "one CUDA-graph replay per step (all layers fwd + bwd; one rank)" if graph[-1] is None
                              else "one CUDA-graph replay per layer (fwd + bwd), allreduce eager"),
                   "l2": "no flush: per-step working set "
                         f"{wl.bytes_working_set() / 1e9:.2f} GB > 126 MB L2"},
        "clocks": clk, "gpu_launches": launches, "roofline": roof,
        "kernels": {c: {"ms": v[0], "launches": v[1], "tflops": (v[2] / (v[0] * 1e-3) / 1e12)
                        if v[0] > 0 and v[2] > 0 else None,
                        "gbs": (v[3] / (v[0] * 1e-3) / 1e9) if v[0] > 0 and v[3] > 0 else None}
                    for c, v in prof.items()},
        "layout_per_pass": lay,
    }
    if emu > 1:
        result["emulated_ranks"] = {
            "ranks": emu, "per_rank_batch": layers[0][1],
            "note": "one rank's shard timed alone on one GPU (no collective): `value` is the "
                    "projected throughput of the job if the allreduce overlaps fully"}
    del wl, st

    # the metric's second half: AlexNet conv stack ms per (global) batch of 128 at this N
    if args.workload != "alexnet" and not args.no_alexnet:
        result["alexnet"] = alexnet_ms_per_batch(args, pt, torch, dist, dev, rank, world)
    elif args.workload == "alexnet":
        result["alexnet"] = {"ms_per_batch": ms_step, "global_batch": glayers[0][1],
                             "per_gpu_batch": layers[0][1], "n_gpus": world}

    # e2e through the public API with HOST buffers (pinned), copies inside the timed region
    if not args.no_e2e:
        result["e2e"] = e2e(args, pt, torch, layers, glayers, dev, world, rank, dist)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            result["cpu_baseline"] = cpu_baseline(glayers, args.cpu_seconds)
        except Exception as ex:  # pragma: no cover
            result["cpu_baseline"] = {"value": None, "error": str(ex)}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def alexnet_ms_per_batch(args, pt, torch, dist, dev, rank, world):
    """AlexNet conv stack fwd+bwd, global batch 128 sharded over the ranks, CUDA-graph
    replay per layer (per step on one rank), allreduce per layer: device ms per global batch
    (max over ranks)."""
    glayers = WORKLOADS["alexnet"]
    layers = local_layers(glayers, rank, world)
    wl = Workload(pt, torch, layers, dev, rank, args.math)
    comm = torch.cuda.Stream(device=dev) if world > 1 else None
    for _ in range(3):
        wl.step(comm)
    wl.capture(one_graph=world == 1 and os.environ.get("BENCH_ONE_GRAPH", "1") != "0")
    for _ in range(2):
        wl.step(comm)
    steps = max(args.steps, 10)
    ms = timed(torch, dist, world, lambda: wl.step(comm), steps) / steps
    flops = sum(layer_flops(l) for l in glayers)
    return {"ms_per_batch": ms, "global_batch": glayers[0][1], "per_gpu_batch": layers[0][1],
            "n_gpus": world, "steps": steps, "gflops": flops / (ms * 1e-3) / 1e9,
            "timing": "CUDA events around `steps` CUDA-graph-replayed steps, max over ranks"}


def e2e(args, pt, torch, layers, glayers, dev, world, rank, dist):
    host = []
    for i, l in enumerate(layers):
        name, N, C, H, W, K, kH, kW, pH, pW, sH, sW = l
        g = pt.ConvGeometry(N, C, H, W, K, kH, kW, pH, pW, sH, sW)
        d = {k: torch.empty(shape, pin_memory=True) for k, shape in
             (("x", g.input_shape()), ("w", g.weight_shape()), ("b", (K,)),
              ("gy", g.output_shape()), ("y", g.output_shape()), ("gx", g.input_shape()),
              ("gw", g.weight_shape()), ("gb", (K,)))}
        for k in ("x", "w", "b", "gy"):
            d[k].uniform_(-1, 1)
        d["g"] = g
        fb = pt.finput_bytes(g, args.math)
        d["finput"] = torch.empty(fb, dtype=torch.uint8, device=dev) if fb else None
        host.append(d)
    h2d = sum(4 * (d["x"].numel() + d["w"].numel() + d["b"].numel() + d["gy"].numel())
              for d in host)
    d2h = sum(4 * (d["y"].numel() + d["gx"].numel() + d["gw"].numel() + d["gb"].numel())
              for d in host)

    # device-side buffers per layer; H2D of layer i+1 and D2H of layer i-1 run on their own
    # streams while layer i computes (PCIe is full duplex: both directions overlap compute)
    for d in host:
        for k in ("x", "w", "b", "gy", "y", "gx", "gw", "gb"):
            d["d" + k] = torch.empty(d[k].shape, device=dev)
        d["in_free"] = None
        d["out_free"] = None
    comp = torch.cuda.current_stream()
    h2d_s, d2h_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

    def step():
        # per layer: x/w/b then gy on the H2D stream (the forward needs only the first three),
        # y goes back as soon as the forward is done, while gy is still arriving — the big
        # first layer then moves its 0.7 GB each way concurrently instead of back to back
        for d in host:
            g = d["g"]
            with torch.cuda.stream(h2d_s):
                if d["in_free"] is not None:
                    h2d_s.wait_event(d["in_free"])
                for k in ("x", "w", "b"):
                    d["d" + k].copy_(d[k], non_blocking=True)
                ev_fwd_in = torch.cuda.Event()
                ev_fwd_in.record(h2d_s)
                d["dgy"].copy_(d["gy"], non_blocking=True)
                ev_gy = torch.cuda.Event()
                ev_gy.record(h2d_s)
            comp.wait_event(ev_fwd_in)
            if d["out_free"] is not None:
                comp.wait_event(d["out_free"])
            pt.conv_forward(g, d["dx"], d["dw"], d["db"], d["dy"], math=args.math, finput=d["finput"])
            ev_y = torch.cuda.Event()
            ev_y.record(comp)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(ev_y)
                d["y"].copy_(d["dy"], non_blocking=True)
            comp.wait_event(ev_gy)
            pt.conv_backward(g, d["dx"], d["dgy"], d["dw"], d["dgx"], d["dgw"], d["dgb"],
                             math=args.math, finput=d["finput"])
            if world > 1:
                dist.all_reduce(d["dgw"])
                dist.all_reduce(d["dgb"])
            ev_done = torch.cuda.Event()
            ev_done.record(comp)
            d["in_free"] = ev_done
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(ev_done)
                for k in ("gx", "gw", "gb"):
                    d[k].copy_(d["d" + k], non_blocking=True)
                ev_out = torch.cuda.Event()
                ev_out.record(d2h_s)
            d["out_free"] = ev_out
        comp.wait_stream(d2h_s)
        comp.wait_stream(h2d_s)

    step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.e2e_steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    flops_step = sum(layer_flops(l) for l in glayers)  # global batch (strong scaling)
    return {"value": flops_step / (ms / args.e2e_steps * 1e-3) / 1e9, "unit": "GFLOP/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
            "path": "paper_1606_04884_b200.conv_* (C ABI) on pinned host tensors, H2D inputs + "
                    "D2H outputs/gradients inside the timed region; per-layer copy streams: "
                    "x/w/b then gy H2D, y D2H right after the forward (while gy arrives), "
                    "gradients D2H after the backward; both PCIe directions overlap compute"}


if __name__ == "__main__":
    main()
