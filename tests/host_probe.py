"""Host-overhead probe (GPU box, not collected by pytest): CPU time per eager C-ABI conv
call (fwd + combined bwd of every convnet layer), i.e. the launch-side cost the plan cache
removes. Run twice, with and without PT_B200_NO_TMAP_CACHE=1. Prints one JSON line."""
import json
import os
import sys
import time

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
import torch  # noqa: E402

import paper_1606_04884_b200 as pt  # noqa: E402
from bench import WORKLOADS  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "convnet"
bufs = []
for name, *gg in WORKLOADS[wl]:
    g = pt.ConvGeometry(*gg)
    t = lambda s: torch.empty(s, device="cuda")  # noqa: E731
    bufs.append((g, t(g.input_shape()), t(g.weight_shape()), t((g.outChannels,)), t(g.output_shape()),
                 t(g.output_shape()), t(g.input_shape()), t(g.weight_shape()), t((g.outChannels,))))


def step():
    for g, x, w, b, y, gy, gx, gw, gb in bufs:
        pt.conv_forward(g, x, w, b, y)
        pt.conv_backward(g, x, gy, w, gx, gw, gb)


for _ in range(3):
    step()
torch.cuda.synchronize()
reps = 20
host = 0.0
for _ in range(reps):
    t0 = time.perf_counter()
    step()
    host += time.perf_counter() - t0
    torch.cuda.synchronize()
h, e = pt.plan_cache_stats()
print(json.dumps({"workload": wl, "tmap_cache": os.environ.get("PT_B200_NO_TMAP_CACHE") is None,
                  "host_ms_per_step": 1e3 * host / reps, "calls_per_step": 2 * len(bufs),
                  "cache_hits": h, "encodes": e}))
