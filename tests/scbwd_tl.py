"""GPU timing probe (not collected): VGG-A conv1 combined backward (the fused small-C
backward, umma_scbwd) timed with CUDA events over three calls."""
import os
import sys
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
import torch  # noqa: E402
import paper_1606_04884_b200 as pt  # noqa: E402
G = pt.ConvGeometry(64, 3, 224, 224, 64, 3, 3, 1, 1, 1, 1)
t = lambda s: torch.randn(s, device="cuda")  # noqa: E731
x, w, gy = t(G.input_shape()), t(G.weight_shape()), t(G.output_shape())
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for r in range(3):
    ev[0].record()
    pt.conv_backward(G, x, gy, w)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"rep {r}: {ev[0].elapsed_time(ev[1]):.3f} ms", flush=True)
