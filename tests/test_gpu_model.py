"""GPU: the model-stack layer — ReLU / max-pool kernels vs the oracle,
the chained AlexNet / VGG-A stacks layer by layer vs the oracle fed the device's own
layer inputs, bench_model's CSV rows / checksums / per-type summary (SPEC acceptance 9:
conv time dominates), checksums equal across conv implementations, and bench_apply's
bandwidth sweep (bandwidth at 1e7 floats >= at 1e3)."""
import numpy as np
import pytest

import pyoracle as po
from helpers import check_exact, check_tf32, tf32_bounds

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _lib():
    from paper_1606_04884_b200 import _lib as L
    return L


def _d(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _s():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("n", [1, 7, 1024, 100003])
def test_relu_exact(n):
    L = _lib()
    x = po.uniform((n,), n, -1, 1)
    gy = po.uniform((n,), n + 1, -1, 1)
    dx, dy, dgy, dgx = _d(x), torch.empty(n, device="cuda"), _d(gy), torch.empty(n, device="cuda")
    L.check(L.lib().pt_b200_relu_fwd(dx.data_ptr(), dy.data_ptr(), n, _s()))
    L.check(L.lib().pt_b200_relu_bwd(dy.data_ptr(), dgy.data_ptr(), dgx.data_ptr(), n, _s()))
    check_exact(dy.cpu().numpy(), po.relu_fwd(x), "relu fwd")
    check_exact(dgx.cpu().numpy(), po.relu_bwd(po.relu_fwd(x), gy), "relu bwd")


POOLS = [((2, 3, 55, 55), (3, 3, 2, 2, 0, 0)), ((2, 4, 224, 224), (2, 2, 2, 2, 0, 0)),
         ((1, 5, 13, 13), (3, 3, 2, 2, 1, 1)), ((2, 2, 9, 11), (3, 2, 1, 2, 1, 0)),
         ((1, 1, 5, 5), (5, 5, 1, 1, 0, 0))]


@pytest.mark.parametrize("shape,p", POOLS)
def test_maxpool_exact(shape, p):
    L = _lib()
    kH, kW, sH, sW, pH, pW = p
    x = po.uniform(shape, sum(shape), -1, 1)
    y, arg = po.maxpool_fwd(x, kH, kW, sH, sW, pH, pW)
    gy = np.random.default_rng(3).integers(-8, 9, y.shape).astype(np.float32)  # exact sums
    dy = torch.empty(y.shape, device="cuda")
    darg = torch.empty(y.shape, dtype=torch.int32, device="cuda")
    dgx = torch.empty(shape, device="cuda")
    L.check(L.lib().pt_b200_maxpool_fwd(_d(x).data_ptr(), dy.data_ptr(), darg.data_ptr(), *shape,
                                        kH, kW, sH, sW, pH, pW, _s()))
    dgy = _d(gy)
    L.check(L.lib().pt_b200_maxpool_bwd(dgy.data_ptr(), darg.data_ptr(), dgx.data_ptr(), *shape,
                                        kH, kW, sH, sW, pH, pW, _s()))
    check_exact(dy.cpu().numpy(), y, "maxpool fwd")
    np.testing.assert_array_equal(darg.cpu().numpy(), arg)
    check_exact(dgx.cpu().numpy(), po.maxpool_bwd(gy, arg, shape), "maxpool bwd")


@pytest.mark.parametrize("name,batch", [("alexnet", 2), ("vgg-a", 1)])
def test_chained_model_layerwise_vs_oracle(name, batch):
    """Forward + backward of the whole chained stack on the device; every layer's output /
    gradients checked against the oracle applied to that layer's device inputs."""
    from paper_1606_04884_b200 import model as M
    layers = M.chain(M.model_spec_load(name), batch)
    m = M.Model(layers)
    m.forward()
    m.backward()
    torch.cuda.synchronize()
    h = lambda t: t.cpu().numpy()  # noqa: E731
    for i, l in enumerate(layers):
        x, y, gy, s = h(m.input_of(i)), h(m.st[i]["y"]), h(m.grad_of(i)), m.st[i]
        tag = f"{name} layer {i} {l.kind}"
        if l.kind == "relu":
            check_exact(y, po.relu_fwd(x), tag)
            check_exact(h(s["gx"]), po.relu_bwd(y, gy), tag + " bwd")
        elif l.kind == "poolmax":
            kH, kW, sH, sW = l.params
            ry, ra = po.maxpool_fwd(x, kH, kW, sH, sW)
            check_exact(y, ry, tag)
            np.testing.assert_array_equal(h(s["arg"]), ra)
            rg = po.maxpool_bwd(gy.astype(np.float64), ra, x.shape)
            np.testing.assert_allclose(h(s["gx"]), rg, rtol=1e-6, atol=1e-7 * np.abs(gy).max())
        else:
            g = po.geom(*l.geom.input_shape(), l.geom.outChannels, l.geom.kernelH, l.geom.kernelW,
                        l.geom.padH, l.geom.padW, l.geom.strideH, l.geom.strideW)
            w, b = h(s["w"]), h(s["b"])
            tol = tf32_bounds(g, x, w, b, gy)
            check_tf32(y, po.conv_forward(g, x, w, b), tag, tol["fwd"])
            rgw, rgb = po.conv_backward_weight(g, x, gy)
            check_tf32(h(s["gw"]), rgw, tag + " gradWeight", tol["wgrad"])
            check_tf32(h(s["gb"]), rgb, tag + " gradBias", tol["gradBias"])
            if i > 0:
                check_tf32(h(s["gx"]), po.conv_backward_input(g, gy, w), tag + " gradInput",
                           tol["dgrad"])


def test_bench_model_rows_summary_and_checksums():
    from paper_1606_04884_b200 import model as M
    spec = M.model_spec_load("alexnet")
    rows, summary = M.bench_model(spec, batch=16, backward=True, reps=3)
    assert [r["index"] for r in rows] == list(range(13))
    assert [r["type"] for r in rows][:3] == ["conv", "relu", "poolmax"]
    assert all(r["mean_time_s"] > 0 for r in rows)
    assert abs(sum(s["fraction"] for s in summary) - 1) < 1e-9
    # the FP32-FFMA implementation gives the same checksums within 1e-3
    rows32, _ = M.bench_model(spec, batch=16, backward=False, impl="implicitgemm-fp32-sm100a", reps=3)
    for a, b in zip(rows, rows32):
        assert abs(a["checksum"] - b["checksum"]) <= 1e-3 * max(1.0, abs(b["checksum"])), (a, b)
    csv = M.to_csv(rows, M.LAYER_COLUMNS).splitlines()
    assert csv[0] == "index,type,geometry,mean_time_s,checksum" and len(csv) == 14


def test_bench_model_vgga_conv_dominates():
    """SPEC acceptance 9 (Fig. 5 qualitative): conv >= 50% of the VGG-A layer time at scale 16."""
    from paper_1606_04884_b200 import model as M
    _, summary = M.bench_model(M.model_spec_load("vgg-a"), scale=16, batch=16, reps=3)
    conv = [s for s in summary if s["type"] == "conv"][0]
    assert conv["fraction"] >= 0.5, summary


def test_bench_apply_sweep():
    """SPEC acceptance 9: bandwidth at 1e7 floats >= bandwidth at 1e3 (launch overhead)."""
    from paper_1606_04884_b200 import model as M
    rows = M.bench_apply([1000, 10000, 100000, 1000000, 10000000], reps=5)
    assert len(rows) == 5 and all(r["gb_per_s"] > 0 for r in rows)
    assert rows[-1]["gb_per_s"] >= rows[0]["gb_per_s"]


def test_cli_writes_csv(tmp_path):
    from paper_1606_04884_b200.bench_cli import main
    out, summ = tmp_path / "layers.csv", tmp_path / "summary.csv"
    assert main(["model", "--name", "alexnet", "--batch", "4", "--reps", "3", "--backward",
                 "--out", str(out), "--summary", str(summ)]) == 0
    assert out.read_text().splitlines()[0] == "index,type,geometry,mean_time_s,checksum"
    assert summ.read_text().splitlines()[0] == "type,layers,total_time_s,fraction"
    bw = tmp_path / "bw.csv"
    assert main(["apply", "--sizes", "1e3,1e5", "--out", str(bw)]) == 0
    assert bw.read_text().splitlines()[0] == "size,reps,mean_time_s,gb_per_s"
