"""CPU: the model-stack layer's host logic — bundled specs and their
shape chains, spec-file parsing and chain errors, the scale divisor, CSV schemas, and the
CLI's exit codes for validation errors (no GPU work is reached)."""
import pytest

from paper_1606_04884_b200 import ValidationError
from paper_1606_04884_b200 import model as M
from paper_1606_04884_b200.bench_cli import main as cli


def test_bundled_alexnet_chain():
    layers = M.chain(M.model_spec_load("alexnet"), 128)
    convs = [l for l in layers if l.kind == "conv"]
    assert len(layers) == 13 and len(convs) == 5
    g = convs[0].geom
    assert (g.kernelH, g.strideH) == (11, 4)            # 11x11 stride-4 first conv
    # the bench's AlexNet conv shapes (bench.WORKLOADS["alexnet"]) are this chain's convs
    from bench import WORKLOADS
    for c, w in zip(convs, WORKLOADS["alexnet"]):
        assert c.geom.input_shape() == (w[1], w[2], w[3], w[4]) and c.geom.outChannels == w[5]
    assert layers[-1].out_shape == (128, 256, 6, 6)


def test_bundled_vgga_chain():
    layers = M.chain(M.model_spec_load("vgg-a"), 64)
    convs = [l for l in layers if l.kind == "conv"]
    assert len(convs) == 8 and layers[0].in_shape == (64, 3, 224, 224)
    from bench import WORKLOADS
    for c, w in zip(convs, WORKLOADS["vgga"]):
        assert c.geom.input_shape() == (w[1], w[2], w[3], w[4]) and c.geom.outChannels == w[5]
    assert layers[-1].out_shape == (64, 512, 7, 7)


def test_scale_divisor():
    layers = M.chain(M.model_spec_load("vgg-a"), 2, 16)
    assert layers[0].geom.inChannels == 3 and layers[0].geom.outChannels == 4
    with pytest.raises(ValidationError, match="scale 7 does not divide"):
        M.chain(M.model_spec_load("vgg-a"), 1, 7)


def test_spec_file_and_chain_break(tmp_path):
    p = tmp_path / "m.txt"
    p.write_text("conv 3 32 32 16 3 3 1 1 1 1  # first\nrelu\npoolmax 2 2 2 2\n"
                 "conv 16 16 16 8 3 3 1 1 1 1\n")
    layers = M.chain(M.model_spec_load(str(p)), 4)
    assert [l.kind for l in layers] == ["conv", "relu", "poolmax", "conv"]
    assert layers[-1].out_shape == (4, 8, 16, 16)
    p.write_text("conv 3 32 32 16 3 3 1 1 1 1\npoolmax 2 2 2 2\nconv 16 32 32 8 3 3 1 1 1 1\n")
    with pytest.raises(ValidationError, match="chain break at layer 2"):
        M.model_spec_load(str(p))
    p.write_text("conv 3 32 32 16 3 3\n")
    with pytest.raises(ValidationError, match="takes 10 integers"):
        M.model_spec_load(str(p))
    with pytest.raises(ValidationError, match="unknown model"):
        M.model_spec_load("googlenet")


def test_csv_schemas():
    rows = [{"index": 0, "type": "conv", "geometry": "N1 C3", "mean_time_s": 1e-3, "checksum": 2.5}]
    assert M.to_csv(rows, M.LAYER_COLUMNS).splitlines()[0] == "index,type,geometry,mean_time_s,checksum"
    bw = [{"size": 1000, "reps": 5, "mean_time_s": None, "gb_per_s": None, "skipped": True}]
    assert M.to_csv(bw, M.BANDWIDTH_COLUMNS).splitlines() == ["size,reps,mean_time_s,gb_per_s",
                                                              "1000,5,skipped,skipped"]


def test_cli_validation_exit_codes(capsys):
    assert cli(["model", "--name", "vgg-a", "--scale", "7"]) == 2
    assert cli(["model", "--name", "nope"]) == 2
    assert cli(["model", "--name", "alexnet", "--reps", "1"]) == 2
    assert cli(["apply", "--sizes", "1e4,1e3"]) == 2
