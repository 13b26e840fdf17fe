"""The product's layout module (reference API, vectorised host + device builders)
against the reference fixtures (layout.py:24-135, test_layout.py)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2512_02371_b200 import layout
from paper_2512_02371_b200.errors import LayoutOutOfBounds, PhaseMismatch


@pytest.fixture(scope="module")
def L():
    with open(os.path.join(GOLDEN, "reference_golden.json")) as f:
        return json.load(f)["layout"]


def test_known_matrices(L):
    assert layout.toeplitz_matrix(np.array([5.0, 7.0, 9.0], np.float32), 2).tolist() == L["toeplitz_3tap_k2"]
    assert layout.strided_toeplitz(np.array([1.0, 1.0], np.float32), 2, 2).tolist() == L["strided_2tap_k2_s2"]
    assert layout.polyphase_toeplitz(np.array([2.0, 3.0], np.float32), 4, 2).tolist() == L["polyphase_1tap_k4_p2"]
    assert layout.shuffle_indices_for(layout.ToeplitzSpec(l=3, k=2), 0, 3) == L["shuffle_l3_k2"]
    assert layout.kway_interleave_indices(2, 4, 2) == L["kway_2_4_2"]


def test_random_specs(L):
    for case in L["random"]:
        spec = layout.ToeplitzSpec(l=case["l"], k=case["k"], s=case["s"], p=case["p"])
        kern = np.array(case["kernel"], np.float32)
        m = layout.matrix_for(kern, spec)
        assert m.shape == (layout.matrix_rows(spec), spec.k)
        assert m.tolist() == case["matrix"]
        assert layout.shuffle_indices_for(spec, case["base"], case["base"] + len(kern) + 2) == case["shuffle"]
        for y in range(m.shape[0]):
            for x in range(spec.k):
                t = layout.kernel_taps(spec, y, x)
                assert (m[y, x] == 0.0) if t is None else (m[y, x] == kern[t])


def test_errors():
    with pytest.raises(PhaseMismatch):
        layout.polyphase_toeplitz(np.zeros(5, np.float32), 4, 2)
    with pytest.raises(PhaseMismatch):
        layout.matrix_for(np.zeros(3, np.float32), layout.ToeplitzSpec(l=4, k=2))
    with pytest.raises(LayoutOutOfBounds):
        layout.shuffle_indices_for(layout.ToeplitzSpec(l=4, k=2), 1, 4)
    with pytest.raises(AssertionError):
        layout.ToeplitzSpec(l=2, k=2, s=2, p=2)


def test_spec_properties():
    assert layout.ToeplitzSpec(l=3, k=4, p=2).kernel_length == 6
    assert layout.ToeplitzSpec(l=3, k=4, p=2).mode == "upsample"
    assert layout.ToeplitzSpec(l=3, k=4, s=2).mode == "downsample"
    assert layout.ToeplitzSpec(l=3, k=4).mode == "convolution"


@pytest.mark.gpu
def test_matrix_for_on_device(L):
    import torch
    for case in L["random"]:
        spec = layout.ToeplitzSpec(l=case["l"], k=case["k"], s=case["s"], p=case["p"])
        kern = torch.tensor(case["kernel"], dtype=torch.float32, device="cuda")
        m = layout.matrix_for(kern, spec, device="cuda")
        torch.cuda.synchronize()
        assert m.cpu().tolist() == case["matrix"]


def test_wire_format_roundtrip_matches_reference(tmp_path):
    # directory written by the reference's save_buffers (tests/golden/wire_conv1d_k8)
    from paper_2512_02371_b200 import wire
    from conftest import GOLDEN
    src = os.path.join(GOLDEN, "wire_conv1d_k8")
    bufs = wire.load_buffers(src)
    assert set(bufs) >= {"K", "I", "output", "conv", "bfvec", "ivec"}
    assert bufs["ivec"][2].tolist() == list(range(-5, 6))
    assert bufs["bfvec"][0] == "bf16" and bufs["bfvec"][2].dtype == np.float32
    wire.save_buffers(bufs, tmp_path)
    for e in wire.read_manifest(src):
        a = open(os.path.join(src, e["name"] + ".bin"), "rb").read()
        b = open(os.path.join(tmp_path, e["name"] + ".bin"), "rb").read()
        assert a == b, e["name"]
    assert json.load(open(os.path.join(src, "manifest.json"))) == \
        json.load(open(os.path.join(tmp_path, "manifest.json")))


@pytest.mark.gpu
def test_wire_format_to_device(tmp_path):
    import torch
    from paper_2512_02371_b200 import wire
    from conftest import GOLDEN
    src = os.path.join(GOLDEN, "wire_conv1d_k8")
    host = wire.load_buffers(src)
    dev = wire.load_buffers(src, device="cuda")
    assert dev["bfvec"][2].dtype == torch.bfloat16 and dev["bfvec"][2].is_cuda
    assert torch.equal(dev["bfvec"][2].float().cpu(), torch.from_numpy(host["bfvec"][2]))
    wire.save_buffers(dev, tmp_path)
    for e in wire.read_manifest(src):
        assert open(os.path.join(src, e["name"] + ".bin"), "rb").read() == \
            open(os.path.join(tmp_path, e["name"] + ".bin"), "rb").read()
