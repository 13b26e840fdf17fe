"""Every kernel must depend only on shared memory it wrote.  Before each
call, a helper kernel fills all shared memory with a bit pattern; the same
call after a NaN fill (0xFFFFFFFF) and after a zero fill must give
bit-identical, finite outputs.  (A kernel whose MMAs read operand rows or
columns outside what it staged multiplies stale shared memory by zero
weights: invisible with finite leftovers, NaN with NaN-pattern leftovers
from a previous kernel — the fused kernel had exactly this with merged
super-blocks on non-integer factors, K2.)  Geometries cover the
fused separable kernel (merged and unmerged, bf16 / f32 out), the axis
passes, the f32 FMA-pipe kernel and the DCT-16 strips."""

import ctypes
import os
import subprocess
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def poison():
    d = tempfile.mkdtemp()
    so = os.path.join(d, "libsmem_poison.so")
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-O2", "-shared", "-Xcompiler", "-fPIC", "-o", so,
                    os.path.join(HERE, "helpers", "smem_poison.cu")], check=True)
    lib = ctypes.CDLL(so)
    lib.smem_poison.argtypes = [ctypes.c_uint, ctypes.c_void_p]
    return lib


def _twice(poison, fn):
    import torch
    outs = []
    for pattern in (0xFFFFFFFF, 0x0):
        torch.cuda.synchronize()
        assert poison.smem_poison(pattern, torch.cuda.current_stream().cuda_stream) == 0
        y = fn()
        torch.cuda.synchronize()
        outs.append(y.clone())
    a, b = outs
    assert torch.isfinite(a.float()).all(), "non-finite output after a NaN shared-memory fill"
    ia = a.view(torch.int16) if a.dtype == torch.bfloat16 else a.view(torch.int32)
    ib = b.view(torch.int16) if b.dtype == torch.bfloat16 else b.view(torch.int32)
    assert torch.equal(ia, ib), "output depends on stale shared memory"


def _x(planes, H, W, seed, dtype=None):
    import torch
    rng = np.random.default_rng(seed)
    t = torch.from_numpy(rng.random((planes, H, W), dtype=np.float32))
    return (t if dtype == "f32" else t.bfloat16()).cuda()


@pytest.mark.parametrize("planes,H,W,oh,ow", [
    (3, 979, 909, 697, 257),      # merged rows: a super-block window past the unmerged span
    (2, 888, 1179, 766, 615),
    (3, 2160, 3840, 1080, 1920),  # c2
    (2, 1000, 1400, 333, 700),
    (2, 2048, 2048, 921, 921),    # axis passes
    (1, 2048, 2048, 143, 143),
    (2, 1114, 97, 961, 4),
    (3, 270, 480, 540, 960),      # upsample
])
@pytest.mark.parametrize("f32out", [False, True])
def test_resample_ignores_stale_shared_memory(poison, planes, H, W, oh, ow, f32out):
    import torch
    from paper_2512_02371_b200 import pipelines
    x = _x(planes, H, W, H + W)
    dt = torch.float32 if f32out else torch.bfloat16
    _twice(poison, lambda: pipelines.resample(x, oh, ow, out_dtype=dt))


@pytest.mark.parametrize("taps", [9, 21, 31, 61, 151])
def test_gaussian_ignores_stale_shared_memory(poison, taps):
    from paper_2512_02371_b200 import pipelines
    x = _x(2, 1111, 1333, taps)
    _twice(poison, lambda: pipelines.gaussian_blur(x, taps))


@pytest.mark.parametrize("shape,oh,ow", [((3, 1080, 1920), 540, 960), ((2, 333, 517), 167, 259)])
def test_f32_kernel_ignores_stale_shared_memory(poison, shape, oh, ow):
    import torch
    from paper_2512_02371_b200 import pipelines
    x = _x(*shape, 5, dtype="f32")
    _twice(poison, lambda: pipelines.resample(x, oh, ow, out_dtype=torch.float32))


@pytest.mark.parametrize("shape,mode", [((3, 2160, 3840), "hard"), ((2, 232, 360), "soft"),
                                        ((1, 16, 24), "hard")])
def test_dct16_ignores_stale_shared_memory(poison, shape, mode):
    import torch
    from paper_2512_02371_b200 import pipelines
    x = _x(*shape, 6)
    _twice(poison, lambda: pipelines.denoise_dct16(x, 0.15, mode, out_dtype=torch.float32))
