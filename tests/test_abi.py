"""The C-ABI library: loads, exports what include/tensorsel_b200.h declares,
and the host half of the weight builder behaves (no GPU needed: axes are
built with device=-1, i.e. host only)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from oracle import layout_ref, pipelines_ref
from paper_2512_02371_b200 import _lib, axis, errors, filters, layout

HEADER = os.path.join(ROOT, "include", "tensorsel_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"TS_API\s+[\w\s\*]+?\b(ts_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTED)
    assert lib.ts_abi_version() == _lib.ABI_VERSION == 2


def test_device_count_is_callable():
    n = _lib.load().ts_device_count()
    assert n >= 0


def bf16(x):
    a = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return (((a + 0x7FFF + ((a >> 16) & 1)) >> 16) << 16).astype(np.uint32).view(np.float32)


@pytest.mark.parametrize("n_in,n_out", [(2160, 1080), (3840, 1920), (1080, 540), (100, 50),
                                        (37, 18), (1000, 700)])
def test_lanczos_axis_matches_oracle_band(n_in, n_out):
    first, w = filters.lanczos3_axis(n_in, n_out)
    a = axis.Axis(n_in, n_out, first, w, device=-1)
    got = a.dense()
    ofirst, ow = pipelines_ref.lanczos3_weights(n_in, n_out)
    want = layout_ref.banded_axis(n_in, ofirst, ow)
    # bf16 rounding (half an ulp) plus at most two ulps of DC rebalance
    mag = np.abs(want)
    ulp = np.where(mag > 0, 2.0 ** (np.floor(np.log2(np.maximum(mag, 1e-30))) - 7), 0.0)
    tol = 2.5 * ulp + 1e-9
    assert np.all(np.abs(got - want) <= tol)
    # DC exactness: every output's taps sum to 1 within f32 noise
    np.testing.assert_allclose(got.sum(1), 1.0, atol=3e-5)
    info = a.info
    assert info["n_in"] == n_in and info["n_out"] == n_out
    assert info["window"] % 16 == 0 and info["blocks"] == -(-n_out // 16)


def test_lanczos_2x_geometry():
    first, w = filters.lanczos3_axis(3840, 1920)
    info = axis.Axis(3840, 1920, first, w, device=-1).info
    # 16 outputs at stride 2 + 12 taps, window aligned to 8: 48 inputs, 3 K-steps
    assert info["window"] == 48 and info["taps"] == 12
    assert info["row_span"] == 272 and info["col_blocks"] == 3 and info["col_span"] == 112
    # interior blocks share one tile; two edge variants + the zero tile
    assert info["unique_tiles"] <= 4


@pytest.mark.parametrize("s,p,l", [(1, 1, 5), (2, 1, 12), (3, 1, 8), (1, 2, 4), (1, 4, 3)])
def test_toeplitz_axis_is_matrix_for_transposed(s, p, l):
    k = 32
    spec = layout.ToeplitzSpec(l=l, k=k, s=s, p=p)
    kern = bf16(np.linspace(-1, 1, spec.kernel_length).astype(np.float32) + 0.1)
    rows = layout.matrix_rows(spec)
    a = axis.Axis.from_toeplitz(spec, kern, n_in=rows, n_out=k, device=-1)
    got = a.dense()
    want = layout.matrix_for(kern, spec).T
    assert np.array_equal(got, want)


def test_builder_errors_map_to_reference_exceptions():
    spec = layout.ToeplitzSpec(l=4, k=8, p=2)
    with pytest.raises(errors.PhaseMismatch):
        axis.Axis.from_toeplitz(spec, np.ones(7, np.float32), 16, 8, device=-1)
    first, w = filters.lanczos3_axis(4096, 64)  # 64x: one block needs > 1024 inputs
    with pytest.raises(errors.UnsupportedGeometry):
        axis.Axis(4096, 64, first, w, device=-1)
    first, w = filters.lanczos3_axis(2048, 143)  # 14x: builds (runs as axis passes)
    big = axis.Axis(2048, 143, first, w, device=-1)
    assert big.info["window"] > 256
    with pytest.raises(errors.EvalError):
        axis.Axis(0, 4, np.zeros(4, np.int32), np.zeros((4, 2), np.float32), device=-1)


def test_separable_plan_for_the_headline_config():
    lib = _lib.load()
    f, w = filters.lanczos3_axis(2160, 1080)
    ra = axis.Axis(2160, 1080, f, w, device=-1)
    f, w = filters.lanczos3_axis(3840, 1920)
    ca = axis.Axis(3840, 1920, f, w, device=-1)
    out = (ctypes.c_int * 8)()
    _lib.check(lib.ts_separable_plan(ra.handle, ca.handle, 3, _lib.TS_BF16, out))
    nst, nmid, resident, smem, r1, nb2, tiles, grid = list(out)
    assert (nst, nmid, resident) == (2, 2, 1)
    assert smem <= 232448 and r1 == 272 and nb2 == 3
    assert tiles == 3 * 9 * 40


def test_pipelines_refuse_host_arrays():
    from paper_2512_02371_b200 import pipelines
    with pytest.raises(errors.NoDevice):
        pipelines.resample(np.zeros((4, 4), np.float32), 2, 2)


def test_missing_library_fails_loudly():
    """No CPU fallback: without the native library every product entry point
    raises NativeLibraryMissing (here: the binding pointed at a missing file)."""
    import subprocess
    import sys
    code = ("import numpy as np, torch\n"
            "from paper_2512_02371_b200 import _lib, axis, executor, pipelines\n"
            "try:\n    _lib.load()\nexcept _lib.NativeLibraryMissing:\n    pass\n"
            "else:\n    raise SystemExit('load() succeeded')\n"
            "try:\n    axis.lanczos3(64, 32, 0)\nexcept _lib.NativeLibraryMissing:\n    print('ok')\n")
    env = {**os.environ, "TSB_LIB_PATH": "/nonexistent/libtsb200.so", "PYTHONPATH": ROOT}
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=ROOT)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stdout + r.stderr
