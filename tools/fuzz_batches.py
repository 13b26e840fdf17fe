"""Batch-consistency sweep: random geometries with many planes (8-40, so
CTAs walk many tiles / units / strips and every pipeline's end-of-work and
phase logic is exercised), shared memory NaN-filled before each call; the
batched result must equal, bit for bit, the same pipeline run on a few
planes on their own.  No oracle needed, so large batches are cheap.

    python tools/fuzz_batches.py [N] [SEED]      (TSB_DYNAMIC_TILES=1 etc. apply)"""
import os as _os, sys as _sys
ROOT = _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))
_sys.path.insert(0, ROOT)
import ctypes, subprocess, tempfile, time
import numpy as np
import torch
from paper_2512_02371_b200 import filters, pipelines

N = int(_sys.argv[1]) if len(_sys.argv) > 1 else 100
SEED = int(_sys.argv[2]) if len(_sys.argv) > 2 else 1
d = tempfile.mkdtemp()
so = _os.path.join(d, "p.so")
subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2",
                "-shared", "-Xcompiler", "-fPIC", "-o", so,
                _os.path.join(ROOT, "tests", "helpers", "smem_poison.cu")], check=True)
poison = ctypes.CDLL(so)
poison.smem_poison.argtypes = [ctypes.c_uint, ctypes.c_void_p]


def run(fn, x):
    torch.cuda.synchronize()
    poison.smem_poison(0xFFFFFFFF, torch.cuda.current_stream().cuda_stream)
    y = fn(x)
    torch.cuda.synchronize()
    return y


def bits(y):
    return y.view(torch.int16) if y.dtype == torch.bfloat16 else y.view(torch.int32)


rng = np.random.default_rng(SEED)
fails, counts = [], {}
t0 = time.time()
for i in range(N):
    op = str(rng.choice(["resample", "filter", "resample_filter", "f32", "dct"]))
    planes = int(rng.integers(8, 41))
    H, W = int(rng.integers(8, 1500)), int(rng.integers(8, 1500))
    odt = torch.float32 if rng.integers(0, 2) else torch.bfloat16
    if op in ("resample", "f32"):
        fh, fw = np.exp(rng.uniform(np.log(0.5), np.log(25.0), 2))
        oh, ow = max(1, int(round(H / fh))), max(1, int(round(W / fw)))
        if op == "f32" and rng.random() < 0.7:
            H, W = 2 * max(2, H // 2), 2 * max(2, W // 2)
            oh, ow = H // 2, W // 2
        fn = lambda t, oh=oh, ow=ow, odt=odt: pipelines.resample(t, oh, ow, out_dtype=odt)
        desc = f"{op} {planes}x{H}x{W}->{oh}x{ow} {odt}"
    elif op == "filter":
        tv, th = int(rng.integers(1, 70)), int(rng.integers(1, 70))
        kv, kh = filters.gaussian_taps(tv), filters.box_taps(th)
        fn = lambda t, kv=kv, kh=kh, odt=odt: pipelines.filter_separable(t, kv, kh, out_dtype=odt)
        desc = f"filter {planes}x{H}x{W} taps {tv}/{th} {odt}"
    elif op == "resample_filter":
        fh, fw = np.exp(rng.uniform(np.log(0.6), np.log(5.0), 2))
        oh, ow = max(8, int(round(H / fh))), max(8, int(round(W / fw)))
        taps = int(2 * rng.integers(1, 8) + 1)
        fn = lambda t, oh=oh, ow=ow, taps=taps, odt=odt: pipelines.resample_filter(t, oh, ow, taps, out_dtype=odt)
        desc = f"resample_filter {planes}x{H}x{W}->{oh}x{ow} taps {taps} {odt}"
    else:
        H, W = 8 * max(2, H // 8), 8 * max(2, W // 8)
        mode = "hard" if rng.random() < 0.5 else "soft"
        fn = lambda t, mode=mode, odt=odt: pipelines.denoise_dct16(t, 0.12, mode, out_dtype=odt)
        desc = f"dct {mode} {planes}x{H}x{W} {odt}"
    counts[op] = counts.get(op, 0) + 1
    x = torch.rand((planes, H, W), device="cuda")
    if op != "f32":
        x = x.bfloat16()
    try:
        y = run(fn, x)
        if not torch.isfinite(y.float()).all():
            fails.append(f"{desc}: non-finite")
            continue
        for p in sorted(set(int(v) for v in rng.integers(0, planes, 3))):
            yp = run(fn, x[p:p + 1].contiguous())
            if not torch.equal(bits(yp[0]), bits(y[p])):
                fails.append(f"{desc}: plane {p} differs from its batched result")
                break
    except Exception as ex:  # noqa: BLE001
        fails.append(f"{desc}: {type(ex).__name__}: {str(ex).splitlines()[0]}")
        if "CUDA error" in str(ex):
            print(f"case {i}: {fails[-1]}", flush=True)
            break
for f in fails:
    print("FAIL", f)
print(f"{N} cases {counts}, {len(fails)} failures, {time.time() - t0:.0f} s")
