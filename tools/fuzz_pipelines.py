"""Exploratory random-geometry sweep of every pipeline against the CPU oracle,
with all shared memory NaN-filled before each call (tests/helpers/
smem_poison.cu).  Prints one line per failure and a summary.

    python tools/fuzz_pipelines.py [N] [SEED]

The committed regression set lives in tests/test_gpu_fuzz.py and
tests/test_gpu_smem_poison.py; this tool is the wider net that found the
merged-window bug (K2)."""
import os as _os, sys as _sys
ROOT = _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))
_sys.path.insert(0, ROOT)
import ctypes, subprocess, tempfile, time
import numpy as np
import torch
from oracle import pipelines_ref as ref
from paper_2512_02371_b200 import filters, pipelines

N = int(_sys.argv[1]) if len(_sys.argv) > 1 else 200
SEED = int(_sys.argv[2]) if len(_sys.argv) > 2 else 1
TOL = 1e-2

d = tempfile.mkdtemp()
so = _os.path.join(d, "p.so")
subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2",
                "-shared", "-Xcompiler", "-fPIC", "-o", so,
                _os.path.join(ROOT, "tests", "helpers", "smem_poison.cu")], check=True)
poison = ctypes.CDLL(so)
poison.smem_poison.argtypes = [ctypes.c_uint, ctypes.c_void_p]


def poisoned(fn):
    torch.cuda.synchronize()
    poison.smem_poison(0xFFFFFFFF, torch.cuda.current_stream().cuda_stream)
    y = fn()
    torch.cuda.synchronize()
    return y.float().cpu().numpy()


def epi(y, ep):
    if ep is None:
        return y
    s, b, lo, hi = ep
    return np.clip(y * s + b, lo, hi)


rng = np.random.default_rng(SEED)
fails, counts = [], {}
t0 = time.time()
for i in range(N):
    op = rng.choice(["resample", "resample", "filter", "resample_filter", "f32", "dct"])
    planes = int(rng.integers(1, 4))
    H, W = int(rng.integers(4, 1400)), int(rng.integers(4, 1400))
    f32out = bool(rng.integers(0, 2))
    odt = torch.float32 if f32out else torch.bfloat16
    ep = None
    if rng.random() < 0.25:
        ep = (float(rng.uniform(0.5, 2)), float(rng.uniform(-0.2, 0.2)), 0.1, 0.9)
    kw = {} if ep is None else dict(scale=ep[0], bias=ep[1], clamp=(ep[2], ep[3]))
    tol = TOL if f32out else TOL + 4e-3 * max(1.0, abs(ep[0]) if ep else 1.0)
    x = rng.random((planes, H, W), dtype=np.float32)
    xb = torch.from_numpy(x).bfloat16()
    xr = xb.float().numpy()
    desc = ""
    try:
        if op in ("resample", "f32"):
            fh, fw = np.exp(rng.uniform(np.log(0.45), np.log(30.0), 2))
            oh, ow = max(1, int(round(H / fh))), max(1, int(round(W / fw)))
            if op == "f32" and rng.random() < 0.6:  # the uniform 2x case the f32 kernel takes
                H, W = 2 * max(2, H // 2), 2 * max(2, W // 2)
                x = rng.random((planes, H, W), dtype=np.float32)
                oh, ow = H // 2, W // 2
            desc = f"{op} {planes}x{H}x{W}->{oh}x{ow} out={'f32' if f32out else 'bf16'} ep={ep}"
            if op == "f32":
                xin = torch.from_numpy(x).cuda()
                want = epi(ref.resample(x, oh, ow), ep)
            else:
                xin = xb.cuda()
                want = epi(ref.resample(xr, oh, ow), ep)
            got = poisoned(lambda: pipelines.resample(xin, oh, ow, out_dtype=odt, **kw))
        elif op == "filter":
            tv, th = int(rng.integers(1, 90)), int(rng.integers(1, 90))
            kv = filters.gaussian_taps(tv) if rng.random() < 0.5 else filters.box_taps(tv)
            kh = filters.gaussian_taps(th) if rng.random() < 0.5 else filters.box_taps(th)
            desc = f"filter {planes}x{H}x{W} taps {tv}/{th} out={'f32' if f32out else 'bf16'} ep={ep}"
            want = epi(ref.separable(xr, ref.centred_axis(H, np.asarray(kv, np.float32)),
                                     ref.centred_axis(W, np.asarray(kh, np.float32))), ep)
            got = poisoned(lambda: pipelines.filter_separable(xb.cuda(), kv, kh, out_dtype=odt, **kw))
        elif op == "resample_filter":
            fh, fw = np.exp(rng.uniform(np.log(0.6), np.log(6.0), 2))
            oh, ow = max(8, int(round(H / fh))), max(8, int(round(W / fw)))
            taps = int(2 * rng.integers(1, 8) + 1)
            desc = f"resample_filter {planes}x{H}x{W}->{oh}x{ow} taps {taps}"
            want = ref.gaussian_blur(ref.resample(xr, oh, ow), taps)
            got = poisoned(lambda: pipelines.resample_filter(xb.cuda(), oh, ow, taps,
                                                             out_dtype=torch.float32))
            tol = 2e-2  # the fused composition rounds once, the oracle twice
        else:
            H, W = 8 * max(2, H // 8), 8 * max(2, W // 8)
            x = rng.random((planes, H, W), dtype=np.float32)
            xb = torch.from_numpy(x).bfloat16()
            xr = xb.float().numpy()
            thr = float(rng.uniform(0.01, 0.4))
            mode = "hard" if rng.random() < 0.5 else "soft"
            desc = f"dct {mode} {planes}x{H}x{W} thr {thr:.3f} ep={ep}"
            want = epi(ref.dct_denoise(xr, thr, mode), ep)
            got = poisoned(lambda: pipelines.denoise_dct16(xb.cuda(), thr, mode,
                                                           out_dtype=odt, **kw))
            if mode == "hard":  # pixels of tiles with a coefficient within EPS_FWD of thr
                excused = ref.dct_flip_mask(xr, thr, 1e-5)   # may flip (tests/test_gpu_dct.py)
                want = np.where(excused, got, want)
        counts[op] = counts.get(op, 0) + 1
        if got.shape != want.shape:
            fails.append(f"{desc}: shape {got.shape} vs {want.shape}")
        elif not np.isfinite(got).all():
            fails.append(f"{desc}: {int((~np.isfinite(got)).sum())} non-finite")
        else:
            e = float(np.abs(got - want).max())
            if e > tol:
                fails.append(f"{desc}: max err {e:.4g} > {tol}")
    except Exception as ex:  # noqa: BLE001 — report and continue
        fails.append(f"{desc}: {type(ex).__name__}: {str(ex).splitlines()[0]}")
        if "CUDA error" in str(ex):  # the context is gone: stop at the first one
            print(f"case {i}: {fails[-1]}", flush=True)
            break
for f in fails:
    print("FAIL", f)
print(f"{N} cases {counts}, {len(fails)} failures, {time.time() - t0:.0f} s")
