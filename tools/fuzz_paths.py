"""Random sweep of the host-side paths around the kernels: run_from_host
(random chunk sizes and stream counts; bitwise vs the device call),
partition.run_sharded (random frame shards over 'devices' that are all
cuda:0; bitwise) and partition.resample_bands (random band counts; within 1e-2 of
the full-image call: a band can get a different super-block plan than the
whole image — different f32 summation grouping — which may flip the bf16
rounding of an intermediate V value, i.e. up to ~1 bf16 ulp of V).

    python tools/fuzz_paths.py [N] [SEED]"""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import time
import numpy as np
import torch
from paper_2512_02371_b200 import partition, pipelines

N = int(_sys.argv[1]) if len(_sys.argv) > 1 else 60
rng = np.random.default_rng(int(_sys.argv[2]) if len(_sys.argv) > 2 else 1)
fails, t0 = [], time.time()


def bits(y):
    return y.view(torch.int16) if y.dtype == torch.bfloat16 else y.view(torch.int32)


for i in range(N):
    kind = str(rng.choice(["host", "sharded", "bands"]))
    frames = int(rng.integers(1, 9))
    H, W = int(rng.integers(16, 1300)), int(rng.integers(16, 1300))
    fh, fw = np.exp(rng.uniform(np.log(0.5), np.log(12.0), 2))
    oh, ow = max(1, int(round(H / fh))), max(1, int(round(W / fw)))
    which = str(rng.choice(["resample", "dct", "gauss", "f32"]))
    if which == "dct":
        H, W = 8 * max(2, H // 8), 8 * max(2, W // 8)
        fn = lambda t: pipelines.denoise_dct16(t, 0.1)
    elif which == "gauss":
        taps = int(2 * rng.integers(1, 12) + 1)
        fn = lambda t, taps=taps: pipelines.gaussian_blur(t, taps)
    else:
        fn = lambda t, oh=oh, ow=ow: pipelines.resample(t, oh, ow)
    dt = torch.float32 if which == "f32" else torch.bfloat16
    x = torch.rand((3 * frames, H, W), dtype=torch.float32).to(dt)
    desc = f"{kind} {which} {3 * frames}x{H}x{W}->{oh}x{ow}"
    try:
        want = fn(x.cuda())
        torch.cuda.synchronize()
        if kind in ("host", "sharded"):
            host_in = x.pin_memory()
            host_out = torch.full(want.shape, 7.0, dtype=want.dtype).pin_memory()
            if kind == "host":
                chunk, lanes = int(rng.integers(1, 7)), int(rng.integers(1, 5))
                desc += f" chunk {chunk} lanes {lanes}"
                pipelines.run_from_host(fn, host_in, host_out, chunk_planes=chunk, lanes=lanes)
            else:
                shards = int(rng.integers(1, 5))
                desc += f" shards {shards}"
                partition.run_sharded(fn, host_in, host_out, [0] * shards,
                                      chunk_planes=int(rng.integers(1, 4)) * 3)
            torch.cuda.synchronize()
            if not torch.equal(bits(host_out), bits(want.cpu())):
                fails.append(desc)
        else:
            if which != "resample":
                continue
            bands = int(rng.integers(2, 6))
            desc += f" bands {bands}"
            full = pipelines.resample(x.cuda(), oh, ow, out_dtype=torch.float32)
            got = partition.resample_bands(x.cuda(), oh, ow, [0] * bands, out_dtype=torch.float32)
            torch.cuda.synchronize()
            if got.shape != full.shape or (got - full).abs().max().item() > 1e-2:
                fails.append(desc + f" err {(got - full).abs().max().item() if got.shape == full.shape else 'shape'}")
    except Exception as ex:  # noqa: BLE001
        fails.append(f"{desc}: {type(ex).__name__}: {str(ex).splitlines()[0]}")
        if "CUDA error" in str(ex):
            break
for f in fails:
    print("FAIL", f)
print(f"{N} cases, {len(fails)} failures, {time.time() - t0:.0f} s")
