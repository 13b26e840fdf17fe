"""Fused separable kernel with and without super-block merging (TSB_NO_MERGE)."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import os, json, torch
from paper_2512_02371_b200 import pipelines
def t(fn, x, n=20):
    for _ in range(3): y = fn(x)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): y = fn(x)
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n, y
cases = [("c2x16", (48, 2160, 3840), pipelines.downsample2x),
         ("c5-like x16", (48, 2160, 3840), lambda z: pipelines.resample_filter(z, 1080, 1920, 9))]
for taps in (9, 15, 21, 31):
    cases.append((f"gauss{taps}", (3, 4320, 7680), (lambda tp: (lambda z: pipelines.gaussian_blur(z, tp)))(taps)))
cases.append(("up2x", (24, 1080, 1920), pipelines.upsample2x))
# launch parameters are cached per process: one process per variant
variant = _sys.argv[1] if len(_sys.argv) > 1 else None
if variant is None:
    import subprocess
    for v in ("merge", "nomerge"):
        env = dict(os.environ)
        if v == "nomerge":
            env["TSB_NO_MERGE"] = "1"
        subprocess.run([_sys.executable, __file__, v], env=env, check=True)
    _sys.exit(0)
for name, shape, fn in cases:
    x = torch.rand(shape, device="cuda").bfloat16()
    ms, y = t(fn, x)
    print(json.dumps({"cfg": name, "variant": variant, "ms": round(ms, 4)}), flush=True)
    del x
