"""The GPU forward chain's coefficient error against the oracle (the `EPS_FWD`
the hard-coring parity test excuses): the diagnostics build writes every
forward coefficient (ts_debug_dct16), compared here with
oracle.pipelines_ref.dct_coefficients on the same bf16 image.

    make -C paper_2512_02371_b200/csrc diag
    python tools/dct_coef_error.py [H W]          -> one JSON line
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("TSB_LIB_PATH", os.path.join(ROOT, "paper_2512_02371_b200", "_native",
                                                   "libtsb200_diag.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import pipelines_ref as R  # noqa: E402
from paper_2512_02371_b200 import _lib, pipelines  # noqa: E402

H, W = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (1080, 1920)
rng = np.random.default_rng(3)
yy, xx = np.mgrid[0:H, 0:W]
clean = 0.5 + 0.4 * np.sin(xx / 17.0) * np.cos(yy / 23.0)
res = {}
for name, img in (("smooth+noise", np.clip(clean + rng.normal(0, 0.05, (1, H, W)), 0, 1)),
                  ("uniform", rng.random((1, H, W)))):
    x = torch.from_numpy(img.astype(np.float32)).bfloat16()
    want = R.dct_coefficients(x.float().numpy())
    buf = torch.full(want.shape, float("nan"), device="cuda")
    lib = _lib.load_diag()
    _lib.check(lib.ts_debug_dct16(buf.data_ptr()))
    pipelines.denoise_dct16(x.cuda(), 0.15, "hard")
    torch.cuda.synchronize()
    _lib.check(lib.ts_debug_dct16(None))
    got = buf.cpu().numpy()
    assert not np.isnan(got).any(), "some coefficients were not written"
    err = np.abs(got - want)
    res[name] = {"max_abs_err": float(err.max()), "p99999_abs_err": float(np.quantile(err, 0.99999)),
                 "mean_abs_err": float(err.mean()), "max_abs_coef": float(np.abs(want).max()),
                 "coefficients": int(err.size)}
print(json.dumps({"image": f"1x{H}x{W} bf16", "forward_error": res}))
