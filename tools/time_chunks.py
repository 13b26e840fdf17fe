"""Two-pass resample over plane chunks through one reused intermediate
(so the intermediate stays in L2 and its dirty lines are overwritten there
instead of written back): GPU time per 48-plane call for chunk sizes, vs one
pair of launches over all planes.  Launches are captured in a CUDA graph so
host overhead does not enter the timing."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import json, torch
from paper_2512_02371_b200 import _lib, axis as _axis, pipelines

lib = _lib.load()
P = 48
cases = [(2048, 2048, 921, 921), (2048, 2048, 450, 450), (2160, 3840, 540, 960), (2048, 2048, 245, 245)]
for H, W, oh, ow in cases:
    x = torch.rand((P, H, W), device="cuda").bfloat16()
    ra, ca = _axis.lanczos3(H, oh, 0), _axis.lanczos3(W, ow, 0)
    owp = -(-ow // 8) * 8
    out = torch.empty((P, oh, owp), dtype=torch.bfloat16, device="cuda")
    res = {"case": f"{H}x{W}->{oh}x{ow}"}
    ref = None
    for n in (48, 24, 16, 12, 8, 6, 4, 3, 2):
        mid = torch.empty((n, oh, W), dtype=torch.bfloat16, device="cuda")
        s = torch.cuda.Stream()
        def run():
            st = s.cuda_stream
            for p0 in range(0, P, n):
                c = min(n, P - p0)
                _lib.check(lib.ts_axis_pass(ra.handle, 0, c, H, W, x[p0].data_ptr(), W, W * H,
                                            mid.data_ptr(), W, W * oh, _lib.TS_BF16, st))
                _lib.check(lib.ts_axis_pass(ca.handle, 1, c, oh, W, mid.data_ptr(), W, W * oh,
                                            out[p0].data_ptr(), owp, owp * oh, _lib.TS_BF16, st))
        with torch.cuda.stream(s):
            run(); run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            run()
        for _ in range(3): g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): g.replay()
        b.record(); torch.cuda.synchronize()
        res[n] = round(a.elapsed_time(b) / 20, 4)
        if ref is None:
            ref = out.clone()
        else:
            assert torch.equal(out.view(torch.int16), ref.view(torch.int16))
        del mid
    alg = P * (H * W + oh * ow) * 2
    res["best_frac"] = round(alg / min(v for k, v in res.items() if isinstance(k, int)) / 1e6 / 6455.6, 3)
    print(json.dumps(res), flush=True)
