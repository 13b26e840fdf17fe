"""Is the fused kernel's per-frame cost a function of the allocation the
frames live in?  16-frame launches over (a) separate 16-frame tensors,
(b) 16-frame slices of one 48-frame tensor, (c) one 48-frame launch."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_02371_b200 import pipelines, axis, _lib

ra, ca = axis.lanczos3(2160, 1080, 0), axis.lanczos3(3840, 1920, 0)
lib = _lib.load()

def launch(x, y):
    P = x.shape[0]
    _lib.check(lib.ts_separable_run(ra.handle, ca.handle, P, x.data_ptr(), 3840, 3840 * 2160,
                                    _lib.TS_BF16, y.data_ptr(), 1920, 1920 * 1080, _lib.TS_BF16,
                                    torch.cuda.current_stream().cuda_stream))

def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

sep_in = [torch.rand((48, 2160, 3840), device="cuda").bfloat16() for _ in range(3)]
sep_out = [torch.empty((48, 1080, 1920), device="cuda", dtype=torch.bfloat16) for _ in range(3)]
big_in = torch.cat(sep_in, 0)
big_out = torch.empty((144, 1080, 1920), device="cuda", dtype=torch.bfloat16)
r = {
    "separate 16-frame tensors, 3 launches": timeit(lambda: [launch(a, b) for a, b in zip(sep_in, sep_out)]),
    "slices of one 48-frame tensor, 3 launches": timeit(lambda: [launch(big_in[i:i + 48], big_out[i:i + 48]) for i in (0, 48, 96)]),
    "one 48-frame launch": timeit(lambda: launch(big_in, big_out)),
    "one 16-frame launch on a slice, x3": timeit(lambda: [launch(big_in[:48], big_out[:48]) for _ in range(3)]),
}
for k, v in r.items():
    print(json.dumps({"case": k, "ms_per_48_frames": round(v, 4)}))
