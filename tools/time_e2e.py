"""c2 end to end through pipelines.run_from_host from pinned host memory:
chunk size / stream count sweep (H2D + kernel + D2H per step)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_02371_b200 import pipelines
F = 16
host_in = torch.rand((F * 3, 2160, 3840)).bfloat16().pin_memory()
host_out = torch.empty((F * 3, 1080, 1920), dtype=torch.bfloat16).pin_memory()
fn = pipelines.downsample2x
for chunk, lanes in ((12, 3), (6, 3), (3, 3), (3, 4), (6, 4), (4, 4), (2, 4), (6, 6)):
    for _ in range(2):
        pipelines.run_from_host(fn, host_in, host_out, chunk_planes=chunk, lanes=lanes)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        pipelines.run_from_host(fn, host_in, host_out, chunk_planes=chunk, lanes=lanes)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(json.dumps({"chunk": chunk, "lanes": lanes, "ms": round(ms, 3),
                      "Mpix_s": round(F * 2160 * 3840 / ms / 1e3, 1),
                      "h2d_GBps": round(host_in.numel() * 2 / ms / 1e6, 1)}))
# raw copy ceiling
d = torch.empty_like(host_in, device="cuda")
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5): d.copy_(host_in, non_blocking=True)
torch.cuda.synchronize(); print(json.dumps({"raw_h2d_GBps": round(5 * host_in.numel() * 2 / (time.perf_counter() - t) / 1e9, 1)}))
