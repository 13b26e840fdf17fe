"""Throughput of the drop-in run_program backend against the
reference interpreter on the same program and inputs.

Program: the image-scale generated Lanczos-3 2x stream (tests/test_cli.py:
_lanczos_stream_program) — a For loop over n 256-output windows of one long
row (12 taps, stride 2), i.e. one image row of 256*n output pixels per
instance.  Both arms consume the same seeded inputs (interp.random_inputs).

  reference: tensorsel.interp.run_program per instance (baseline/_ref), 1 core
  gpu      : executor.run_program_batch over all instances (host planning,
             H2D, kernels, D2H included: the public API's wall clock)

    python tools/bench_executor.py [n_windows] [instances]   -> one JSON line
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

import numpy as np  # noqa: E402

from test_cli import _lanczos_stream_program  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
T = int(sys.argv[2]) if len(sys.argv) > 2 else 16
text = _lanczos_stream_program(n)

from tensorsel import interp, ir  # noqa: E402  (the reference, from baseline/_ref)
from paper_2512_02371_b200 import executor, irlite  # noqa: E402

p_ref = ir.parse_program(text)
p_gpu = irlite.parse_program(text)
ins = [interp.random_inputs(p_ref, s) for s in range(T)]
outs = 256 * n

# reference arm: one instance per run_program call, single core
t = time.perf_counter()
k = 0
ref_out = []
while True:
    ref_out.append(interp.run_program(p_ref, ins[k % T])["output"].data)
    k += 1
    if time.perf_counter() - t > 10 or k >= T:
        break
ref_s = (time.perf_counter() - t) / k

# GPU arm: all instances in one run_program_batch (warm once: builds the plan caches)
import torch  # noqa: E402
executor.run_program_batch(p_gpu, ins[:2])
torch.cuda.synchronize()
reps = 5
t = time.perf_counter()
for _ in range(reps):
    got = executor.run_program_batch(p_gpu, ins)
torch.cuda.synchronize()
gpu_s = (time.perf_counter() - t) / reps
same = all(got[i]["output"].data.tobytes() == ref_out[i].tobytes() for i in range(min(k, T)))
print(json.dumps({
    "program": f"lanczos stream, {n} windows x 256 outputs (12 taps, stride 2)",
    "instances": T, "outputs_per_instance": outs,
    "reference_Mpix_s": round(outs / ref_s / 1e6, 4),
    "reference_s_per_instance": round(ref_s, 4),
    "gpu_Mpix_s": round(T * outs / gpu_s / 1e6, 2),
    "gpu_s_per_batch": round(gpu_s, 4),
    "speedup": round((T * outs / gpu_s) / (outs / ref_s), 1),
    "bitwise_equal": bool(same),
}))
