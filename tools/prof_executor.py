import cProfile, pstats, sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from test_cli import _lanczos_stream_program
from paper_2512_02371_b200 import executor, irlite
from oracle import interp_ref
import torch
p = irlite.parse_program(_lanczos_stream_program(512))
params = [(q.name, q.kind, q.length) for q in p.params]
ins = [interp_ref.random_fill(params, s) for s in range(16)]
executor.run_program_batch(p, ins); torch.cuda.synchronize()
cProfile.run("for _ in range(5): executor.run_program_batch(p, ins)", "/tmp/pe")
pstats.Stats("/tmp/pe").sort_stats("tottime").print_stats(14)
