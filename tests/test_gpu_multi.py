"""Multi-GPU product paths on the real kernels.

The round-end box has one B200, so every "device" below is cuda:0: what is
tested is that the sharded paths (frame shards from one process, row bands
of one image, one process per rank) reproduce a single full call when the
same kernels run on each shard.  Reference loops being parallelised: the
tile loop of interp.run_program (interp.py:608-612) and the trial loop of
the CLI difftest (cli.py:167-182).
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _frames(n, H, W, seed):
    import torch
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.rand((n * 3, H, W), generator=g).bfloat16()


def test_run_sharded_frames_bitwise_equal_to_one_call():
    """c5's pipeline (4K -> 1080p Lanczos-3 + 9-tap Gaussian as one fused
    pass) over 5 frames split into frame shards on two 'devices'."""
    import torch
    from paper_2512_02371_b200 import partition, pipelines
    x = _frames(5, 540, 960, 1)
    fn = lambda t: pipelines.resample_filter(t, 270, 480, 9)  # noqa: E731
    want = fn(x.cuda()).cpu()
    host_in = x.pin_memory()
    host_out = torch.empty_like(want).pin_memory()
    partition.run_sharded(fn, host_in, host_out, [0, 0], chunk_planes=6)
    assert torch.equal(host_out.view(torch.int16), want.view(torch.int16))
    # uneven split: 5 frames over 3 shards
    host_out.zero_()
    partition.run_sharded(fn, host_in, host_out, [0, 0, 0], chunk_planes=3)
    assert torch.equal(host_out.view(torch.int16), want.view(torch.int16))


@pytest.mark.parametrize("bands,shape,out", [
    (2, (3, 1080, 1920), (540, 960)),
    (3, (1, 2160, 3840), (1080, 1920)),
    (4, (2, 1000, 1400), (333, 700)),
])
def test_row_bands_match_full_image(bands, shape, out):
    """One image as output row bands (band-local rows axis via band_axis ->
    Axis -> the fused kernel) against the full-image call."""
    import torch
    from paper_2512_02371_b200 import partition, pipelines
    g = torch.Generator(device="cpu").manual_seed(bands)
    x = torch.rand(shape, generator=g).bfloat16().cuda()
    full = pipelines.resample(x, *out, out_dtype=torch.float32)
    got = partition.resample_bands(x, *out, [0] * bands, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert got.shape == full.shape
    d = (got - full).abs().max().item()
    # same bf16 weights and window alignment; only the f32 summation grouping
    # can differ (a band may get another super-block plan than the whole
    # image), which can flip the bf16 rounding of an intermediate V value —
    # up to ~1 bf16 ulp of V in general (tools/fuzz_paths.py); these three
    # geometries keep identical plans
    assert d <= 1e-5, d


def _rank(rank, ws, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2512_02371_b200 import partition, pipelines
    x = _frames(7, 432, 768, 3)
    s, c = partition.frame_shard(7, ws, rank)
    mine = pipelines.resample(x[3 * s:3 * (s + c)].cuda(), 216, 384).cpu()
    parts = [None] * ws
    dist.all_gather_object(parts, (s, mine.view(torch.int16).numpy()))
    if rank == 0:
        want = pipelines.resample(x.cuda(), 216, 384).cpu().view(torch.int16).numpy()
        got = np.concatenate([m for _, m in sorted(parts, key=lambda t: t[0])], 0)
        q.put(bool(np.array_equal(got, want)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_gloo_ranks_on_one_gpu_bitwise():
    """Two ranks (torch.distributed, gloo for the result gather only), both
    running the real kernels on cuda:0 over their frame shards; the
    concatenated shards equal one call over all frames, bit for bit."""
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True


def test_dynamic_tile_claiming_over_concurrent_streams():
    """In-order tile claiming (the fused kernel's long-launch mode, forced
    here for short launches with TSB_DYNAMIC_TILES=1) keeps one counter pair
    per stream: run_from_host's three concurrent streams and a large single
    launch must reproduce the static-order result bit for bit."""
    import subprocess
    import sys
    code = r"""
import os, sys, torch
from paper_2512_02371_b200 import pipelines
g = torch.Generator(device="cpu").manual_seed(9)
x = torch.rand((36, 540, 960), generator=g).bfloat16()
want = torch.load(sys.argv[1])
one = pipelines.downsample2x(x.cuda()).cpu()
host_out = torch.empty_like(one).pin_memory()
for _ in range(3):
    pipelines.run_from_host(pipelines.downsample2x, x.pin_memory(), host_out, chunk_planes=3)
    torch.cuda.synchronize()
    assert torch.equal(host_out.view(torch.int16), want.view(torch.int16))
assert torch.equal(one.view(torch.int16), want.view(torch.int16))
print("ok")
"""
    import tempfile
    import torch
    from paper_2512_02371_b200 import pipelines
    g = torch.Generator(device="cpu").manual_seed(9)
    x = torch.rand((36, 540, 960), generator=g).bfloat16()
    want = pipelines.downsample2x(x.cuda()).cpu()  # this process: static order
    with tempfile.NamedTemporaryFile(suffix=".pt") as f:
        torch.save(want, f.name)
        env = {**os.environ, "TSB_DYNAMIC_TILES": "1"}
        r = subprocess.run([sys.executable, "-c", code, f.name], capture_output=True, text=True,
                           env=env, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_mixed_pipelines_on_concurrent_streams_match_sequential():
    """Four pipelines (fused separable with in-order tile claiming forced
    on, the persistent axis passes, the f32 kernel and the DCT-16 strips),
    each enqueued repeatedly on its own stream so their kernels overlap —
    programmatic dependent launch, per-stream claim counters and persistent
    CTAs included — reproduce their sequential results bit for bit."""
    import subprocess
    import sys
    code = r"""
import torch
from paper_2512_02371_b200 import pipelines
g = torch.Generator(device="cpu").manual_seed(11)
xs = [torch.rand((6, 1080, 1920), generator=g).bfloat16().cuda(),
      torch.rand((6, 2048, 2048), generator=g).bfloat16().cuda(),
      torch.rand((6, 1080, 1920), generator=g).cuda(),
      torch.rand((3, 1080, 1920), generator=g).bfloat16().cuda()]
fns = [lambda x: pipelines.downsample2x(x), lambda x: pipelines.resample(x, 450, 450),
       lambda x: pipelines.downsample2x(x), lambda x: pipelines.denoise_dct16(x, 0.15)]
want = [f(x) for f, x in zip(fns, xs)]
torch.cuda.synchronize()
streams = [torch.cuda.Stream() for _ in fns]
outs = [[] for _ in fns]
for rep in range(4):
    for i, (f, x, s) in enumerate(zip(fns, xs, streams)):
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            outs[i].append(f(x))
torch.cuda.synchronize()
for w, o in zip(want, outs):
    iw = w.view(torch.int16) if w.dtype == torch.bfloat16 else w.view(torch.int32)
    for y in o:
        iy = y.view(torch.int16) if y.dtype == torch.bfloat16 else y.view(torch.int32)
        assert torch.equal(iy, iw)
print("ok")
"""
    env = {**os.environ, "TSB_DYNAMIC_TILES": "1"}
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=300, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
