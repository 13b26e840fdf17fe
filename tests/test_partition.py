"""Partitioner index arithmetic on CPU: frame shards, row bands
with read-only halos, band-local axes and composed axes, checked by
evaluating them with the oracle — including a 2-process gloo run of that
index math.  The same paths on the real kernels (frame shards, row bands,
two ranks on one GPU) are tests/test_gpu_multi.py."""

import os
import socket

import numpy as np
import pytest

from oracle import pipelines_ref
from paper_2512_02371_b200 import filters, partition


@pytest.mark.parametrize("n,ws", [(512, 1), (512, 2), (512, 8), (7, 3), (3, 8), (0, 2)])
def test_frame_shard_covers_exactly(n, ws):
    seen = []
    for r in range(ws):
        s, c = partition.frame_shard(n, ws, r)
        seen.extend(range(s, s + c))
    assert seen == list(range(n))


def test_row_bands_cover_outputs_and_halo():
    first, w = filters.lanczos3_axis(2160, 1080)
    prev = 0
    for r in range(4):
        o0, o1, i0, i1 = partition.row_bands(first, w.shape[1], 2160, 4, r)
        assert o0 == prev and o0 % 16 == 0
        prev = o1
        assert i0 <= max(first[o0], 0) and i1 >= min(first[o1 - 1] + w.shape[1], 2160)
    assert prev == 1080


def _band_result(img, rank, ws, oh, ow):
    H, W = img.shape[-2:]
    rf, rw = pipelines_ref.lanczos3_weights(H, oh)
    o0, o1, i0, i1 = partition.row_bands(rf, rw.shape[1], H, ws, rank)
    bf, bw, bn = partition.band_axis(rf, rw, H, o0, o1, i0, i1)
    return o0, o1, pipelines_ref.separable(img[..., i0:i1, :], (bf, bw),
                                          pipelines_ref.lanczos3_weights(W, ow))


def test_band_axis_matches_full_image():
    rng = np.random.default_rng(0)
    img = rng.random((1, 300, 200), dtype=np.float32)
    full = pipelines_ref.resample(img, 150, 100)
    got = np.zeros_like(full)
    for r in range(3):
        o0, o1, part = _band_result(img, r, 3, 150, 100)
        got[..., o0:o1, :] = part
    np.testing.assert_allclose(got, full, atol=2e-6)


def test_composed_axis_equals_two_passes():
    rng = np.random.default_rng(1)
    img = rng.random((2, 96, 128), dtype=np.float32)
    k = filters.gaussian_taps(9)
    two = pipelines_ref.gaussian_blur(pipelines_ref.resample(img, 48, 64), 9)
    rows = partition.compose_axes(filters.conv_axis(48, k), filters.lanczos3_axis(96, 48), 48, 96)
    cols = partition.compose_axes(filters.conv_axis(64, k), filters.lanczos3_axis(128, 64), 64, 128)
    one = pipelines_ref.separable(img, rows, cols)
    np.testing.assert_allclose(one, two, atol=1e-5)
    assert rows[1].shape[1] <= 30  # 12 Lanczos taps + 8 x stride 2 + alignment


def _worker(rank, ws, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    rng = np.random.default_rng(7)
    img = rng.random((1, 256, 96), dtype=np.float32)
    o0, o1, part = _band_result(img, rank, ws, 128, 48)
    bands = [None] * ws
    dist.all_gather_object(bands, (o0, o1, part))
    # frame sharding of a small batch
    frames = rng.random((5, 32, 32), dtype=np.float32)
    s, c = partition.frame_shard(5, ws, rank)
    mine = pipelines_ref.resample(frames[s:s + c], 16, 16)
    outs = [None] * ws
    dist.all_gather_object(outs, (s, mine))
    if rank == 0:
        full = pipelines_ref.resample(img, 128, 48)
        got = np.zeros_like(full)
        for a, b, p in bands:
            got[..., a:b, :] = p
        ok1 = np.abs(got - full).max() <= 2e-6
        ref = pipelines_ref.resample(frames, 16, 16)
        cat = np.concatenate([m for _, m in sorted(outs, key=lambda t: t[0])], 0)
        ok2 = np.array_equal(cat, ref)
        q.put((bool(ok1), bool(ok2)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_index_math():
    """Index math only: each rank evaluates its row band / frame shard with
    the oracle; the gathered bands equal the full-image oracle."""
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) == (True, True)
