"""Sharding the image pipelines across the GPUs of one box.

The path has no exchange step: frames are independent, and a row band of
one image needs only a read-only halo of input rows.  So the partitioner is
pure index arithmetic; ``torch.distributed`` is used by callers only for
barriers / timing and for gathering results outside the timed region.

* :func:`frame_shard`  — contiguous frame range of a rank (config 5).
* :func:`row_bands`    — output row range + input halo band of a rank for a
  single large image; :func:`band_axis` rebuilds the rows axis for the band
  so clamp-to-edge still refers to the true image edges.
* :class:`FrameSharder` — runs a pipeline over a rank's frame shard in
  chunks, on the rank's own GPU and stream.
* :func:`run_sharded`  — one process driving several GPUs: a batch of
  frames in pinned host memory is split into contiguous frame shards, each
  streamed host -> device -> host on its own device (own streams, own
  weight-axis cache) with no inter-GPU traffic.
* :func:`separable_bands` / :func:`resample_bands` — one large image split
  into output row bands, one per device: each device reads its band plus a
  read-only halo, runs the fused kernel on a band-local rows axis and writes
  disjoint output rows.
"""

from __future__ import annotations

import numpy as np


def frame_shard(n_frames: int, world_size: int, rank: int):
    """(start, count) of rank's frames: contiguous, sizes differ by <= 1."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError(f"bad rank {rank} / world size {world_size}")
    base, extra = divmod(n_frames, world_size)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def row_bands(first, taps: int, n_in: int, world_size: int, rank: int, align: int = 16,
              in_align: int = 16):
    """Split the outputs of an axis into `world_size` bands (multiples of
    `align` rows except the last) and return rank's
    (out_start, out_stop, in_start, in_stop) — the input rows its outputs
    read, clamped to the image.  in_start is rounded down to a multiple of
    `in_align`, so the band-local axis keeps the full axis's window
    alignment (the builder places 16-output windows on multiples of 8)."""
    first = np.asarray(first)
    n_out = len(first)
    blocks = -(-n_out // align)
    b0, nb = frame_shard(blocks, world_size, rank)
    o0, o1 = b0 * align, min((b0 + nb) * align, n_out)
    if o0 >= o1:
        return o0, o0, 0, 0
    lo = int(first[o0:o1].min())
    hi = int(first[o0:o1].max()) + taps
    lo = max(lo, 0) // in_align * in_align
    return o0, o1, lo, min(hi, n_in)


def band_axis(first, weights, n_in: int, out_start: int, out_stop: int, in_start: int,
              in_stop: int):
    """(first, weights, n_in) of the rows axis restricted to a band.  Taps
    are clamped against the *image* [0, n_in) first, then re-based to the
    band, so a band-local run is identical to the full-image run."""
    first = np.asarray(first, np.int64)[out_start:out_stop]
    weights = np.asarray(weights, np.float32)[out_start:out_stop]
    taps = weights.shape[1]
    idx = np.clip(first[:, None] + np.arange(taps)[None, :], 0, n_in - 1) - in_start
    if idx.size and (idx.min() < 0 or idx.max() >= in_stop - in_start):
        raise ValueError("band does not cover the outputs' taps")
    # re-express with per-output explicit indices: first = min index, dense weights
    f2 = idx.min(axis=1)
    span = int((idx.max(axis=1) - f2).max()) + 1 if idx.size else 1
    w2 = np.zeros((len(f2), span), np.float32)
    for t in range(taps):
        np.add.at(w2, (np.arange(len(f2)), idx[:, t] - f2), weights[:, t])
    return f2.astype(np.int32), w2, in_stop - in_start


def compose_axes(outer, inner, n_mid: int, n_in: int):
    """Compose two banded axes: outer (n_out x n_mid) after inner
    (n_mid x n_in), each given as (first, weights) with clamp-to-edge on its
    own input.  Returns (first, weights) of the product axis, indices
    already clamped into [0, n_in) (the builder's clamp is then a no-op).
    Used to fuse resample -> filter into a single pass (config 5)."""
    of, ow = np.asarray(outer[0], np.int64), np.asarray(outer[1], np.float64)
    inf_, iw = np.asarray(inner[0], np.int64), np.asarray(inner[1], np.float64)
    n_out, to = ow.shape
    ti = iw.shape[1]
    # inner rows as dense segments over clamped input indices
    rows = []
    for j in range(n_mid):
        idx = np.clip(inf_[j] + np.arange(ti), 0, n_in - 1)
        rows.append((idx, iw[j]))
    firsts, segs = [], []
    for o in range(n_out):
        acc = {}
        for t in range(to):
            j = min(max(int(of[o]) + t, 0), n_mid - 1)
            idx, w = rows[j]
            for i, v in zip(idx, w):
                acc[int(i)] = acc.get(int(i), 0.0) + ow[o, t] * v
        lo, hi = min(acc), max(acc)
        seg = np.zeros(hi - lo + 1)
        for i, v in acc.items():
            seg[i - lo] = v
        firsts.append(lo)
        segs.append(seg)
    taps = max(len(s) for s in segs)
    w = np.zeros((n_out, taps), np.float32)
    for o, s in enumerate(segs):
        w[o, :len(s)] = s
    return np.asarray(firsts, np.int32), w


class FrameSharder:
    """Run `fn(batch)` over this rank's shard of `n_frames` planar frames
    (`planes_per_frame` planes each) in chunks of `chunk` frames."""

    def __init__(self, n_frames: int, world_size: int = 1, rank: int = 0,
                 planes_per_frame: int = 3, chunk: int = 16):
        self.start, self.count = frame_shard(n_frames, world_size, rank)
        self.ppf = planes_per_frame
        self.chunk = max(1, chunk)

    def chunks(self):
        f = self.start
        end = self.start + self.count
        while f < end:
            n = min(self.chunk, end - f)
            yield f, n
            f += n

    def run(self, frames, fn, out=None):
        """frames: (n_local*ppf, H, W) tensor holding this rank's frames
        (local index 0 = global frame `start`); returns fn over all chunks
        concatenated along dim 0 (or writes into `out`)."""
        results = []
        for f, n in self.chunks():
            lo = (f - self.start) * self.ppf
            y = fn(frames[lo:lo + n * self.ppf])
            if out is not None:
                out[lo:lo + n * self.ppf].copy_(y)
            else:
                results.append(y)
        if out is not None:
            return out
        import torch
        return torch.cat(results, 0) if results else None


def run_sharded(fn, host_in, host_out, devices, *, planes_per_frame: int = 3,
                chunk_planes: int = 3):
    """Run `fn` (a pipeline of :mod:`pipelines`) over a batch of frames held in
    (pinned) host memory on several devices from ONE process: frame shards
    (:func:`frame_shard`) go to ``devices`` in order, each streamed through
    :func:`pipelines.run_from_host` on that device (its own copy/compute
    streams and weight-axis cache).  All shards are enqueued before any is
    waited on, so the devices run concurrently; returns host_out once every
    device has finished.  No data moves between devices."""
    import torch

    from . import pipelines
    devices = [int(d) for d in devices]
    if not devices:
        raise ValueError("run_sharded needs at least one device")
    P = host_in.shape[0]
    if P % planes_per_frame:
        raise ValueError(f"{P} planes is not a whole number of {planes_per_frame}-plane frames")
    n_frames = P // planes_per_frame
    done = []
    for r, d in enumerate(devices):
        s, c = frame_shard(n_frames, len(devices), r)
        if c == 0:
            continue
        lo, hi = s * planes_per_frame, (s + c) * planes_per_frame
        with torch.cuda.device(d):
            pipelines.run_from_host(fn, host_in[lo:hi], host_out[lo:hi], chunk_planes=chunk_planes)
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(d))
            done.append(ev)
    for ev in done:
        ev.synchronize()
    return host_out


def separable_bands(x, rows, cols, n_out_rows: int, n_out_cols: int, devices, *,
                    out_dtype=None):
    """One large image (planes x H x W, on any device) as output row bands,
    one per entry of ``devices``: band r reads input rows [in_start, in_stop)
    (its outputs' taps, clamped to the image) and writes output rows
    [out_start, out_stop).  rows / cols are (first, weights) of the two
    axes over the FULL image; each band runs the fused kernel on a
    band-local rows axis (:func:`band_axis`).  Returns the assembled output
    on x's device."""
    import torch

    from . import axis as _axis, pipelines
    H, W = x.shape[-2:]
    rf, rw = np.asarray(rows[0]), np.asarray(rows[1], np.float32)
    cf, cw = np.asarray(cols[0]), np.asarray(cols[1], np.float32)
    taps = rw.shape[1]
    out_dtype = out_dtype or x.dtype
    out = torch.empty(x.shape[:-2] + (n_out_rows, n_out_cols), dtype=out_dtype, device=x.device)
    parts = []
    for r, d in enumerate(devices):
        o0, o1, i0, i1 = row_bands(rf, taps, H, len(devices), r)
        if o0 >= o1:
            continue
        bf, bw, bn = band_axis(rf, rw, H, o0, o1, i0, i1)
        # cached: an Axis frees its device tiles when collected, and the
        # band's kernel is still in flight when this function returns
        ra = _axis.cached(("band", bn, o1 - o0, bf.tobytes(), bw.tobytes(), int(d)),
                          lambda: _axis.Axis(bn, o1 - o0, bf, bw, device=int(d)))
        ca = _axis.cached(("cols", W, n_out_cols, cf.tobytes(), cw.tobytes(), int(d)),
                          lambda d=d: _axis.Axis(W, n_out_cols, cf, cw, device=int(d)))
        with torch.cuda.device(int(d)):
            xb = x[..., i0:i1, :].to(f"cuda:{int(d)}", non_blocking=True)
            yb = pipelines.separable(xb, ra, ca, out_dtype=out_dtype)
        parts.append((o0, o1, yb))
    for o0, o1, yb in parts:
        out[..., o0:o1, :].copy_(yb, non_blocking=True)
    return out


def resample_bands(x, out_h: int, out_w: int, devices, *, out_dtype=None):
    """Lanczos-3 resample of one large image split into row bands over
    ``devices`` (:func:`separable_bands`)."""
    from . import filters
    H, W = x.shape[-2:]
    return separable_bands(x, filters.lanczos3_axis(H, out_h), filters.lanczos3_axis(W, out_w),
                           out_h, out_w, devices, out_dtype=out_dtype)
