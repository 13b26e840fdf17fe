#!/usr/bin/env python
"""Benchmark: Mpixels/s of the B200 image pipelines (BASELINE.json metric).

Default workload (config c2 of BASELINE.json): 4K (3840x2160) RGB bf16
frames -> 1080p with separable Lanczos-3 2x resampling, fp32 accumulate,
bf16 out, planar; a *step* is one fused-kernel pass over a batch of
``--frames`` frames per GPU.  Pixels are input-frame pixels (W x H, RGB
counted once).

    python bench.py [--gpus N --steps K --warmup W]            # B200 arm
    python bench.py --impl reference [--steps K --warmup W]    # reference CPU arm
    torchrun --nproc-per-node N bench.py --gpus N ...          # N GPUs, weak scaling

Prints ONE JSON line (rank 0).  ``value`` is device-timed (CUDA events,
barrier + synchronize around the timed region, max over ranks) with inputs
resident in HBM; two alternating input batches larger than L2 are used.
``e2e`` runs the same workload through the public API from pinned host
memory (H2D of the frames + kernel + D2H of the result, every step).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 0x251202371

CONFIGS = {
    # name: (H, W, out_h, out_w, op, taps, description)
    "c2": (2160, 3840, 1080, 1920, "lanczos", 0,
           "c2: 4K (3840x2160) RGB bf16 -> 1080p, separable Lanczos-3 2x, fp32 accumulate, bf16 out"),
    "c1": (1080, 1920, 540, 960, "lanczos", 0,
           "c1: 1080p RGB f32 -> 540p, separable Lanczos-3 2x, f32 throughout (FMA pipe, bit-exact to the reference), f32 out"),
    "c3-9": (4320, 7680, 4320, 7680, "gauss", 9, "c3: 8K RGB bf16 separable Gaussian, 9 taps"),
    "c3-15": (4320, 7680, 4320, 7680, "gauss", 15, "c3: 8K RGB bf16 separable Gaussian, 15 taps"),
    "c3-21": (4320, 7680, 4320, 7680, "gauss", 21, "c3: 8K RGB bf16 separable Gaussian, 21 taps"),
    "c3-31": (4320, 7680, 4320, 7680, "gauss", 31, "c3: 8K RGB bf16 separable Gaussian, 31 taps"),
    "c4": (2160, 3840, 2160, 3840, "dct16", 0,
           "c4: 4K RGB bf16 DCT-16 transform-domain denoise (16x16 tiles, stride 8, hard coring "
           "threshold 0.15, windowed overlap-add), one fused kernel, bf16 out"),
    "c5": (2160, 3840, 1080, 1920, "lanczos+gauss", 9,
           "c5: batch of 512 4K RGB bf16 frames -> 1080p Lanczos-3 2x then 9-tap Gaussian "
           "(composed into one fused pass), frame-sharded across GPUs"),
}
# the paper's non-integer block-sparse table, 2048^2 -> N^2
for _n in (143, 245, 450, 921):
    CONFIGS[f"c6-{_n}"] = (2048, 2048, _n, _n, "lanczos", 0,
                           f"c6: 2048x2048 RGB bf16 -> {_n}x{_n} Lanczos-3 (non-integer "
                           f"{2048 / _n:.2f}x), fp32 accumulate, bf16 out")
C5_FRAMES = 512


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--frames", type=int, default=16, help="frames per GPU per step")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled in-process through
    NVML every `period` seconds on a background thread while the GPU is
    under load.  `mark()` splits the samples into the pre-roll (the loaded
    warm-up just before the timed region) and the timed region itself, so
    even a few-millisecond timed region reports clocks under load."""

    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20),
               ("hw_thermal_slowdown", 0x40), ("sw_power_cap", 0x4), ("hw_power_brake", 0x80))

    def __init__(self, gpu_index, period=0.0005):
        self.gpu, self.period = gpu_index, period
        self.samples, self.t_mark = [], None
        self._stop = None
        self._th = None

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = None
            try:  # NVML numbers GPUs ignoring CUDA_VISIBLE_DEVICES: match by PCI bus id
                import torch
                pr = torch.cuda.get_device_properties(self.gpu)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = None
            if h is None:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # no NVML: report why instead of inventing clocks
            self.err = f"nvml unavailable: {e}"
            return
        self.err = None
        self._stop = threading.Event()

        def loop():
            while not self._stop.is_set():
                try:
                    mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:
                    break
                self.samples.append((time.perf_counter(), mhz, rs))
                time.sleep(self.period)

        self._th = threading.Thread(target=loop, daemon=True)
        self._th.start()

    def mark(self):
        self.t_mark = time.perf_counter()

    def stop(self):
        if self._stop is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err], "samples": 0}
        self._stop.set()
        self._th.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        timed = [x for x in self.samples if self.t_mark is not None and x[0] >= self.t_mark]
        mhz = [m for _, m, _ in self.samples]
        reasons = sorted({n for _, _, r in self.samples for n, bit in self.REASONS if r & bit})
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples),
                "samples_timed": len(timed),
                "sm_mhz_timed": statistics.median([m for _, m, _ in timed]) if timed else None,
                "source": f"NVML every {self.period * 1e3:.1f} ms during the timed region"}


# --------------------------------------------------------------- B200 arm
def make_op(cfg):
    from paper_2512_02371_b200 import pipelines
    H, W, oh, ow, op, taps, _ = CONFIGS[cfg]
    if op == "lanczos":
        return lambda x: pipelines.resample(x, oh, ow)
    if op == "lanczos+gauss":
        return lambda x: pipelines.resample_filter(x, oh, ow, taps)
    if op == "dct16":
        return lambda x: pipelines.denoise_dct16(x, 0.15, "hard")
    return lambda x: pipelines.gaussian_blur(x, taps)


def run_b200(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)  # before the NCCL group: each rank on its own GPU
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    H, W, oh, ow, op, taps, desc = CONFIGS[args.config]
    F = args.frames
    strong = args.config == "c5"
    if strong:
        from paper_2512_02371_b200 import partition
        _, F = partition.frame_shard(C5_FRAMES, ws, rank)
    in_dtype = torch.float32 if args.config == "c1" else torch.bfloat16
    out_es = 4 if args.config == "c1" else 2
    fn = make_op(args.config)

    g = torch.Generator(device=dev)
    g.manual_seed(SEED + rank)
    nbuf = 1 if strong else 2  # c5: the whole 512-frame batch is resident (> L2 by 200x)
    xs = []
    if op == "dct16":  # smooth pattern + N(0, 0.05^2), clipped
        yy = torch.arange(H, device=dev, dtype=torch.float32)[:, None]
        xx = torch.arange(W, device=dev, dtype=torch.float32)[None, :]
        clean = 0.5 + 0.4 * torch.sin(xx / 17.0) * torch.cos(yy / 23.0)
    for _ in range(nbuf):
        x = torch.empty((F * 3, H, W), dtype=in_dtype, device=dev)
        for c0 in range(0, F * 3, 48):  # fill in chunks to bound the f32 temporary
            n = min(48, F * 3 - c0)
            if op == "dct16":
                x[c0:c0 + n] = (clean + 0.05 * torch.randn((n, H, W), generator=g, device=dev)
                                ).clamp_(0, 1)
            else:
                x[c0:c0 + n] = torch.rand((n, H, W), generator=g, device=dev)
        xs.append(x)
    xs = xs * (2 // nbuf)
    in_bytes = xs[0].numel() * xs[0].element_size()
    out_bytes = F * 3 * oh * ow * out_es
    stream = torch.cuda.current_stream(dev)

    for i in range(max(args.warmup, 3)):
        y = fn(xs[i % 2])
    torch.cuda.synchronize()

    # ---- device-timed region
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(K)]
    clocks = ClockSampler(local)
    clocks.start()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("bench.timed")
    t0.record(stream)
    for i in range(K):
        ev[i][0].record(stream)
        y = fn(xs[i % 2])
        ev[i][1].record(stream)
    t1.record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = t0.elapsed_time(t1)
    # sustained: the same step back to back for ~1 s after the timed region
    # (reported beside `value`, which is the K-step region above): under
    # sustained load the B200 reaches its power cap and the SM clock drops
    sus = ClockSampler(local, period=0.005)
    sus.start()
    sus.mark()
    n_sus, s0, s1 = 0, torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    t_sus = time.perf_counter()
    while time.perf_counter() - t_sus < 1.0:
        for i in range(8):
            y = fn(xs[i % 2])
        n_sus += 8
        torch.cuda.synchronize()
    s1.record(stream)
    torch.cuda.synchronize()
    sus_clk = sus.stop()
    sus_ms = s0.elapsed_time(s1) / n_sus
    per_step = [a.elapsed_time(b) for a, b in ev]
    launch_ms = sum(per_step) / K
    median_ms = statistics.median(per_step)
    t = torch.tensor([total_ms, launch_ms], device=dev, dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, launch_ms = float(t[0]), float(t[1])
    ms_step = total_ms / K
    pix_step = (C5_FRAMES if strong else F * ws) * H * W
    value = pix_step / (ms_step / 1e3) / 1e6

    # ---- end to end through the public API from pinned host memory: every
    # step moves all of the step's frames host->device and the results back
    # (in chunks of <= 32 frames through one pinned staging pair)
    ch = min(F, 32)
    host_in = xs[0][:ch * 3].cpu().pin_memory()
    host_out = torch.empty((ch * 3, oh, ow), dtype=y.dtype).pin_memory()
    n_chunks = -(-F // ch)

    from paper_2512_02371_b200 import pipelines as _pipes

    def e2e_step():
        # pipelines.run_from_host overlaps H2D / kernels / D2H over 3 streams
        for c in range(n_chunks):
            n = min(ch, F - c * ch) * 3
            _pipes.run_from_host(fn, host_in[:n], host_out[:n], chunk_planes=3)

    E = max(1, min(args.e2e_steps, K))
    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("bench.e2e")
    e0.record(stream)
    for _ in range(E):
        e2e_step()
    e1.record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / E], device=dev, dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms[0])

    peak, peak_kind = measured_peaks()
    launches_per_step = 1
    if op == "dct16":
        kernel_name = "tsb::dct::dct16_kernel (fused DCT-16 denoise)"
    else:
        from paper_2512_02371_b200 import axis as _ax, pipelines as _pl
        ra = _ax.lanczos3(H, oh, local) if op.startswith("lanczos") else None
        fused = ra is None or _pl.fused_supported(ra, _ax.lanczos3(W, ow, local), F * 3)
        kernel_name = ("tsb::separable_kernel (fused V+H tcgen05 pass)" if fused else
                       "tsb::axis_pass_kernel x2 (vertical + horizontal, bf16 intermediate; "
                       "alg bytes exclude the intermediate)")
        launches_per_step = 1 if fused else 2
        if in_dtype == torch.float32:  # pipelines._run_f32: one f32 kernel, no bf16 copy
            kernel_name = "tsb::separable_f32_kernel<2,12,3> (f32 FMA-pipe fused H+V pass" + (", exact roundings)" if _pl.F32_EXACT else ")")
            launches_per_step = 1
    alg_bytes = in_bytes + out_bytes  # per launch per GPU
    achieved = alg_bytes / (launch_ms / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            d = json.load(open(prof)).get(args.config)
            if d and d.get("frames"):
                traffic = d["dram_bytes_per_frame"] * F
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config)

    if rank == 0:
        line = {
            "metric": "Mpixels/sec per pipeline (input pixels, RGB counted once)",
            "value": round(value, 1),
            "unit": "Mpixel/s",
            "n_gpus": ws,
            "steps": K,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 5),
            "ms_per_step_median": round(median_ms, 5),  # median of >= 20 steps
            "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": ("synthetic (smooth pattern + N(0, 0.05^2) noise, clipped to [0,1], planar RGB, "
                     "seed 0x251202371+rank)" if op == "dct16" else
                     "synthetic (uniform [0,1) planar RGB, seed 0x251202371+rank)"),
            "config": {
                "workload": desc,
                "frames_per_step_per_gpu": F,
                "input": f"{F}x3x{H}x{W} {'f32' if in_dtype == torch.float32 else 'bf16'} per GPU",
                "output": f"{F}x3x{oh}x{ow}",
                "l2": (f"resident batch of {in_bytes / 1e6:.0f} MB per GPU (> 126 MB L2)" if strong
                       else f"two alternating input batches of {in_bytes / 1e6:.0f} MB each (> 126 MB L2)"),
                "parallelism": f"frame-sharded dp{ws}, no collectives on the data path",
            },
            "e2e": {"value": round(pix_step / (e2e_ms / 1e3) / 1e6, 1), "unit": "Mpixel/s",
                    "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": out_bytes,
                    "api": "paper_2512_02371_b200.pipelines.run_from_host (pinned host -> device -> "
                           "host, copies overlapped with kernels over 3 streams)"},
            "gpu_launches": K * launches_per_step,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1),
                         "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                         "traffic": traffic,
                         "alg_bytes_per_launch": alg_bytes,
                         "kernel": kernel_name,
                         "avg_launch_ms": round(launch_ms, 5)},
            "cpu_baseline": cpu,
            "clocks": clk,
            "sustained": {"value": round(pix_step / (sus_ms / 1e3) / 1e6, 1), "unit": "Mpixel/s",
                          "ms_per_step": round(sus_ms, 5), "steps": n_sus,
                          "roofline_frac": round(alg_bytes / (sus_ms / 1e3) / 1e9 / peak, 4),
                          "sm_mhz": sus_clk.get("sm_mhz"), "reasons": sus_clk.get("reasons"),
                          "note": "same step back to back for ~1 s after the timed region "
                                  "(synchronised every 8 steps); not the headline"},
        }
        print(json.dumps(line))
    if ws > 1:
        dist.destroy_process_group()


_CPU = {}


def _cpu_band(band):
    """One output row band of the oracle pipeline (worker process; numpy
    single-threaded): the band's input rows plus halo are sliced from the
    full image, the row axis keeps the full image's clamp-to-edge."""
    from oracle import pipelines_ref as R
    img, op, taps, oh, ow = (_CPU[k] for k in ("img", "op", "taps", "oh", "ow"))
    o0, o1 = band
    H, W = img.shape[-2:]
    if op == "dct16":  # 8-row halo: every kept output row sees both its tile rows
        i0, i1 = max(o0 - 8, 0), min(o1 + 8, H)
        return R.dct_denoise(img[:, i0:i1], 0.15, "hard")[:, o0 - i0:o0 - i0 + (o1 - o0)]
    if op in ("lanczos", "lanczos+gauss"):  # (c5's 9-tap filter runs on the assembled frame)
        rows, cols = R.lanczos3_weights(H, oh), R.lanczos3_weights(W, ow)
    else:
        k = R.gaussian_kernel(taps)
        rows, cols = R.centred_axis(H, k), R.centred_axis(W, k)
    f, w = rows
    idx = np.clip(f[o0:o1, None] + np.arange(w.shape[1])[None, :], 0, H - 1)
    i0, i1 = int(idx.min()), int(idx.max()) + 1
    h = R.axis_pass(img[:, i0:i1], cols[0], cols[1], axis=-1)
    return R.axis_pass(h, np.asarray(f[o0:o1]) - i0, w[o0:o1], axis=-2)


def cpu_baseline(cfg):
    """The oracle (numpy restatement) on a bounded sample, spread over all
    host cores: output row bands of the frame, one process per core."""
    import multiprocessing as mp
    from oracle import pipelines_ref
    H, W, oh, ow, op, taps, _ = CONFIGS[cfg]
    rng = np.random.default_rng(SEED)
    planes = 3 if H * W <= 2160 * 3840 else 1
    img = rng.random((planes, H, W), dtype=np.float32)
    cores = os.cpu_count() or 1
    n_out = H if op in ("dct16", "gauss") else oh
    step = 8 if op == "dct16" else 1
    nb = max(1, min(cores * 4, n_out // max(step, 16)))
    edges = [(i * n_out // nb) // step * step for i in range(nb)] + [n_out]
    bands = [(a, b) for a, b in zip(edges[:-1], edges[1:]) if b > a]
    _CPU.update(img=img, op=op, taps=taps, oh=oh, ow=ow)
    env_threads = os.environ.get("OMP_NUM_THREADS")
    os.environ["OMP_NUM_THREADS"] = "1"
    ctx = mp.get_context("fork")
    t = time.perf_counter()
    reps = 0
    with ctx.Pool(cores) as pool:
        while True:  # a bounded sample of ~10 s of CPU work (at least one pass)
            parts = pool.map(_cpu_band, bands)
            if op == "lanczos+gauss":  # the 9-tap filter over the assembled 1080p frame
                pipelines_ref.gaussian_blur(np.concatenate(parts, axis=-2), taps)
            reps += 1
            dt = time.perf_counter() - t
            if dt >= 10.0:
                break
    if env_threads is None:
        os.environ.pop("OMP_NUM_THREADS", None)
    else:
        os.environ["OMP_NUM_THREADS"] = env_threads
    return {"value": round(reps * H * W * planes / 3 / dt / 1e6, 3), "unit": "Mpixel/s",
            "cores": cores, "kind": "port",
            "sample": f"oracle/pipelines_ref over {len(bands)} output row bands of {planes} "
                      f"plane(s) of {H}x{W}, {reps} pass(es) in {dt:.1f} s, {cores} processes"}


# ---------------------------------------------------------- reference arm
_REF = {}


def _ref_init(taps, stride, n_out, in_len):
    sys.dont_write_bytecode = True
    refdir = os.path.join(ROOT, "baseline", "_ref")
    sys.path.insert(0, refdir)
    from tensorsel import interp, selector
    from tensorsel.ir import (Allocate, Bop, Broadcast, Cast, Imm, Load, Param, Program, Ramp,
                              ShapeDecl, Store, VecType, VectorReduceAdd)

    def i32(v):
        return Imm("i32", v)

    lanes = n_out * taps
    i_idx = Ramp(Ramp(i32(0), i32(1), taps), Broadcast(i32(stride), taps), n_out)
    i_op = Cast(VecType("f32", lanes), Load("I", VecType("f16", lanes), i_idx))
    k_op = Broadcast(Cast(VecType("f32", taps), Load("K", VecType("f16", taps),
                                                     Ramp(i32(0), i32(1), taps))), n_out)
    flat = Ramp(i32(0), i32(1), n_out)
    acc = Load("conv", VecType("f32", n_out), flat)
    body = (Allocate("conv", "f32", n_out, "wmma"),
            Store("conv", flat, Broadcast(Imm("f32", 0.0), n_out)),
            Store("conv", flat, Bop("+", VectorReduceAdd(n_out, Bop("*", i_op, k_op)), acc)),
            Store("output", flat, Load("conv", VecType("f32", n_out), flat)))
    m, n = 32, n_out // 32
    shapes = (ShapeDecl("wmma", m, stride * n + taps, n),)
    prog = Program((Param("K", "f16", taps), Param("I", "f16", in_len),
                    Param("output", "f32", n_out)), body, shapes)
    low, rep = selector.select_program(prog, selector.SelectionConfig(target="wmma"))
    _REF.update(interp=interp, prog=low if rep.ok else prog, lowered=bool(rep.ok),
                K=np.asarray(interp.round_f16(np.linspace(-0.1, 0.5, taps)), np.float32),
                I=np.asarray(interp.round_f16(np.random.default_rng(1).random(in_len)), np.float32),
                out=np.zeros(n_out, np.float32))


def _ref_work(n):
    interp = _REF["interp"]
    t = time.perf_counter()
    for _ in range(n):
        interp.run_program(_REF["prog"], {"K": _REF["K"], "I": _REF["I"], "output": _REF["out"]})
    return time.perf_counter() - t, _REF["lowered"]


def run_reference(args):
    """The reference's own CPU path: interp.run_program on lowered 256-output
    tile statements (tools/make_corpus.py:142-150 template, (wmma-shape 32 k 8)
    declared), one process per host core; the frame rate is extrapolated from
    the measured statements/s."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    H, W, oh, ow, op, taps, desc = CONFIGS[args.config]
    stride = 2 if op == "lanczos" else 1
    taps = 12 if op == "lanczos" else taps
    n_out = 256
    in_len = (32 - 1) * (stride * (n_out // 32)) + stride * (n_out // 32) + taps
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    have_ref = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "tensorsel"))
    if not have_ref:
        return run_reference_port(args, cores)
    # statements per frame: H pass over every input row, V pass over every output column
    planes = 3
    stmts = planes * (H * -(-ow // n_out) + ow * -(-oh // n_out))
    per_proc = 8
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_ref_init, initargs=(taps, stride, n_out, in_len)) as pool:
        pool.map(_ref_work, [1] * cores)
        times = []
        for i in range(args.warmup + args.steps):
            t = time.perf_counter()
            res = pool.map(_ref_work, [per_proc] * cores)
            dt = time.perf_counter() - t
            if i >= args.warmup:
                times.append(dt)
        lowered = all(r[1] for r in res)
    sec = statistics.median(times)
    stmt_rate = cores * per_proc / sec
    frame_s = stmts / stmt_rate
    value = H * W / frame_s / 1e6
    line = {
        "impl": "reference",
        "metric": "Mpixels/sec per pipeline (input pixels, RGB counted once)",
        "value": round(value, 4), "unit": "Mpixel/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16 (reference lowers f16 only)",
        "data": "synthetic",
        "config": {"workload": desc, "statements_per_frame": stmts,
                   "statement": f"{n_out}-output conv statement, {taps} taps, stride {stride}, "
                                f"{'lowered to wmma_mma' if lowered else 'source form'}"},
        "cpu_baseline": {"value": round(value, 4), "unit": "Mpixel/s", "cores": cores,
                         "kind": "reference",
                         "sample": f"{cores}x{per_proc} tile statements per step via "
                                   "baseline/_ref tensorsel interp.run_program"},
        "e2e": {"value": round(value, 4), "unit": "Mpixel/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_reference_port(args, cores):
    from oracle import pipelines_ref
    H, W, oh, ow, op, taps, desc = CONFIGS[args.config]
    rng = np.random.default_rng(SEED)
    band = 64
    img = rng.random((1, band * 2, W), dtype=np.float32)
    times = []
    for i in range(args.warmup + args.steps):
        t = time.perf_counter()
        if op == "lanczos":
            pipelines_ref.resample(img, band, ow)
        else:
            pipelines_ref.gaussian_blur(img, taps)
        if i >= args.warmup:
            times.append(time.perf_counter() - t)
    sec = statistics.median(times)
    value = img.shape[1] * W / sec / 1e6 / 3
    print(json.dumps({
        "impl": "reference", "metric": "Mpixels/sec per pipeline (input pixels, RGB counted once)",
        "value": round(value, 4), "unit": "Mpixel/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": desc},
        "cpu_baseline": {"value": round(value, 4), "unit": "Mpixel/s", "cores": 1, "kind": "port",
                         "sample": f"oracle row band {img.shape[1]}x{W} (baseline/_ref absent)"},
        "e2e": {"value": round(value, 4), "unit": "Mpixel/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}))


def launch_ranks(args):
    """`bench.py --gpus N` without a torchrun environment: relaunch this
    script under torch.distributed.run with N ranks (one process per GPU) and
    pass its output through.  Returns the exit code."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    ws = int(os.environ.get("WORLD_SIZE", "0"))
    if ws == 0 and args.gpus > 1:
        if args.impl != "reference":
            import torch
            if torch.cuda.device_count() < args.gpus:
                sys.exit(f"bench.py: --gpus {args.gpus} but only {torch.cuda.device_count()} "
                         "CUDA device(s) are visible")
        sys.exit(launch_ranks(args))
    if ws and ws != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; refusing to time a "
                 "different number of GPUs than asked for")
    if args.impl == "reference":
        run_reference(args)
    else:
        import torch
        if torch.cuda.device_count() < max(1, args.gpus):
            sys.exit(f"bench.py: --gpus {args.gpus} but only {torch.cuda.device_count()} "
                     "CUDA device(s) are visible")
        run_b200(args)


if __name__ == "__main__":
    main()
