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
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


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
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
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
    time.sleep(0.05)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(K):
        ev[i][0].record(stream)
        y = fn(xs[i % 2])
        ev[i][1].record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = t0.elapsed_time(t1)
    launch_ms = sum(a.elapsed_time(b) for a, b in ev) / K
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
            _pipes.run_from_host(fn, host_in[:n], host_out[:n], chunk_planes=12)

    E = max(1, min(args.e2e_steps, K))
    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(E):
        e2e_step()
    e1.record(stream)
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
        }
        print(json.dumps(line))
    if ws > 1:
        dist.destroy_process_group()


def cpu_baseline(cfg):
    """The oracle (numpy restatement, 1 thread) on a bounded sample."""
    from oracle import pipelines_ref
    H, W, oh, ow, op, taps, _ = CONFIGS[cfg]
    rng = np.random.default_rng(SEED)
    planes = 3 if H * W <= 2160 * 3840 else 1
    img = rng.random((planes, H, W), dtype=np.float32)
    t = time.perf_counter()
    reps = 0
    while True:  # a bounded sample of ~10 s of CPU work (at least one pass)
        if op == "lanczos":
            pipelines_ref.resample(img, oh, ow)
        elif op == "lanczos+gauss":
            pipelines_ref.gaussian_blur(pipelines_ref.resample(img, oh, ow), taps)
        elif op == "dct16":
            pipelines_ref.dct_denoise(img, 0.15, "hard")
        else:
            pipelines_ref.gaussian_blur(img, taps)
        reps += 1
        dt = time.perf_counter() - t
        if dt >= 10.0:
            break
    return {"value": round(reps * H * W * planes / 3 / dt / 1e6, 3), "unit": "Mpixel/s", "cores": 1,
            "kind": "port",
            "sample": f"oracle/pipelines_ref, {reps} pass(es) over {planes} plane(s) of {H}x{W} "
                      f"({dt:.1f} s, 1 thread)"}


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


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
