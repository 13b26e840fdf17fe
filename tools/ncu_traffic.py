"""DRAM traffic per frame of every bench config's kernels, for bench.py's
roofline.traffic (profiles/ncu_summary.json).

  on the GPU box:  python tools/ncu_traffic.py run CONFIG FRAMES   (the workload, one call)
                   tools/ncu_traffic.sh                            (ncu --set full per config)
  here:            python tools/ncu_traffic.py merge gpurun_out/traffic/*.csv

Each capture runs the config's pipeline call once on FRAMES frames (no
warm-up: ncu replays every kernel with caches flushed, so the bytes are
cold-cache, like the first launch of a step), and sums DRAM read + write
bytes over the call's kernels (f32 cast + fused kernel for c1; both axis
passes, i.e. including the bf16 intermediate, for the two-pass c6 configs)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(cfg, frames):
    import torch
    import bench
    H, W, oh, ow, op, taps, _ = bench.CONFIGS[cfg]
    dt = torch.float32 if cfg == "c1" else torch.bfloat16
    x = torch.rand((frames * 3, H, W), device="cuda").to(dt)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("step")
    bench.make_op(cfg)(x)
    torch.cuda.synchronize()


def merge(paths, prof=None):
    prof = prof or os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(prof)) if os.path.exists(prof) else {}
    for p in paths:
        cfg, frames = os.path.basename(p)[:-4].rsplit("_", 1)
        frames = int(frames)
        out = subprocess.run(["ncu", "-i", p[:-4] + ".ncu-rep", "--page", "raw", "--csv"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        h = rows[0]
        ir, iw, ik = (h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"),
                      h.index("Kernel Name"))
        unit = rows[1][ir]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot, names = 0.0, []
        for r in rows[2:]:
            name = r[ik]
            if not any(k in name for k in ("separable", "axis_pass", "dct16", "cast")):
                continue  # input generation
            tot += float(r[ir].replace(",", "")) * scale[rows[1][ir]]
            tot += float(r[iw].replace(",", "")) * scale[rows[1][iw]]
            names.append(name.split("(")[0][:60])
        summary[cfg] = {"frames": frames, "dram_bytes_per_frame": tot / frames,
                        "source": f"tools/ncu_traffic.py ({cfg}, {frames} frames, --set full)",
                        "kernel": " + ".join(names)}
        print(cfg, frames, f"{tot / frames / 1e6:.1f} MB/frame", names)
    json.dump(summary, open(prof, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], int(sys.argv[3]))
    else:  # merge [--out FILE] CSV...
        args = sys.argv[2:]
        out = None
        if args and args[0] == "--out":
            out, args = args[1], args[2:]
        merge(args, out)
