"""Summarise an ncu report (--set full) and a launch list into profiles/.

    python tools/ncu_summary.py REPORT.ncu-rep LAUNCHES.csv|- OUT_PREFIX [frames] [alg_bytes_per_frame]

(the default algorithmic bytes per frame are config c2's: 4K RGB bf16 in, 1080p bf16 out)
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
        "sm__cycles_elapsed.avg", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        # tensor pipe (tcgen05) and TMEM activity; ncu 2025 prefixes these with their section
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active"]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            name = h.split(".", 2)[-1] if h.split(".")[0] in ("TPC", "SM_C", "GPC", "SM_A") else h
            if name in KEYS or h == "Kernel Name":
                d[name] = (v, u)
        res.append(d)
    return res


def to_bytes(v, u):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def launches(path):
    agg = defaultdict(list)
    for r in csv.DictReader(l for l in open(path) if l.startswith('"')):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            agg[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    return [{"kernel": k, "launches": len(v), "total_us": sum(v) / 1e3,
             "avg_us": sum(v) / len(v) / 1e3, "share": sum(v) / tot}
            for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))]


def main():
    report, lcsv, prefix = sys.argv[1:4]
    frames = int(sys.argv[4]) if len(sys.argv) > 4 else 8
    k = raw(report)[0]
    v, u = k["gpu__time_duration.sum"]
    dur_us = float(v.replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
                                          "msecond": 1e3, "ms": 1e3, "second": 1e6,
                                          "s": 1e6}.get(u.strip(), 1.0)
    rd = to_bytes(*k["dram__bytes_read.sum"])
    wr = to_bytes(*k["dram__bytes_write.sum"])
    per_frame = int(sys.argv[5]) if len(sys.argv) > 5 else 3 * 2160 * 3840 * 2 + 3 * 1080 * 1920 * 2
    alg = frames * per_frame
    summary = {
        "kernel": k["Kernel Name"][0][:120],
        "frames": frames,
        "duration_us": dur_us,
        "dram_read_bytes": rd, "dram_write_bytes": wr,
        "dram_bytes_per_frame": (rd + wr) / frames,
        "alg_bytes": alg, "alg_bytes_per_frame": per_frame, "traffic_over_alg": (rd + wr) / alg,
        "achieved_alg_GBps": alg / dur_us / 1e3,
        "metrics": {h: " ".join(v) for h, v in k.items() if h != "Kernel Name"},
        "launch_list": launches(lcsv) if lcsv != "-" else None,
    }
    json.dump(summary, open(prefix + ".json", "w"), indent=1)
    print(json.dumps({x: summary[x] for x in ("duration_us", "traffic_over_alg",
                                              "achieved_alg_GBps", "dram_bytes_per_frame")}))
    for l in summary["launch_list"] or []:
        print(f"  {l['share']*100:5.1f}%  {l['launches']:4d} x {l['avg_us']:9.2f} us  {l['kernel'][:90]}")


if __name__ == "__main__":
    main()
