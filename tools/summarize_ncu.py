"""Summarise gpurun_out ncu artefacts into profiles/ (tracked evidence).

  python tools/summarize_ncu.py launches <launches.csv> <out.txt> [header]
  python tools/summarize_ncu.py full <report.ncu-rep> <out.txt> [header]
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path, out, header):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"]
        v = float(d["Metric Value"].replace(",", ""))
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    with open(out, "w") as f:
        f.write(f"# {header}\n# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised)\n")
        f.write("# kernel | launches | total_ns | avg_ns | share\n")
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k} | {c} | {t:.0f} | {t / c:.0f} | {t / tot:.4f}\n")


KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Issued Warp Per Scheduler", "Eligible Warps Per Scheduler", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Block Size", "Grid Size", "Theoretical Occupancy", "Achieved Occupancy", "Block Limit Registers",
        "Block Limit Shared Mem", "FP64", "fp64", "Bank Conflicts", "Local", "Roofline"]


def full(path, out, header):
    txt = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    lines = []
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        name = d.get("Metric Name", "")
        sec = d.get("Section Name", "")
        if any(k in name or k in sec or k in d.get("Metric Value", "")[:200] for k in KEYS):
            lines.append(f"{d.get('Kernel Name', '')[:40]} | {sec} | {name} | {d.get('Metric Unit', '')} | "
                         f"{d.get('Metric Value', '')[:400]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active",
            "sm__inst_executed_pipe_fp64", "smsp__inst_executed_pipe_fp64", "sm__throughput",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared", "sm__pipe_tensor", "smsp__average_warp",
            "gpu__time_duration.sum", "sm__warps_active"]
    if len(rr) >= 3:
        h, units, vals = rr[0], rr[1], rr[2:]
        kn = h.index("Kernel Name") if "Kernel Name" in h else None
        for v in vals:
            kname = v[kn][:60] if kn is not None and kn < len(v) else ""
            lines.append(f"# kernel: {kname}")
            for i, col in enumerate(h):
                if any(col.startswith(w) for w in want) and i < len(v):
                    lines.append(f"raw | {col} | {units[i]} | {v[i]}")
    with open(out, "w") as f:
        f.write(f"# {header}\n")
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    header = sys.argv[4] if len(sys.argv) > 4 else src
    (launches if mode == "launches" else full)(src, dst, header)
