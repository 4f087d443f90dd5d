#!/usr/bin/env python
"""Summarise an ncu report (or a launch-list CSV) into the markdown kept under profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep  > profiles/rNN_ncu_full.md
    python tools/ncu_summary.py --launches gpurun_out/launches.csv > profiles/rNN_launches.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "time (ms)"),
    ("dram__bytes_read.sum", "DRAM read (GB)"),
    ("dram__bytes_write.sum", "DRAM write (MB)"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe % active"),
    ("smsp__inst_executed_pipe_fp64.sum", "FP64 warp-instr"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue % active"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary: `{path}`\n")
    print("| kernel | grid | " + " | ".join(n for _, n in METRICS) + " | top stalls |")
    print("|---" * (len(METRICS) + 3) + "|")
    for r in rows[2:]:
        name = short(r[hdr.index("Kernel Name")])
        vals = []
        for m, _ in METRICS:
            v = r[hdr.index(m)] if m in hdr else ""
            vals.append(v)
        st = []
        for h, v in zip(hdr, r):
            if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(v), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        st.sort(reverse=True)
        stalls = ", ".join(f"{n} {v:.1f}" for v, n in st[:3])
        print(f"| {name} | {r[hdr.index('Grid Size')]} | " + " | ".join(vals) + f" | {stalls} |")
    print("\nUnits as reported by ncu: " + ", ".join(f"{m}={units[hdr.index(m)]}" for m, _ in METRICS if m in hdr))


def short(n):
    """Kernel name without return type, namespaces or argument list (template args kept)."""
    n = n.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    depth, cut = 0, len(n)
    for i, ch in enumerate(n):
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif ch == "(" and depth == 0:
            cut = i
            break
    head = n[:cut].strip()
    parts, depth, cur = [], 0, ""
    for i, ch in enumerate(head):
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        if depth == 0 and head.startswith("::", i):
            parts.append(cur)
            cur = ""
            continue
        if depth == 0 and ch == ":" and i > 0 and head[i - 1] == ":":
            continue
        cur += ch
    parts.append(cur)
    last = parts[-1].strip()
    if last.startswith("void "):
        last = last[5:]
    return last.split(" ")[-1] if "<" not in last else last


MATVEC = ("stageA", "stageB", "p2p", "permute_in", "unpad", "combine")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    k, v = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        agg[short(r[k])].append(float(r[v]))
    tot = sum(sum(x) for x in agg.values())
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none): `{path}`\n")
    print("| kernel | launches | mean (us) | share of listed time |")
    print("|---|---|---|---|")
    for name, xs in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| {name} | {len(xs)} | {sum(xs) / len(xs) / 1e3:.1f} | {100 * sum(xs) / tot:.1f} % |")
    mv = {n: xs for n, xs in agg.items() if n.startswith(MATVEC)}
    mtot = sum(sum(x) for x in mv.values())
    if mtot:
        print("\nMatvec kernels only (one matvec = one launch of each; serialised, cold-cache):\n")
        print("| kernel | launches | mean (us) | share of the matvec |")
        print("|---|---|---|---|")
        for name, xs in sorted(mv.items(), key=lambda kv: -sum(kv[1])):
            print(f"| {name} | {len(xs)} | {sum(xs) / len(xs) / 1e3:.1f} | {100 * sum(xs) / mtot:.1f} % |")


STAGE_OF = {"stageA_tma_kernel": "stageA_VTx", "stageB_tma_kernel": "stageB_Ut",
            "p2p_fast_kernel": "p2p_near", "stageA_dual_kernel": "stageA_dual"}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def traffic(path, cfg, out):
    """Per-launch DRAM bytes (read + write) of the matvec kernels -> profiles/ncu_traffic.json."""
    import json
    import os
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    acc = defaultdict(list)
    for r in rows[2:]:
        name = short(r[hdr.index("Kernel Name")]).split("<")[0]
        if name in STAGE_OF:
            b = float(r[ir]) * SCALE[units[ir]] + float(r[iw]) * SCALE[units[iw]]
            acc[STAGE_OF[name]].append(b)
    data = json.load(open(out)) if os.path.exists(out) else {}
    data[cfg] = {k: int(sum(v) / len(v)) for k, v in acc.items()}
    data[cfg]["source"] = os.path.basename(path)
    with open(out, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)
    print(json.dumps(data[cfg]))


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "--traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        full(sys.argv[1])
