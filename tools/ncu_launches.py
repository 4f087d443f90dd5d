#!/usr/bin/env python
"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv`)
as a markdown table: launches, mean duration and share of the listed time per kernel.

    python tools/ncu_launches.py gpurun_out/launches.csv ["kernel-name regex"] > profiles/rNN_launches.md
"""
import csv
import re
import sys
from collections import OrderedDict


def short(name: str) -> str:
    name = name.removeprefix("void ")
    for pre in ("(anonymous namespace)::", "<unnamed>::", "unnamed>::", "h2d::"):
        name = name.replace(pre, "")
    if name.endswith(")"):   # cut the argument list: the '(' matching the final ')'
        depth = 0
        for i in range(len(name) - 1, -1, -1):
            depth += name[i] == ")"
            depth -= name[i] == "("
            if depth == 0:
                return name[:i]
    return name


def main(path: str, keep: str = "") -> None:
    with open(path) as f:
        lines = f.readlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    tot = OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
        k = short(r["Kernel Name"])
        if keep and not re.search(keep, k):
            continue
        n, t = tot.get(k, (0, 0.0))
        tot[k] = (n + 1, t + float(r["Metric Value"].replace(",", "")) * scale)
    all_t = sum(t for _, t in tot.values())
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none): `{path}`"
          + (f", kernels matching `{keep}`" if keep else "") + "\n")
    print("Serialised, cold-cache per-launch times: compare SHARES with the bench's live stage times.\n")
    print("| kernel | launches | mean (us) | share of listed time |")
    print("|---|---|---|---|")
    for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {n} | {t / n:.1f} | {100 * t / all_t:.1f} % |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
