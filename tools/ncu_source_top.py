#!/usr/bin/env python
"""Top SASS lines of one kernel in an ncu report, by instructions executed and by stall samples.

    python tools/ncu_source_top.py gpurun_out/prof.ncu-rep stageA_tma [N]
"""
import csv
import io
import subprocess
import sys


def num(x):
    try:
        return int(float(x))
    except ValueError:
        return 0


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    i_s, i_e, i_w = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    i_x = hdr.index("L1 Wavefronts Shared Excessive") if "L1 Wavefronts Shared Excessive" in hdr else None
    data = [(r[i_s].strip(), num(r[i_e]), num(r[i_w])) for r in rows[2:] if len(r) > i_e and r[0] != "Address"]
    if i_x is not None:
        ex = [(r[i_s].strip(), num(r[i_x])) for r in rows[2:] if len(r) > i_x and r[0] != "Address"]
        tx = sum(e for _, e in ex) or 1
        print(f"-- by excessive shared wavefronts (bank conflicts), total {tx}")
        for src, e in sorted(ex, key=lambda d: -d[1])[:10]:
            print(f"{e:>11} {100 * e / tx:5.1f}%  {src[:80]}")
    tot = sum(d[1] for d in data) or 1
    totw = sum(d[2] for d in data) or 1
    print(f"{kern}: {tot} warp-instructions executed, {totw} stall samples")
    print("-- by instructions executed")
    for s, e, w in sorted(data, key=lambda d: -d[1])[:n]:
        print(f"{e:>11} {100 * e / tot:5.1f}%  samples {100 * w / totw:5.1f}%  {s[:80]}")
    print("-- by stall samples")
    for s, e, w in sorted(data, key=lambda d: -d[2])[:n]:
        print(f"{e:>11} {100 * e / tot:5.1f}%  samples {100 * w / totw:5.1f}%  {s[:80]}")


if __name__ == "__main__":
    main()
