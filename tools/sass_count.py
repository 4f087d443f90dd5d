"""Count SASS instruction classes of the kernels whose mangled name matches a pattern
(libhodlr2d.so), e.g. python tools/sass_count.py p2p_warp_kernelILi0ELi2"""
import collections
import re
import subprocess
import sys

lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2204_05536_b200/libhodlr2d.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, counts = None, {}
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1) if sys.argv[1] in m.group(1) else None
        if cur:
            counts[cur] = collections.Counter()
        continue
    if cur:
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m:
            counts[cur][m.group(2).split(".")[0]] += 1
for f, c in counts.items():
    fp64 = sum(v for k, v in c.items() if k in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX", "DSEL"))
    print(f[-60:], "total", sum(c.values()), "fp64", fp64, dict(c.most_common(14)))
