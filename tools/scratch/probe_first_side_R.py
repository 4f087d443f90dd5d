#!/usr/bin/env python
"""Widest first-side panel (sum of ranks of the blocks (X, Y), Y > X, of one box X) of a few
symmetric builds: picks parameters that drive stage B' onto its wide (R > 256) path."""
import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2204_05536_b200 as h2d, workloads as W
def firstR(op):
    best = 0
    for l in range(1, op.info()["kappa"] + 1):
        off, col = op.lists(l); r = op.ranks(l)
        for X in range(len(off) - 1):
            s = sum(max(0, r[e]) for e in range(off[X], off[X + 1]) if col[e] > X)
            best = max(best, s)
    return best
for (n, kern, leaf, tol, kw) in [(1 << 14, "test_lowrank", 64, 1e-10, dict(test_rank=60, shift=0.5)),
                                 (1 << 14, "imq", 256, 1e-13, dict(c=0.05)),
                                 (1 << 14, "log", 256, 1e-14, {}),
                                 (1 << 15, "imq", 512, 1e-13, dict(c=0.02)),
                                 (1 << 14, "one_over_r", 256, 1e-13, {})]:
    pts = W.uniform_points(n, 4343)
    op = h2d.Hodlr2d.build(torch.from_numpy(pts).cuda(), kern, leaf, tol, box_lo=(-1, -1), box_side=2.0, symmetric=True, **kw)
    print(n, kern, leaf, tol, kw, "rank_max", op.info()["rank_max"], "first-side R max", firstR(op), flush=True)
