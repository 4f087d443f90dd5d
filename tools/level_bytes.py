import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np, torch, paper_2204_05536_b200 as h2d, workloads as W
for name in ("c3", "c5s"):
    if name == "c3":
        cfg = W.CONFIGS["c3"]; pts = W.config_points(cfg); kw = {}
    else:
        cfg = W.CONFIGS["c5"]; pts = W.config_points(cfg); kw = dict(world=8, rank=0)
    op = h2d.Hodlr2d.build(torch.from_numpy(pts).cuda(), cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale,
                           shift=cfg.shift, box_lo=cfg.box_lo, box_side=cfg.box_side, **kw)
    inf = op.info(); perm, ls = op.tree(); kappa = inf["kappa"]
    tot = 0; rows = []
    for l in range(1, kappa + 1):
        r = op.ranks(l); off, col = op.lists(l)
        sh = 2 * (kappa - l)
        bsz = ls[(np.arange(1 << (2 * l)) + 1) << sh] - ls[np.arange(1 << (2 * l)) << sh]
        X = np.repeat(np.arange(1 << (2 * l)), np.diff(off))
        m = bsz[X]; n = bsz[col]; rr = np.maximum(r, 0)
        b = float((rr * (m + n)).sum()) * 8
        # smem for the pair {X, Y} (both directions' factors once): r (m + n) * 8 bytes
        pair = rr * (m + n) * 8
        rows.append((l, b / 1e9, float(np.median(pair[rr > 0]) / 1e3) if (rr > 0).any() else 0, float(rr.mean())))
        tot += b
    print(name, "total GB", tot / 1e9)
    for l, gb, kb, rm in rows: print(f"  level {l}: {gb:6.2f} GB ({100*gb*1e9/tot:4.1f} %), median pair factors {kb:9.1f} KB, mean rank {rm:5.1f}")
