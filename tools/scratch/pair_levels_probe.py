# Runs one matvec of the pair apply restricted to levels lo..hi (H2D_PAIR_LEVELS); prints ok / the error.
import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2204_05536_b200 as h2d
import workloads as W
cfg = W.CONFIGS[sys.argv[1]]
pts = W.config_points(cfg)
op = h2d.Hodlr2d.build(torch.from_numpy(pts).cuda(), cfg.kernel_name if hasattr(cfg, "kernel_name") else cfg.kernel,
                       cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale, shift=cfg.shift, box_lo=cfg.box_lo,
                       box_side=cfg.box_side, symmetric=True)
x = torch.from_numpy(W.config_x(cfg, 0)).cuda()
try:
    y = op.matvec(x)
    torch.cuda.synchronize()
    print(os.environ.get("H2D_PAIR_LEVELS"), "ok", float(y.norm()))
except Exception as e:
    print(os.environ.get("H2D_PAIR_LEVELS"), "ERR", str(e)[:100])
