#!/usr/bin/env python
"""Build C3 and run hodlr2d_matvec_multi (nrhs vectors) a few times: a target for ncu.

    ncu --metrics gpu__time_duration.sum -k regex:multi python tools/multi_probe.py 8 [c3 [sym]]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2204_05536_b200 as h2d  # noqa: E402
import workloads as W  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = W.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c3"]
sym = len(sys.argv) > 3 and sys.argv[3] == "sym"
pts = W.config_points(cfg)
op = h2d.Hodlr2d.build(torch.from_numpy(pts).cuda(), cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c,
                       scale=cfg.scale, shift=cfg.shift, box_lo=cfg.box_lo, box_side=cfg.box_side, symmetric=sym)
X = torch.from_numpy(np.stack([W.config_x(cfg, k) for k in range(K)])).cuda()
Y = torch.empty_like(X)
for _ in range(3):
    op.matvec_multi_raw(X.data_ptr(), Y.data_ptr(), K, h2d.ORDER_ORIGINAL)
torch.cuda.synchronize()
print("ok")
