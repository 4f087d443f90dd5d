#!/usr/bin/env python
"""Where the e2e (host-pointer) matvec time goes: device pointers vs host x / host y / both."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2204_05536_b200 as h2d  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.CONFIGS["c3"]
op = h2d.Hodlr2d.build(torch.from_numpy(W.config_points(cfg)).cuda(), cfg.kernel, cfg.leaf_size, cfg.tol,
                       box_lo=cfg.box_lo, box_side=cfg.box_side)
xd = torch.from_numpy(W.config_x(cfg, 0)).cuda()
yd = torch.empty_like(xd)
xh = xd.cpu().pin_memory()
yh = torch.empty(cfg.n, dtype=torch.float64).pin_memory()
xp = xd.cpu()            # pageable
yp = torch.empty(cfg.n, dtype=torch.float64)
cases = {"device x, device y": (xd, yd), "pinned x, device y": (xh, yd), "device x, pinned y": (xd, yh),
         "pinned x, pinned y": (xh, yh), "pageable x, pageable y": (xp, yp)}
for name, (x, y) in cases.items():
    for _ in range(3):
        op.matvec_raw(x.data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(30):
        op.matvec_raw(x.data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
    torch.cuda.synchronize()
    print("%-24s %.3f ms per call" % (name, (time.perf_counter() - t0) / 30 * 1e3))
