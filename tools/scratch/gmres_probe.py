#!/usr/bin/env python
"""Matvec time vs GMRES time on the paper's RBF system (bench.py --mode gmres workload):
how much of T_G is matvecs and how much is the Arnoldi / host loop."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2204_05536_b200 as h2d  # noqa: E402
import workloads as W  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 500
kern = sys.argv[2] if len(sys.argv) > 2 else "rbf_phi1"
pts = W.chebyshev_grid(m)
n = pts.shape[0]
op = h2d.Hodlr2d.build(torch.from_numpy(pts).cuda(), kern, 500, 1e-12, c=1e-3, scale=1.0, shift=float(n),
                       box_lo=(-1, -1), box_side=2.0, depth=-2)
lam = torch.from_numpy(np.random.default_rng(1048).uniform(-1.0, 1.0, n)).cuda()
f = op.matvec(lam)
y = torch.empty_like(f)
for _ in range(3):
    op.matvec_raw(lam.data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    op.matvec_raw(lam.data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
e1.record()
torch.cuda.synchronize()
mv = e0.elapsed_time(e1) / 20
inf = op.info()
op.set_timing(True)
op.stage_times(reset=True)
for _ in range(10):
    op.matvec_raw(lam.data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
torch.cuda.synchronize()
st, cnt = op.stage_times(reset=True)
op.set_timing(False)
print("kappa", inf["kappa"], "near_pairs", inf["near_pairs"], "factor bytes", inf["stageA_bytes"] + inf["stageB_bytes"],
      "stages", {k: round(v / cnt, 4) for k, v in st.items()}, flush=True)
op.gmres(f, tol=1e-10)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.time()
    lam_hat, its, rr = op.gmres(f, tol=1e-10)
    torch.cuda.synchronize()
    tg = (time.time() - t0) * 1e3
    print(f"n {n} matvec {mv:.3f} ms  gmres {tg:.2f} ms  iterations {its}  -> {tg / max(its, 1):.2f} ms/iteration "
          f"(matvecs ~{(its + 2) * mv:.2f} ms)", flush=True)
