"""Adaptive symmetric matvec on the Chebyshev RBF system: per-stage times (one-off probe).

python tools/scratch/adsym_probe.py --m 1000 [--directed] [--reps 20]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_2204_05536_b200 as h2d  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=1000)
ap.add_argument("--directed", action="store_true")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--nmax", type=int, default=64)
ap.add_argument("--kernel", default="rbf_phi1")
ap.add_argument("--balanced", action="store_true", help="the paper depth rule (depth = -2) instead of adaptive")
args = ap.parse_args()
torch.cuda.set_device(0)
pts = W.chebyshev_grid(args.m)
n = pts.shape[0]
t0 = time.time()
op = h2d.Hodlr2d.build(torch.from_numpy(pts).cuda(), args.kernel, args.nmax, 1e-12, c=1e-3, scale=1.0,
                       shift=float(n), box_lo=(-1, -1), box_side=2.0, depth=-2 if args.balanced else -3, symmetric=not args.directed)
torch.cuda.synchronize()
t_b = time.time() - t0
inf = op.info()
x = torch.from_numpy(np.random.default_rng(7).uniform(-1.0, 1.0, n)).cuda()
y = torch.empty_like(x)
for _ in range(3):
    op.matvec_raw(x.data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.reps):
    op.matvec_raw(x.data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
e1.record()
torch.cuda.synchronize()
mv = e0.elapsed_time(e1) / args.reps
op.set_timing(True)
op.stage_times(reset=True)
for _ in range(5):
    op.matvec_raw(x.data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
st, cnt = op.stage_times(reset=True)
op.set_timing(False)
print(json.dumps({"m": args.m, "balanced": args.balanced, "nmax": args.nmax, "symmetric": not args.directed, "build_s": round(t_b, 3), "matvec_ms": round(mv, 4),
                  "stage_ms": {k: round(v / max(cnt, 1), 4) for k, v in st.items()},
                  "matvec_gb": inf["matvec_bytes"] / 1e9, "small_items": inf["small_items"],
                  "kappa": inf["kappa"], "n_leaves": inf["n_leaves"],
                  "gbs": round(inf["matvec_bytes"] / mv / 1e6, 1)}), flush=True)
