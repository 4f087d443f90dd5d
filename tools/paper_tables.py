#!/usr/bin/env python
"""The paper's HODLR2D table columns on the GPU build: Tables tab:1byr_init / tab:1byr_mat
(1/r: r_m, memory, eps_r), tab:ker1_init (phi_1: r_m, CR), tab:ker2_init (phi_2: r_m, CR),
rows N = 100^2 ... 500^2 Chebyshev grids, N_max 500 with the paper's depth rule, ACA 1e-12.
eps_r = max_i |b_hat - b|_i / |b|_i over sampled rows (exact rows from the CPU
oracle) for two input vectors psi ~ U(0,1) (R17).  --max-rank=R raises the ACA rank cap.
Prints one JSON line per (kernel, N)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2204_05536_b200 as h2d  # noqa: E402
import workloads as W  # noqa: E402

KID = {"one_over_r": 2, "rbf_phi1": 3, "rbf_phi2": 4}
args = [a for a in sys.argv[1:] if not a.startswith("--")]
max_rank = int(next((a.split("=")[1] for a in sys.argv[1:] if a.startswith("--max-rank=")), "128"))
ms = [int(a) for a in args] or [100, 150, 200, 250, 300, 400, 500]
for kernel in ("one_over_r", "rbf_phi1", "rbf_phi2"):
    for m in ms:
        pts = W.chebyshev_grid(m)
        n = pts.shape[0]
        kw = dict(c=1e-3, shift=float(n)) if kernel != "one_over_r" else {}
        op = h2d.Hodlr2d.build(torch.from_numpy(pts).cuda(), kernel, 500, 1e-12, box_lo=(-1, -1), box_side=2.0,
                               depth=-2, max_rank=max_rank, **kw)
        inf = op.info()
        line = {"kernel": kernel, "N": n, "kappa": inf["kappa"], "r_m": inf["rank_max"],
                "cr": inf["compression_ratio"], "memory_gb": inf["compression_ratio"] * n * n * 8 / 1e9,
                "truncated": inf["truncated"]}
        if kernel == "one_over_r":
            rows = np.random.default_rng(m).choice(n, size=min(n, 256), replace=False)
            eps = 0.0
            for k in range(2):
                x = np.random.default_rng(1000 + k).uniform(0.0, 1.0, n)   # psi ~ U(0,1) (R17)
                y = op.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
                b = oracle.dense_rows(pts, x, rows, KID[kernel])
                eps = max(eps, float(np.max(np.abs(y[rows] - b) / np.abs(b))))
            line["eps_r_sampled"] = eps
        # matvec time (CUDA events, device pointers) and, for the RBF systems, the GMRES solve
        # time T_G to residual 1e-10 (median of 3) — the paper's single-core times are context
        x = torch.from_numpy(np.random.default_rng(7).uniform(0.0, 1.0, n)).cuda()
        y = torch.empty_like(x)
        for _ in range(3):
            op.matvec_raw(x.data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            op.matvec_raw(x.data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
        e1.record()
        torch.cuda.synchronize()
        line["matvec_s"] = e0.elapsed_time(e1) / 20 / 1e3
        if kernel != "one_over_r":
            f = op.matvec(x)
            op.gmres(f, tol=1e-10)
            tg = []
            for _ in range(3):
                torch.cuda.synchronize()
                t0 = time.time()
                _, its, rr = op.gmres(f, tol=1e-10)
                torch.cuda.synchronize()
                tg.append(time.time() - t0)
            line["T_G_s"] = float(np.median(tg))
            line["gmres_iterations"] = its
        print(json.dumps(line), flush=True)
        op.close()
