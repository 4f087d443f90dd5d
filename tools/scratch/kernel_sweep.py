#!/usr/bin/env python
"""Every kernel family once at small sizes with self-checks (compute-sanitizer is not
available on the GPU pool): directed and symmetric builds, single and multi-RHS
(16 + 2 + 1 / 8 + 8 + 3 vectors), GMRES, clustered Chebyshev input (warp P2P, small-item
kernels), host pointers (bitwise equal to device pointers), multi-RHS columns equal to
single matvecs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2204_05536_b200 as h2d  # noqa: E402
import workloads as W  # noqa: E402

os.environ["H2D_SMALL_MIN"] = "1"
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
cases = [(W.uniform_points(3000, 1), "log", 64, 1e-8, {}),
         (W.chebyshev_grid(60), "rbf_phi1", 100, 1e-10, dict(c=1e-3, shift=3600.0, depth=-2)),
         (W.uniform_points(2000, 2), "imq", 32, 1e-9, dict(c=0.2))]
for pts, kernel, leaf, tol, kw in cases:
    for sym in (False, True):
        op = h2d.Hodlr2d.build(dev(pts), kernel, leaf, tol, box_lo=(-1, -1), box_side=2.0, symmetric=sym, **kw)
        n = pts.shape[0]
        x = W.random_vector(n, 3)
        y = op.matvec(dev(x)).cpu().numpy()
        yh = op.matvec(x.copy())
        assert np.array_equal(y, yh)
        X = np.stack([W.random_vector(n, 10 + k) for k in range(19)])   # 16 + 2 + 1 / 8 + 8 + 3
        Y = op.matvec_multi(dev(X)).cpu().numpy()
        for k in (0, 15, 16, 18):
            yk = op.matvec(dev(X[k])).cpu().numpy()
            assert np.linalg.norm(Y[k] - yk) <= 1e-13 * np.linalg.norm(yk), k
        if kernel == "rbf_phi1":
            xs, its, rr = op.gmres(dev(y), tol=1e-10)
        op.close()
        torch.cuda.synchronize()
        print("ok", kernel, "symmetric" if sym else "directed", flush=True)
