"""Multi-RHS probe: C3 operator, hodlr2d_matvec_multi at K vectors per call (CUDA events).
Run alone for the rate; under ncu --metrics gpu__time_duration.sum for per-kernel times."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2204_05536_b200 as h2d  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.CONFIGS[os.environ.get("CFG", "c3")]
K = int(os.environ.get("K", "16"))
calls = int(os.environ.get("CALLS", "10"))
pts = torch.from_numpy(W.config_points(cfg)).cuda()
op = h2d.Hodlr2d.build(pts, cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale, shift=cfg.shift,
                       box_lo=cfg.box_lo, box_side=cfg.box_side,
                       symmetric=os.environ.get("SYM", "0") == "1")
if "NF" in os.environ:
    op.set_diag("multi_stored_near", int(os.environ["NF"]))
if "MT" in os.environ:
    op.set_diag("multi_log_table", int(os.environ["MT"]))
X = torch.rand(K, cfg.n, dtype=torch.float64, device="cuda") * 2 - 1
Y = torch.empty_like(X)
s = torch.cuda.current_stream()
for _ in range(2):
    op.matvec_multi_raw(X.data_ptr(), Y.data_ptr(), K, h2d.ORDER_ORIGINAL)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(calls):
    op.matvec_multi_raw(X.data_ptr(), Y.data_ptr(), K, h2d.ORDER_ORIGINAL)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / calls
print(f"multi K={K} {cfg.name if hasattr(cfg, 'name') else ''}: {ms:.3f} ms per call, {1e3 * K / ms:.1f} matvecs/s")
if os.environ.get("CHECK", "1") == "1":
    y0 = op.matvec(X[0].contiguous())
    yk = op.matvec(X[K - 1].contiguous())
    e = max(float((Y[0] - y0).norm() / y0.norm()), float((Y[K - 1] - yk).norm() / yk.norm()))
    print(f"multi vs single-vector rel-l2 {e:.3e}")
