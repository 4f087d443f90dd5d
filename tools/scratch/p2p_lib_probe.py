"""P2P variant probe: the library named by H2D_LIBRARY (or the in-tree one) on the configs in
CFGS: matvec ms (near field beside stage A), near-field ms alone (p2p_serial) and beside the
streams; y of x0 saved to OUT_<cfg>.npy for a cross-library comparison."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2204_05536_b200 as h2d  # noqa: E402
import workloads as W  # noqa: E402

steps = int(os.environ.get("STEPS", "30"))
tag = os.environ.get("TAG", "lib")
for name in os.environ.get("CFGS", "c3").split(","):
    cfg = W.CONFIGS[name]
    pts = torch.from_numpy(W.config_points(cfg)).cuda()
    s = torch.cuda.current_stream()
    op = h2d.Hodlr2d.build(pts, cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale, shift=cfg.shift,
                           box_lo=cfg.box_lo, box_side=cfg.box_side, stream=s.cuda_stream)
    del pts
    xs = [torch.from_numpy(W.config_x(cfg, k)).cuda() for k in range(4)]
    y = torch.empty(cfg.n, dtype=torch.float64, device="cuda")
    op.matvec_raw(xs[0].data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
    torch.cuda.synchronize()
    np.save(f"/tmp/{tag}_{name}.npy", y.cpu().numpy())
    for serial in (0, 1, 0, 1):
        op.set_diag("p2p_serial", serial)
        for k in range(4):
            op.matvec_raw(xs[k].data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for k in range(steps):
            op.matvec_raw(xs[k % 4].data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        op.set_timing(True)
        op.stage_times(reset=True)
        for k in range(steps):
            op.matvec_raw(xs[k % 4].data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
        torch.cuda.synchronize()
        st, cnt = op.stage_times(reset=True)
        op.set_timing(False)
        print(f"{tag} {name} serial={serial} {ms:.3f} ms/matvec  p2p_near={st['p2p_near'] / cnt:.4f}  "
              f"A={st['stageA_VTx'] / cnt:.3f} B={st['stageB_Ut'] / cnt:.3f}", flush=True)
    del op
    torch.cuda.empty_cache()
