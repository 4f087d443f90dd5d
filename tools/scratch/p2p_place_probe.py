"""Near-field placement probe: matvec time and stage times with the near field beside stage A
(set_diag p2p_place 0), beside stage B (p2p_place 1), timed (auto, -1) and alone before stage A (p2p_serial), on
the configs in CFGS (CUDA events; results compared with the default placement)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2204_05536_b200 as h2d  # noqa: E402
import workloads as W  # noqa: E402

steps = int(os.environ.get("STEPS", "20"))
for name in os.environ.get("CFGS", "c3,c4").split(","):
    cfg = W.CONFIGS[name]
    pts = torch.from_numpy(W.config_points(cfg)).cuda()
    s = torch.cuda.current_stream()
    op = h2d.Hodlr2d.build(pts, cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale, shift=cfg.shift,
                           box_lo=cfg.box_lo, box_side=cfg.box_side, stream=s.cuda_stream)
    del pts
    xs = [torch.from_numpy(W.config_x(cfg, k)).cuda() for k in range(4)]
    y = torch.empty(cfg.n, dtype=torch.float64, device="cuda")
    ref = None
    modes = os.environ.get("MODES", "default,p2p_beside_b,p2p_serial,default").split(",")
    for mode in modes * int(os.environ.get("REPS", "1")):
        op.set_diag("p2p_serial", 1 if mode == "p2p_serial" else 0)
        op.set_diag("p2p_place", {"p2p_beside_b": 1, "auto": -1}.get(mode, 0))
        for k in range(4):
            op.matvec_raw(xs[k % 4].data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
        torch.cuda.synchronize()
        if ref is None:
            ref = y.clone()
        op.matvec_raw(xs[3].data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
        diff = float((y - ref).norm() / ref.norm())
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
        per = " ".join(f"{k}={v / max(cnt, 1):.3f}" for k, v in st.items())
        print(f"{name} {mode:13s} {ms:.3f} ms/matvec ({1e3 / ms:.1f}/s)  diff {diff:.1e}  {per}", flush=True)
    del op
    torch.cuda.empty_cache()
