"""Adaptive Chebyshev phi_1 matvec (N_max 64, tol 1e-12) with the list near field's 512-bin /
replicated log table (H2D_P2P_TABLE) / timed pick: ms per matvec (CUDA events), stage times."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2204_05536_b200 as h2d  # noqa: E402
import workloads as W  # noqa: E402

m = int(os.environ.get("M", "1000"))
pts = torch.from_numpy(W.chebyshev_grid(m)).cuda()
x = torch.rand(m * m, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for sym in (False, True):
    for t in ("0", "1", None, "0", "1"):
        if t is None:
            os.environ.pop("H2D_P2P_TABLE", None)
        else:
            os.environ["H2D_P2P_TABLE"] = t
        op = h2d.Hodlr2d.build(pts, "rbf_phi1", 64, 1e-12, c=1e-3, shift=float(m * m), box_lo=(-1, -1),
                               box_side=2.0, depth=-3, symmetric=sym)
        s = torch.cuda.current_stream()
        for _ in range(3):
            op.matvec_raw(x.data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(20):
            op.matvec_raw(x.data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
        e1.record(s)
        torch.cuda.synchronize()
        op.set_timing(True)
        op.stage_times(reset=True)
        for _ in range(10):
            op.matvec_raw(x.data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
        torch.cuda.synchronize()
        st, cnt = op.stage_times(reset=True)
        print(f"{m}^2 sym={int(sym)} table={t} picked={op.info()['p2p_log_table']} "
              f"{e0.elapsed_time(e1) / 20:.3f} ms  " + " ".join(f"{k}={v / cnt:.3f}" for k, v in st.items()), flush=True)
        op.close()
        del op
        torch.cuda.empty_cache()
