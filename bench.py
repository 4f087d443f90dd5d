#!/usr/bin/env python
"""HODLR2D fp64 matvec benchmark (BASELINE.json metric: matvecs/sec at N = 2^20..2^24).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

One step = one HODLR2D matvec (Alg. 2: every row of SURVEY §8(a) S7-S10 on
the hot path) of a fresh seeded x over the config's N points; the operator is built once
before timing (build seconds reported separately).  N = 1: the whole matvec on one GPU.
N > 1 (torchrun): contiguous Morton row ranges per rank, one NCCL all-gather of x per
matvec, max over ranks; total work is fixed -> "scaling": "strong".

Rank 0 prints ONE JSON line.  --impl reference times the CPU oracle (oracle/) on the same
workload (the full operator where it fits in host RAM; this tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(W.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c4", action="store_true",
                    help="skip the C4 (N = 2^22) sub-result the default C3 line carries")
    ap.add_argument("--c5-min-world", type=int, default=4,
                    help="at --gpus >= this, the C3 line also carries the C5 multi-GPU sub-result "
                         "(build + 50 matvecs, max over ranks, E_N from per-rank slice timings)")
    ap.add_argument("--c5-config", default="c5", choices=sorted(W.CONFIGS),
                    help="config of that sub-result (c2: functional check on one shared GPU)")
    ap.add_argument("--symmetric", action="store_true",
                    help="symmetric build + apply (one ACA per unordered pair, DESIGN.md R23)")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the symmetric-storage (NEXT N1) variant measured beside the headline")
    ap.add_argument("--multi-rhs", type=int, default=16,
                    help="also time hodlr2d_matvec_multi with this many vectors per call (0: skip)")
    ap.add_argument("--rank-slice", type=int, default=None,
                    help="informational: build and time rank G's slice of a --slice-world partition "
                         "on this one GPU, full x resident (per-GPU compute of the multi-GPU run)")
    ap.add_argument("--slice-world", type=int, default=8)
    ap.add_argument("--leaf-weights", default=None,
                    help="rank-slice mode: .npy of per-leaf loads for the partition (hodlr2d_leaf_costs "
                         "summed over the slices of a first run)")
    ap.add_argument("--dump-leaf-costs", default=None,
                    help="rank-slice mode: save this slice's hodlr2d_leaf_costs to this .npy")
    ap.add_argument("--mode", default="matvec", choices=["matvec", "gmres"],
                    help="gmres: the paper's RBF application (P:1020-1048) at --grid-m^2 Chebyshev "
                         "points, informational line with T_I / T_G (paper values as context)")
    ap.add_argument("--grid-m", type=int, default=500)
    ap.add_argument("--rbf-kernel", default="rbf_phi1", choices=["rbf_phi1", "rbf_phi2"])
    ap.add_argument("--nmax", type=int, default=500, help="gmres mode: N_max (the paper's 500, P:921)")
    ap.add_argument("--adaptive", action="store_true",
                    help="gmres mode: the adaptive quadtree (depth = -3, DESIGN.md R24) instead of the "
                         "balanced tree at the paper's depth rule (R22)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: functional check of the multi-rank path (host-staged gather)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.p = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        busy = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- oracle arm

# Host RAM the oracle needs for a config (factors + dense leaf blocks + tree; survey census,
# SURVEY §8(d)): the full operator is built when it fits in 60 % of the host's RAM.
ORACLE_GB = {"c1": 0.05, "c2": 2.5, "c3": 24.0, "c4": 112.0, "c5": 420.0}


def host_info():
    """nproc, CPU model and RAM of the host the oracle runs on."""
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 1e9
    except (ValueError, OSError):
        ram = 0.0
    return {"nproc": os.cpu_count(), "cpu_model": model, "ram_gb": round(ram, 1)}


def oracle_operator(cfg, name):
    """The oracle as it stands: the FULL operator when it fits in host RAM (C1-C3 here), else
    the rows of Morton box 0 at level 2 (1/16 of the rows; C4 / C5), whose matvec time is
    extrapolated by the row fraction and labelled so."""
    import oracle
    pts = W.config_points(cfg)
    kw = dict(c=cfg.c, scale=cfg.scale, shift=cfg.shift, box_lo=cfg.box_lo, box_side=cfg.box_side)
    if ORACLE_GB[name] <= 0.6 * host_info()["ram_gb"]:
        t0 = time.time()
        op = oracle.Operator(pts, cfg.kernel, cfg.leaf_size, cfg.tol, **kw)
        return op, 1.0, time.time() - t0, (f"the full oracle operator (C++ -O2 -ffp-contract=off, OpenMP; "
                                           f"Alg. 1 build + Alg. 2 matvec) on all {cfg.n} points, no extrapolation")
    kappa = oracle.depth(cfg.n, cfg.leaf_size)
    lvl = min(2, kappa)
    _, _, ls = oracle.tree(pts, cfg.box_lo, cfg.box_side, kappa)
    rows = int(ls[1 << (2 * (kappa - lvl))])
    t0 = time.time()
    op = oracle.Operator(pts, cfg.kernel, cfg.leaf_size, cfg.tol, row_range=(0, rows), **kw)
    build_s = time.time() - t0
    frac = rows / cfg.n
    desc = (f"EXTRAPOLATED: the full operator needs ~{ORACLE_GB[name]:.0f} GB of host RAM; oracle restricted "
            f"to TREE rows [0, {rows}) = Morton box 0 of level {lvl} ({frac:.4f} of the rows), matvec time "
            f"x{1 / frac:.1f} (its V^T x work at levels < {lvl} is whole-block, so this overstates the "
            f"oracle's time slightly)")
    return op, frac, build_s, desc


def time_oracle(op, cfg, frac, steps, warmup):
    """Mean wall time of `steps` oracle matvecs (fresh seeded x each) after `warmup`."""
    xs = [W.config_x(cfg, k) for k in range(min(steps + warmup, 4))]
    for k in range(warmup):
        op.matvec(xs[k % len(xs)])
    ts = []
    for k in range(steps):
        t0 = time.perf_counter()
        op.matvec(xs[k % len(xs)])
        ts.append(time.perf_counter() - t0)
    t_full = statistics.mean(ts) / frac
    return 1.0 / t_full, t_full


def cpu_baseline(cfg, name):
    """The oracle timed on the host cores in the same run: build once, then
    the mean of 10 matvecs after one warm-up on all cores, and of 2 on 1 thread."""
    import oracle
    op, frac, build_s, desc = oracle_operator(cfg, name)
    cores = oracle.max_threads()
    value, t_all = time_oracle(op, cfg, frac, 10, 1)
    oracle.set_threads(1)
    try:
        value1, t_one = time_oracle(op, cfg, frac, 2, 0)
    finally:
        oracle.set_threads(cores)
    op.close()
    return {"value": value, "unit": "matvecs/s", "cores": cores, "kind": "oracle",
            "sample": desc + "; mean of 10 matvecs after 1 warm-up (all cores) and of 2 (1 thread)",
            "extrapolated": frac < 1.0, "ms_per_matvec": round(t_all * 1e3, 2),
            "value_1thread": value1, "ms_per_matvec_1thread": round(t_one * 1e3, 1),
            "build_seconds": round(build_s, 2), "host": host_info()}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    op, frac, build_s, desc = oracle_operator(cfg, args.config)
    value, t_full = time_oracle(op, cfg, frac, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": "HODLR2D fp64 matvecs/sec", "value": value,
        "unit": "matvecs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_full * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, args.gpus),
        "cpu_baseline": {"value": value, "unit": "matvecs/s", "cores": oracle.max_threads(),
                         "kind": "oracle", "sample": desc + f"; build {build_s:.1f} s untimed",
                         "extrapolated": frac < 1.0, "host": host_info()},
        "e2e": {"value": value, "unit": "matvecs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(cfg, ngpu):
    kname = {0: "log", 1: "imq", 2: "one_over_r"}[cfg.kernel]
    return {"workload": f"{cfg.name}: N={cfg.n} {cfg.points} points, kernel {kname}"
                        + (f" c={cfg.c}" if cfg.kernel == 1 else "")
                        + (f", A = {cfg.shift:g} I + {cfg.scale:g} K" if cfg.shift or cfg.scale != 1 else "")
                        + f", leaf {cfg.leaf_size}, ACA tol {cfg.tol:g}, fresh x per matvec",
            "n_points": cfg.n, "leaf_size": cfg.leaf_size, "aca_tol": cfg.tol,
            "parallelism": f"morton-rows{ngpu}" if ngpu > 1 else "single",
            "l2": "factor stream (>= 20 GB) far exceeds the 126 MB L2; no flush needed"}


# ---------------------------------------------------------------------------- GPU arm

def run_ours(args, cfg):
    import torch
    import paper_2204_05536_b200 as h2d

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    stream = torch.cuda.current_stream()
    pts = W.config_points(cfg)
    d_pts = torch.from_numpy(pts).cuda()
    t0 = time.time()
    # N > 1: the handle owns the S11 communicator (an NCCL communicator whose unique id is
    # broadcast over the torch.distributed group; gloo: host-staged gather) and each matvec
    # takes only the rank's slice of x (H2D_ORDER_LOCAL): no torch collective in the loop
    op = h2d.Hodlr2d.build(d_pts, cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale,
                           shift=cfg.shift, box_lo=cfg.box_lo, box_side=cfg.box_side,
                           stream=stream.cuda_stream, symmetric=args.symmetric,
                           **({"group": dist.group.WORLD} if dist else {}))
    torch.cuda.synchronize()
    build_s = time.time() - t0
    del d_pts
    inf = op.info()
    nx = min(args.steps + args.warmup, 100)
    # fresh x per matvec, generated on the host (seeded) and resident in HBM before timing
    if world == 1:
        xs = torch.stack([torch.from_numpy(W.config_x(cfg, k)) for k in range(nx)]).cuda()
        y = torch.empty(cfg.n, dtype=torch.float64, device="cuda")

        def step(k):
            op.matvec_raw(xs[k % nx].data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
    else:
        perm, _ = op.tree()
        rb, re_ = inf["row_begin"], inf["row_end"]
        assert inf["comm_kind"] == (1 if args.dist_backend == "nccl" else 2), inf["comm_kind"]
        # each rank owns x_tree[rb:re] and passes only that slice; the library gathers it
        xs = torch.stack([torch.from_numpy(W.config_x(cfg, k)[perm][rb:re_].copy()) for k in range(nx)]).cuda()
        y = torch.empty(re_ - rb, dtype=torch.float64, device="cuda")

        def step(k):
            op.matvec_raw(xs[k % nx].data_ptr(), y.data_ptr(), h2d.ORDER_LOCAL)

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    op.stage_times(reset=True)
    op.set_timing(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ev0.record(stream)
        for k in range(args.steps):
            step(args.warmup + k)
        ev1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    op.set_timing(False)
    ms = ev0.elapsed_time(ev1)
    stages, cnt = op.stage_times(reset=True)
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda" if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = 1e3 / ms_step  # whole-job matvecs/s (each matvec covers all N rows)

    # roofline: dominant kernel, algorithmic bytes / its CUDA-event duration on this stream
    peak, peak_kind = peaks()
    per = {k: v / max(cnt, 1) for k, v in stages.items()}
    a_ms, b_ms = per["stageA_VTx"], per["stageB_Ut"]
    if b_ms >= a_ms:
        dom, dom_ms, dom_bytes = "stageB_Ut", b_ms, inf["stageB_bytes"]
    else:
        dom, dom_ms, dom_bytes = "stageA_VTx", a_ms, inf["stageA_bytes"]
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    other = "stageA_VTx" if dom == "stageB_Ut" else "stageB_Ut"
    other_bytes = inf["stageA_bytes"] if dom == "stageB_Ut" else inf["stageB_bytes"]
    clk_mhz = None
    other_ms = per[other]
    dom_traffic = ncu_traffic(args.config, dom)
    if inf.get("symmetric_apply"):
        # the capture of the symmetric run is keyed "<config>_symmetric": A'+B' = stageA_tma +
        # stageA_dual, C' = stageB_tma
        parts = ["stageA_VTx", "stageA_dual"] if dom == "stageA_VTx" else ["stageB_Ut"]
        tr = [ncu_traffic(args.config + "_symmetric", k) for k in parts]
        dom_traffic = sum(tr) if all(t is not None for t in tr) else None   # slot 1 = A' + B' (two kernels), slot 2 = C'
        dom = {"stageA_VTx": "symmetric A'+B' (stageA_tma + stageA_dual)",
               "stageB_Ut": "symmetric C' (stageB_tma)"}[dom]
        other = {"stageA_VTx": "symmetric A'+B' (stageA_tma + stageA_dual)",
                 "stageB_Ut": "symmetric C' (stageB_tma)"}[other]
        per = {"symA+B" if k == "stageA_VTx" else "symC" if k == "stageB_Ut" else k: v for k, v in per.items()}
    roof = {"kernel": dom, "bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
            "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
            "traffic": dom_traffic, "bytes_per_launch": dom_bytes, "ms_per_launch": round(dom_ms, 4),
            "other_hbm_kernel": {"kernel": other, "ms_per_launch": round(other_ms, 4),
                                 "bytes_per_launch": other_bytes,
                                 "frac": round(other_bytes / (other_ms * 1e-3) / 1e9 / peak, 4)},
            "stage_ms_per_matvec": {k: round(v, 4) for k, v in per.items()},
            "whole_matvec_frac": round(inf["matvec_bytes"] / (ms_step * 1e-3) / 1e9 / peak, 4)}
    try:   # context: the practical ceiling of a pure-read stream (tools/read_bw.cu)
        with open(os.path.join(ROOT, "profiles", "read_bw_measured.json")) as f:
            rp = json.load(f)["read_gbs_best"]
        roof["read_peak_microbench"] = {"gbs": rp, "frac": round(achieved / rp, 4),
                                        "source": "profiles/read_bw_measured.json (tools/read_bw.cu)"}
    except Exception:
        pass

    # e2e through the public API with host (pinned) buffers, copies inside the timed region
    e2e = None
    if world == 1 and not args.no_e2e:
        xh = torch.empty(cfg.n, dtype=torch.float64).pin_memory()
        yh = torch.empty(cfg.n, dtype=torch.float64).pin_memory()
        xh.copy_(xs[0].cpu())
        for _ in range(2):
            op.matvec_raw(xh.data_ptr(), yh.data_ptr(), h2d.ORDER_ORIGINAL)
        torch.cuda.synchronize()
        ke = max(10, args.steps // 2)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ke):
            op.matvec_raw(xh.data_ptr(), yh.data_ptr(), h2d.ORDER_ORIGINAL)
        e1.record(stream)
        torch.cuda.synchronize()
        sync_value = 1e3 * ke / e0.elapsed_time(e1)
        # the headline e2e: hodlr2d_matvec_async, fresh pinned x per step (the device run's
        # vectors), y into two alternating pinned buffers; upload of step k + 1 and download of
        # step k - 1 overlap step k's kernels (two copy-engine streams, library staging slots).
        # Host wall clock from a synchronised start to hodlr2d_wait: every copy is inside.
        xhs = [xs[k % len(xs)].cpu().pin_memory() for k in range(min(len(xs), 4))]
        yhs = [torch.empty(cfg.n, dtype=torch.float64).pin_memory() for _ in range(2)]
        for k in range(4):
            op.matvec_async_raw(xhs[k % len(xhs)].data_ptr(), yhs[k % 2].data_ptr(), h2d.ORDER_ORIGINAL)
        op.wait()
        torch.cuda.synchronize()
        ka = max(20, args.steps)
        t0 = time.perf_counter()
        for k in range(ka):
            op.matvec_async_raw(xhs[k % len(xhs)].data_ptr(), yhs[k % 2].data_ptr(), h2d.ORDER_ORIGINAL)
        op.wait()
        ta = time.perf_counter() - t0
        e2e = {"value": ka / ta, "unit": "matvecs/s",
               "h2d_bytes_per_step": 8 * cfg.n, "d2h_bytes_per_step": 8 * cfg.n,
               "buffers": "pinned host (torch pin_memory), hodlr2d_matvec_async pipeline",
               "timing": f"host wall clock over {ka} steps, synchronised start, ends at hodlr2d_wait",
               "sync_calls": {"value": sync_value, "unit": "matvecs/s",
                              "timing": "hodlr2d_matvec_ex per step (returns after y is on the host), CUDA events"}}
        # the same with pageable host buffers (numpy): the library stages them through its
        # own pinned buffers (multi-threaded host copies)
        xp = xh.numpy().copy()
        yp = np.empty(cfg.n)
        op.matvec_raw(xp.ctypes.data, yp.ctypes.data, h2d.ORDER_ORIGINAL)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(ke):
            op.matvec_raw(xp.ctypes.data, yp.ctypes.data, h2d.ORDER_ORIGINAL)
        e2e["pageable"] = {"value": ke / (time.perf_counter() - t0), "unit": "matvecs/s",
                           "timing": "host wall clock (each call returns after y is written)"}

    # multi-RHS (NEXT N2): the same fresh vectors, nrhs per call; reported beside the
    # single-vector headline, never in place of it
    multi = None
    if world == 1 and args.multi_rhs > 1 and nx >= args.multi_rhs:
        K = args.multi_rhs
        Ym = torch.empty(K, cfg.n, dtype=torch.float64, device="cuda")
        nb = max(3, min(20, args.steps // K))
        for _ in range(2):
            op.matvec_multi_raw(xs[:K].data_ptr(), Ym.data_ptr(), K, h2d.ORDER_ORIGINAL)
        torch.cuda.synchronize()
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record(stream)
        for b in range(nb):
            k0 = (b * K) % (nx - K + 1)
            op.matvec_multi_raw(xs[k0:k0 + K].data_ptr(), Ym.data_ptr(), K, h2d.ORDER_ORIGINAL)
        m1.record(stream)
        torch.cuda.synchronize()
        ms_b = m0.elapsed_time(m1) / nb
        # bytes per call: the factor panels once per chunk (16 / 8 / 4 / 2 vectors), plus the
        # stored near-field blocks (Alg. 1 l.5) that 16-vector chunks read
        chunks, left, n16 = 0, K, 0
        for c in (16, 8, 4, 2, 1):
            chunks += left // c
            n16 += left // c if c == 16 else 0
            left %= c
        nf_bytes = 8 * op.info()["stored_near_values"] * n16
        fbytes = inf["stageA_bytes"] + inf["stageB_bytes"]
        mbytes = fbytes * chunks + nf_bytes
        multi = {"nrhs": K, "matvecs_per_s": 1e3 * K / ms_b, "ms_per_call": ms_b, "calls": nb,
                 "factor_bytes_per_call": fbytes * chunks, "stored_near_bytes_per_call": nf_bytes,
                 "hbm_frac": round(mbytes / (ms_b * 1e-3) / 1e9 / peaks()[0], 4),
                 "note": "hodlr2d_matvec_multi: factor panels streamed once per chunk of <= 16 "
                         "vectors (16-vector chunks also read the stored near-field blocks); a "
                         "batched-throughput figure, not the per-vector headline"}

    # symmetric block storage (NEXT N1, R23): the same workload built with one ACA
    # per unordered pair and applied by the three-pass symmetric apply; reported beside the
    # directed (paper's) headline, never in place of it
    variants = None
    if world == 1 and not args.symmetric and not args.no_variants:
        variants = {"symmetric_N1": symmetric_variant(h2d, op, cfg, xs, nx, y, stream, args)}

    # near-field P2P against the FP64 pipe.  The kernel that runs on the uniform configs is
    # p2p_warp_kernel (every leaf <= 96 points): it evaluates each leaf's self block in full
    # (sum m^2) and each edge-neighbour leaf pair once, i.e. sum m^2 + (near_pairs - sum m^2)
    # / 2 kernel evaluations, each P2P_FP64_OPS_PER_EVAL FP64-pipe instructions (counted in
    # its SASS).  In the timed matvec it runs concurrently with stages A/B on
    # the spare SM resources, so its FP64 fraction is also probed standalone (set_diag
    # "p2p_serial": the near field alone, before stage A).
    csum = clk.summary()
    alone_ms = p2p_standalone_ms(op, step, args) if world == 1 else None
    p2p = p2p_roofline(op, inf, cfg, per, csum["sm_mhz"], alone_ms)
    roof["p2p"] = p2p
    # C5 (N = 2^24) is the config BASELINE quotes on 8 GPUs: at N >= --c5-min-world ranks the
    # line carries it too (every rank takes part: the all-gather is collective)
    c5 = None
    if dist and world >= args.c5_min_world and args.config == "c3":
        op.close()
        del xs
        torch.cuda.empty_cache()
        try:
            c5 = multi_gpu_config(h2d, args, stream, dist, world, rank, dev)
        except Exception as ex:  # the headline stands on its own
            c5 = {"error": str(ex)}
    if rank == 0:
        line = {
            "metric": "HODLR2D fp64 matvecs/sec", "value": value, "unit": "matvecs/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(cfg, world),
            "points_matvecs_per_s": value * cfg.n,
            "build_seconds": round(build_s, 3),
            "operator": {k: inf[k] for k in ("kappa", "rank_max", "u_values", "v_values", "near_pairs",
                                               "compression_ratio", "truncated", "matvec_bytes",
                                               "tree_seconds", "aca_seconds", "pack_seconds")},
            "roofline": roof, "e2e": e2e, "multi_rhs": multi, "variants": variants,
            "gpu_launches": args.steps * launches_per_matvec(inf, world),
            "clocks": csum,
        }
        if c5 is not None:
            line["c5"] = c5
        # BASELINE's metric spans N = 2^20 .. 2^24: the default (C3) line also carries C4
        # (N = 2^22, 96 GB of factors) measured in the same run on the same GPU
        if world == 1 and args.config == "c3" and not args.no_c4:
            op.close()
            del xs
            torch.cuda.empty_cache()
            try:
                line["c4"] = sub_config(h2d, "c4", args, stream)
            except Exception as ex:  # the headline stands on its own
                line["c4"] = {"error": str(ex)}
        if not args.no_cpu_baseline and world == 1:   # the contract: rank 0 at N = 1 only
            try:
                line["cpu_baseline"] = cpu_baseline(cfg, args.config)
            except Exception as ex:  # the GPU number stands on its own
                line["cpu_baseline"] = {"error": str(ex)}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def multi_gpu_config(h2d, args, stream, dist, world, rank, dev):
    """BASELINE config 5 on `world` GPUs: build (max over ranks) plus 50
    matvecs through the library's LOCAL order (the x all-gather inside, NCCL), timed with
    CUDA events and reduced with MAX over ranks; then each rank times its slice alone with the
    full TREE-order x resident (no gather): T1_virt = the sum over ranks, E_N = T1_virt /
    (N T_N) (SURVEY's E_8 definition; C5 does not fit one GPU)."""
    import torch
    cfg = W.CONFIGS[args.c5_config]
    pts = torch.from_numpy(W.config_points(cfg)).cuda()
    dist.barrier()
    t0 = time.time()
    op = h2d.Hodlr2d.build(pts, cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale, shift=cfg.shift,
                           box_lo=cfg.box_lo, box_side=cfg.box_side, stream=stream.cuda_stream,
                           group=dist.group.WORLD)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    del pts
    inf = op.info()
    perm, _ = op.tree()
    rb, re_ = inf["row_begin"], inf["row_end"]
    nx = 4
    xfull = [W.config_x(cfg, k)[perm] for k in range(nx)]
    xs = torch.stack([torch.from_numpy(x[rb:re_].copy()) for x in xfull]).cuda()
    y = torch.empty(re_ - rb, dtype=torch.float64, device="cuda")
    for k in range(3):
        op.matvec_raw(xs[k % nx].data_ptr(), y.data_ptr(), h2d.ORDER_LOCAL)
    steps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()
    e0.record(stream)
    for k in range(steps):
        op.matvec_raw(xs[k % nx].data_ptr(), y.data_ptr(), h2d.ORDER_LOCAL)
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    ms = e0.elapsed_time(e1) / steps
    # this rank's slice alone: full x resident, TREE order, no all-gather
    xt = torch.from_numpy(xfull[0]).cuda()
    for _ in range(2):
        op.matvec_raw(xt.data_ptr(), y.data_ptr(), h2d.ORDER_TREE)
    e0.record(stream)
    for _ in range(10):
        op.matvec_raw(xt.data_ptr(), y.data_ptr(), h2d.ORDER_TREE)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_slice = e0.elapsed_time(e1) / 10
    on = "cuda" if dist.get_backend() == "nccl" else "cpu"
    v = torch.tensor([ms, build_s, ms_slice, inf["device_bytes"] / 1e9], dtype=torch.float64, device=on)
    vmax, vsum = v.clone(), v.clone()
    dist.all_reduce(vmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(vsum, op=dist.ReduceOp.SUM)
    op.close()
    del xs, xt
    torch.cuda.empty_cache()
    t_n, b_max, t1_virt = float(vmax[0]), float(vmax[1]), float(vsum[2])
    return {"config": config_dict(cfg, world), "n_gpus": world, "value": 1e3 / t_n, "unit": "matvecs/s",
            "ms_per_step": t_n, "steps": steps, "build_seconds_max": round(b_max, 2),
            "build_plus_50_matvecs_s": round(b_max + 50 * t_n / 1e3, 3),
            "points_matvecs_per_s": 1e3 / t_n * cfg.n,
            "slice_ms_max": float(vmax[2]), "T1_virt_ms": t1_virt,
            "efficiency_vs_virtual_1gpu": t1_virt / (world * t_n),
            "device_gb_max": float(vmax[3]),
            "note": "LOCAL-order matvecs (S11 inside the library: ncclAllGather on the handle's "
                    "communicator); T1_virt = sum over ranks of each slice timed alone with the full "
                    "x resident (SURVEY §8(e) E_8 definition); E_4->8 = 4 T_4 / (8 T_8) from the "
                    "driver's N = 4 and N = 8 lines"}


def sub_config(h2d, name, args, stream):
    """Another BASELINE config measured in the same run (device-timed matvecs/s after
    warm-up, the roofline of its dominant kernel, e2e with pinned host buffers)."""
    import torch
    cfg = W.CONFIGS[name]
    pts = torch.from_numpy(W.config_points(cfg)).cuda()
    t0 = time.time()
    op = h2d.Hodlr2d.build(pts, cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale, shift=cfg.shift,
                           box_lo=cfg.box_lo, box_side=cfg.box_side, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    del pts
    inf = op.info()
    nx = 8
    xs = torch.stack([torch.from_numpy(W.config_x(cfg, k)) for k in range(nx)]).cuda()
    y = torch.empty(cfg.n, dtype=torch.float64, device="cuda")
    for k in range(max(3, args.warmup)):
        op.matvec_raw(xs[k % nx].data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
    torch.cuda.synchronize()
    steps = max(10, min(args.steps, 50))
    op.stage_times(reset=True)
    op.set_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for k in range(steps):
            op.matvec_raw(xs[k % nx].data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
        e1.record(stream)
        torch.cuda.synchronize()
    op.set_timing(False)
    ms = e0.elapsed_time(e1) / steps
    st, cnt = op.stage_times(reset=True)
    per = {k: v / max(cnt, 1) for k, v in st.items()}
    peak, peak_kind = peaks()
    a_ms, b_ms = per["stageA_VTx"], per["stageB_Ut"]
    dom, dom_ms, dom_bytes = (("stageB_Ut", b_ms, inf["stageB_bytes"]) if b_ms >= a_ms
                              else ("stageA_VTx", a_ms, inf["stageA_bytes"]))
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    roof = {"kernel": dom, "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
            "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": ncu_traffic(name, dom),
            "bytes_per_launch": dom_bytes, "ms_per_launch": round(dom_ms, 4),
            "stage_ms_per_matvec": {k: round(v, 4) for k, v in per.items()},
            "whole_matvec_frac": round(inf["matvec_bytes"] / (ms * 1e-3) / 1e9 / peak, 4)}
    alone_ms = p2p_standalone_ms(
        op, lambda k: op.matvec_raw(xs[k % nx].data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL), args)
    roof["p2p"] = p2p_roofline(op, inf, cfg, per, clk.summary()["sm_mhz"], alone_ms)
    xh = torch.empty(cfg.n, dtype=torch.float64).pin_memory()
    yh = torch.empty(cfg.n, dtype=torch.float64).pin_memory()
    xh.copy_(xs[0].cpu())
    op.matvec_raw(xh.data_ptr(), yh.data_ptr(), h2d.ORDER_ORIGINAL)
    ke = 10
    e0.record(stream)
    for _ in range(ke):
        op.matvec_raw(xh.data_ptr(), yh.data_ptr(), h2d.ORDER_ORIGINAL)
    e1.record(stream)
    torch.cuda.synchronize()
    sync_value = 1e3 * ke / e0.elapsed_time(e1)
    xhs = [xs[k % nx].cpu().pin_memory() for k in range(min(nx, 2))]
    yhs = [torch.empty(cfg.n, dtype=torch.float64).pin_memory() for _ in range(2)]
    for k in range(2):
        op.matvec_async_raw(xhs[k % len(xhs)].data_ptr(), yhs[k % 2].data_ptr(), h2d.ORDER_ORIGINAL)
    op.wait()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(ke):
        op.matvec_async_raw(xhs[k % len(xhs)].data_ptr(), yhs[k % 2].data_ptr(), h2d.ORDER_ORIGINAL)
    op.wait()
    e2e = {"value": ke / (time.perf_counter() - t0), "unit": "matvecs/s",
           "h2d_bytes_per_step": 8 * cfg.n, "d2h_bytes_per_step": 8 * cfg.n,
           "buffers": "pinned host, hodlr2d_matvec_async pipeline (host wall clock)",
           "sync_calls": {"value": sync_value, "unit": "matvecs/s"}}
    out = {"value": 1e3 / ms, "unit": "matvecs/s", "ms_per_step": ms, "steps": steps,
           "config": config_dict(cfg, 1), "points_matvecs_per_s": 1e3 / ms * cfg.n,
           "build_seconds": round(build_s, 3),
           "operator": {k: inf[k] for k in ("kappa", "rank_max", "u_values", "v_values", "near_pairs",
                                            "truncated", "matvec_bytes", "device_bytes")},
           "roofline": roof, "e2e": e2e, "clocks": clk.summary(),
           "gpu_launches": steps * launches_per_matvec(inf, 1)}
    op.close()
    return out


def symmetric_variant(h2d, op_dir, cfg, xs, nx, y, stream, args):
    """Device-timed matvecs/s of the symmetric build (options.symmetric = 1) on the same
    fresh x vectors, with its relative difference from the directed operator on x_0 (both
    approximate A to aca_tol, so the difference is O(tol))."""
    import torch
    pts = torch.from_numpy(W.config_points(cfg)).cuda()
    t0 = time.time()
    op = h2d.Hodlr2d.build(pts, cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale, shift=cfg.shift,
                           box_lo=cfg.box_lo, box_side=cfg.box_side, stream=stream.cuda_stream, symmetric=True)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    del pts
    inf = op.info()
    ys = torch.empty_like(y)
    for k in range(max(3, args.warmup)):
        op.matvec_raw(xs[k % nx].data_ptr(), ys.data_ptr(), h2d.ORDER_ORIGINAL)
    torch.cuda.synchronize()
    op.stage_times(reset=True)
    op.set_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(args.steps):
        op.matvec_raw(xs[(args.warmup + k) % nx].data_ptr(), ys.data_ptr(), h2d.ORDER_ORIGINAL)
    e1.record(stream)
    torch.cuda.synchronize()
    op.set_timing(False)
    ms = e0.elapsed_time(e1) / args.steps
    st, cnt = op.stage_times(reset=True)
    op.matvec_raw(xs[0].data_ptr(), ys.data_ptr(), h2d.ORDER_ORIGINAL)
    yd = torch.empty_like(y)
    op_dir.matvec_raw(xs[0].data_ptr(), yd.data_ptr(), h2d.ORDER_ORIGINAL)
    torch.cuda.synchronize()
    rel = float(torch.linalg.norm(ys - yd) / torch.linalg.norm(yd))
    dev_bytes = inf["device_bytes"]
    op.close()
    del ys, yd
    return {"value": 1e3 / ms, "unit": "matvecs/s", "ms_per_step": ms, "steps": args.steps,
            "build_seconds": round(build_s, 3), "aca_seconds": inf["aca_seconds"],
            "symmetric_apply": bool(inf["symmetric_apply"]), "matvec_bytes": inf["matvec_bytes"],
            "frac_hbm_whole_matvec": round(inf["matvec_bytes"] / (ms * 1e-3) / 1e9 / peaks()[0], 4),
            "stage_ms_per_matvec": {("symA+B" if k == "stageA_VTx" else "symC" if k == "stageB_Ut" else k):
                                    round(v / max(cnt, 1), 4) for k, v in st.items()},
            "device_bytes": dev_bytes, "rel_diff_vs_directed_x0": rel}


def launches_per_matvec(inf, world):
    # permute-in (1-GPU ORIGINAL order) or unpad (gathered), the low-rank apply kernels
    # (stage A / B rings + small-item kernels; symmetric: A', B', C'), the P2P kernels
    # (warp-per-leaf / CTA fast / generic, those with leaves), combine
    return 2 + inf.get("apply_launches", 2) + inf.get("p2p_launches", 1)


# FP64-pipe instructions per kernel evaluation in p2p_warp_kernel's self-block loop
# (DESIGN.md §6); keyed by kernel id.  log (p2p_warp_kernel<kLogNoSel, 2>, round 2, counted in
# `cuobjdump -sass` of the unrolled self loop: 48 FP64 per 4 evaluations): distance 2 DADD +
# DMUL + DFMA, table log 6 DFMA + 1 DADD (exponent; ln2 / 2 without its lo part),
# accumulation 1 DFMA = 12; a neighbour-block evaluation adds its column-sum DFMA (13).
# (Round 1: 16 with the select and I2F.F64; round 2 before the high-word log: 13.)  IMQ / 1/r:
# distance + rsqrt (MUFU.RSQ64H seed + Newton) + the accumulation, ~12 (estimate).
P2P_FP64_OPS_PER_EVAL = {0: 12, 1: 12, 2: 12}


def p2p_roofline(op, inf, cfg, per, sm_mhz, alone_ms):
    """Near-field P2P against the FP64 pipe.  The kernel that runs on the uniform / grid
    configs is p2p_warp_kernel (every leaf <= 96 points): it evaluates each leaf's self block
    in full (sum m^2) and each edge-neighbour leaf pair once, i.e. sum m^2 + (near_pairs -
    sum m^2) / 2 kernel evaluations, each P2P_FP64_OPS_PER_EVAL FP64-pipe instructions
    (counted in its SASS; + 2 DFMAs with the replicated log table,
    info p2p_log_table = 1).  In the timed matvec it runs concurrently with stages A/B on the
    spare SM resources, so its FP64 fraction is also probed standalone (set_diag
    "p2p_serial": the near field alone, before stage A)."""
    p2p_ms = per["p2p_near"]
    ops_eval = P2P_FP64_OPS_PER_EVAL.get(cfg.kernel)
    if ops_eval is not None and inf.get("p2p_log_table") == 1:
        ops_eval += 2
    sm_hz = (sm_mhz or 1965.0) * 1e6
    self_evals = 0.0
    if inf.get("adaptive"):   # p2p_list_kernel: every directed pair of the dense blocks
        evals = float(inf["p2p_pairs"])
    else:
        _, ls = op.tree()
        msz = np.diff(ls[inf["leaf_begin"]: inf["leaf_end"] + 1]).astype(np.float64)
        self_pairs = float((msz * msz).sum())
        warp = msz <= 96   # warp-per-leaf path: full self blocks; CTA paths: i <= j only
        self_evals = float((msz[warp] ** 2).sum() + (msz[~warp] * (msz[~warp] + 1) / 2).sum())
        evals = self_evals + (inf["p2p_pairs"] - self_pairs) / 2.0
    if ops_eval is not None and cfg.kernel == 0 and self_evals > 0:
        # log: a neighbour-block evaluation adds its column-sum DFMA to the self-block count
        ops_eval = (self_evals * ops_eval + (evals - self_evals) * (ops_eval + 1)) / evals
    peak_ops, peak_ops_kind = 148 * 64 * sm_hz, "nominal: 148 SMs x 64 FP64 lanes x SM clock"
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peaks_measured.json")) as f:
            peak_ops = json.load(f)["fp64_dfma_tflops"] * 1e12 / 2.0   # FP64-pipe instr/s
        peak_ops_kind = "measured: tools/fp64_peak.cu sustained DFMA (profiles/fp64_peaks_measured.json)"
    except Exception:
        pass

    def frac(ms):
        return evals * ops_eval / (ms * 1e-3) / peak_ops if (ms and ops_eval) else None

    return {"directed_pairs": int(inf["p2p_pairs"]), "evaluations": int(evals),
            "log_table": {1: "replicated 64 bins", 0: "512 bins"}.get(inf.get("p2p_log_table")),
            "ms_per_launch_concurrent": round(p2p_ms, 4),
            "ms_per_launch_standalone": round(alone_ms, 4) if alone_ms else None,
            "fp64_ops_per_eval": ops_eval, "peak_fp64_lane_ops_per_s": peak_ops,
            "peak_kind": peak_ops_kind,
            "frac_fp64_pipe_standalone": frac(alone_ms),
            "frac_fp64_pipe_concurrent": frac(p2p_ms),
            "overlapped_with": "stageA_VTx + stageB_Ut (low-priority stream, co-resident CTAs)",
            "exposed_ms": round(per["p2p_join_wait"], 4)}


def p2p_standalone_ms(op, step, args, n=10):
    """P2P time with the kernel running alone (H2D_P2P_SERIAL=1), CUDA events of the library."""
    op.set_diag("p2p_serial", 1)
    try:
        op.set_timing(True)
        op.stage_times(reset=True)
        for k in range(n):
            step(k)
        st, cnt = op.stage_times(reset=True)
        return st["p2p_near"] / max(cnt, 1)
    finally:
        op.set_timing(False)
        op.set_diag("p2p_serial", 0)


def ncu_traffic(cfg_name, kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu --set full
    capture of this config (profiles/ncu_traffic.json, written by tools/ncu_summary.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        return t[cfg_name][kernel]
    except Exception:
        return None


def run_rank_slice(args, cfg):
    """One rank's slice of the Morton-range partition on this GPU: the per-GPU
    compute time of the --slice-world run.  The x all-gather is not run (one process); its
    NVLink time is estimated from the measured peer bandwidth (B200_PROFILING.md, 770 GB/s
    per direction).  Prints one informational JSON line (not the driver's bench line)."""
    import torch
    import paper_2204_05536_b200 as h2d
    torch.cuda.set_device(0)
    P, g = args.slice_world, args.rank_slice
    stream = torch.cuda.current_stream()
    pts = W.config_points(cfg)
    t0 = time.time()
    lw = np.load(args.leaf_weights) if args.leaf_weights else None
    op = h2d.Hodlr2d.build(torch.from_numpy(pts).cuda(), cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c,
                           scale=cfg.scale, shift=cfg.shift, box_lo=cfg.box_lo, box_side=cfg.box_side,
                           world=P, rank=g, stream=stream.cuda_stream, leaf_weights=lw, symmetric=args.symmetric)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    inf = op.info()
    if args.dump_leaf_costs:
        np.save(args.dump_leaf_costs, op.leaf_costs())
    perm, _ = op.tree()
    nx = min(args.steps + args.warmup, 8)
    xs = [torch.from_numpy(np.ascontiguousarray(W.config_x(cfg, k)[perm])).cuda() for k in range(nx)]
    y = torch.empty(inf["row_end"] - inf["row_begin"], dtype=torch.float64, device="cuda")
    for k in range(args.warmup):
        op.matvec_raw(xs[k % nx].data_ptr(), y.data_ptr(), h2d.ORDER_TREE)
    op.set_timing(True)
    op.stage_times(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for k in range(args.steps):
            op.matvec_raw(xs[k % nx].data_ptr(), y.data_ptr(), h2d.ORDER_TREE)
        e1.record(stream)
        torch.cuda.synchronize()
    op.set_timing(False)
    ms = e0.elapsed_time(e1) / args.steps
    st, cnt = op.stage_times(reset=True)
    peak, peak_kind = peaks()
    gather_ms = 8.0 * cfg.n * (P - 1) / P / 770e9 * 1e3
    line = {"mode": "rank_slice", "config": config_dict(cfg, P), "slice_world": P, "rank": g,
            "symmetric": bool(args.symmetric), "symmetric_apply": bool(inf["symmetric_apply"]),
            "partition": "measured leaf costs (--leaf-weights)" if lw is not None else "geometric weight",
            "rows": [inf["row_begin"], inf["row_end"]], "build_seconds": round(build_s, 2),
            "ms_per_matvec_compute": ms, "steps": args.steps, "warmup": args.warmup,
            "stage_ms_per_matvec": {k: round(v / max(cnt, 1), 4) for k, v in st.items()},
            "matvec_bytes": inf["matvec_bytes"],
            "hbm_frac_of_measured": inf["matvec_bytes"] / (ms * 1e-3) / 1e9 / peak,
            "allgather_ms_estimate": gather_ms,
            "projected_matvecs_per_s_at_world": 1e3 / (ms + gather_ms),
            "device_gb": inf["device_bytes"] / 1e9, "rank_max": inf["rank_max"],
            "clocks": clk.summary(), "dtype": "f64", "data": "synthetic"}
    print(json.dumps(line), flush=True)


# The paper's T_I / T_G for the largest RBF rows (N = 250000, one laptop core):
# Table tab:ker1_init / tab:k1_sol (phi_1) and tab:ker2_init / tab:ker2_sol (phi_2).
PAPER_RBF_250000 = {"rbf_phi1": {"T_I_s": 105.4, "T_G_s": 12.2752, "r_m": 59, "CR": 0.013},
                    "rbf_phi2": {"T_I_s": 147.6, "T_G_s": 8.93127, "r_m": 118, "CR": 0.021}}


def run_gmres(args):
    """The paper's application (§5.2): A lambda = f, A = N I + phi(|x_i - x_j|), a = 0.001,
    on the m x m Chebyshev grid, ACA 1e-12, N_max 500 with the paper's depth rule (R22),
    GMRES residual 1e-10.  f = A lambda with the HODLR2D operator itself (a
    dense product at N = 250000 is beyond this run); prints one informational line."""
    import torch
    import paper_2204_05536_b200 as h2d
    torch.cuda.set_device(0)
    pts = W.chebyshev_grid(args.grid_m)
    n = pts.shape[0]
    t0 = time.time()
    op = h2d.Hodlr2d.build(torch.from_numpy(pts).cuda(), args.rbf_kernel, args.nmax, 1e-12, c=1e-3, scale=1.0,
                           shift=float(n), box_lo=(-1, -1), box_side=2.0, depth=-3 if args.adaptive else -2,
                           symmetric=args.symmetric)
    torch.cuda.synchronize()
    t_i = time.time() - t0
    inf = op.info()
    lam = torch.from_numpy(np.random.default_rng(1048).uniform(-1.0, 1.0, n)).cuda()
    f = op.matvec(lam)
    op.gmres(f, tol=1e-10)                      # warm-up (allocations, schedules)
    torch.cuda.synchronize()
    tgs = []
    for _ in range(5):                          # median of 5 solves (host-synchronous loop)
        t0 = time.time()
        lam_hat, its, rr = op.gmres(f, tol=1e-10)
        torch.cuda.synchronize()
        tgs.append(time.time() - t0)
    t_g = float(np.median(tgs))
    y = torch.empty_like(f)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        op.matvec_raw(lam.data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
    e1.record()
    torch.cuda.synchronize()
    mv_ms = e0.elapsed_time(e1) / 20
    op.set_timing(True)
    op.stage_times(reset=True)
    for _ in range(5):
        op.matvec_raw(lam.data_ptr(), y.data_ptr(), h2d.ORDER_ORIGINAL)
    st, cnt = op.stage_times(reset=True)
    op.set_timing(False)
    stage_ms = {k: round(v / max(cnt, 1), 4) for k, v in st.items()}
    err = float(torch.linalg.norm(lam_hat - lam) / torch.linalg.norm(lam))
    line = {"mode": "gmres", "workload": f"{args.rbf_kernel}, {args.grid_m}^2 Chebyshev grid, a = 0.001, "
                                         f"beta = N, ACA 1e-12, N_max {args.nmax} "
                                         + ("(adaptive quadtree, R24)" if args.adaptive else "(paper depth rule)")
                                         + (", symmetric build + apply (R23)" if args.symmetric else ""),
            "n_leaves": inf["n_leaves"], "near_pairs": inf["near_pairs"],
            "factor_gb": (inf["u_values"] + inf["v_values"]) * 8e-9,
            "n": n, "kappa": inf["kappa"], "rank_max": inf["rank_max"],
            "compression_ratio": inf["compression_ratio"], "T_I_s": round(t_i, 3), "T_G_s": round(t_g, 4),
            "T_G_runs_s": [round(v, 4) for v in tgs], "matvec_ms": round(mv_ms, 3), "stage_ms_per_matvec": stage_ms,
            "matvec_gbytes": inf["matvec_bytes"] / 1e9,
            "p2p_leaves_warp_fast_generic": inf["p2p_leaves"], "small_items_A_B": inf["small_items"],
            "iterations": its, "rel_residual": rr, "solution_rel_error": err,
            "paper_context": PAPER_RBF_250000.get(args.rbf_kernel) if n == 250000 else None,
            "note": "paper numbers: one laptop core (P:1022), context only"}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    cfg = W.CONFIGS[args.config]
    if args.mode == "gmres":
        run_gmres(args)
        return
    if args.rank_slice is not None:
        run_rank_slice(args, cfg)
        return
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
