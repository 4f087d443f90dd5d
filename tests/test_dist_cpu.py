"""Multi-rank host logic of the Morton-range partition on CPU with gloo.

World size 2 and 3 processes: each rank takes its leaf range from the C ABI's host-only
hodlr2d_partition, builds the ORACLE restricted to its rows (the GPU path is not
available here), contributes its TREE-order x slice to ONE equal-count all_gather (padded
to the max slice, exactly the layout of H2D_ORDER_GATHERED), unpads it, computes its y
rows and gathers them.  The union must equal the single-process oracle matvec bitwise
(same summation order per row).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import paper_2204_05536_b200 as h2d
    import workloads as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    oracle.set_threads(1)
    cfg = W.CONFIGS["c1"]
    pts = W.config_points(cfg)
    kappa = oracle.depth(cfg.n, cfg.leaf_size)
    _, perm, ls = oracle.tree(pts, cfg.box_lo, cfg.box_side, kappa)
    lb, le = h2d.partition(ls, kappa, world, rank)
    a, b = int(ls[lb]), int(ls[le])
    # every rank's count -> padded slot size
    cnt = torch.tensor([b - a], dtype=torch.int64)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt)
    stride = int(max(c.item() for c in counts))
    op = oracle.Operator(pts, cfg.kernel, cfg.leaf_size, cfg.tol, box_lo=cfg.box_lo,
                         box_side=cfg.box_side, row_range=(a, b))
    x = W.config_x(cfg, 7)
    xt_local = x[perm][a:b]
    send = torch.zeros(stride, dtype=torch.float64)
    send[: b - a] = torch.from_numpy(xt_local)
    recv = torch.zeros(world * stride, dtype=torch.float64)
    dist.all_gather_into_tensor(recv, send)              # ONE collective per matvec
    starts = [0]
    for c in counts:
        starts.append(starts[-1] + int(c.item()))
    xt = np.concatenate([recv[r * stride: r * stride + int(counts[r].item())].numpy()
                         for r in range(world)])
    assert xt.shape[0] == cfg.n
    y = op.matvec(xt, order="tree")[a:b]
    ys = [torch.zeros(stride, dtype=torch.float64) for _ in range(world)]
    ysend = torch.zeros(stride, dtype=torch.float64)
    ysend[: b - a] = torch.from_numpy(y)
    dist.all_gather(ys, ysend)
    if rank == 0:
        full = np.concatenate([ys[r][: int(counts[r].item())].numpy() for r in range(world)])
        np.save(os.path.join(out_dir, f"y_{world}.npy"), full)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_partition_allgather_union(world, tmp_path):
    import oracle
    import workloads as W
    port = free_port()
    mp.spawn(worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    y = np.load(tmp_path / f"y_{world}.npy")
    cfg = W.CONFIGS["c1"]
    pts = W.config_points(cfg)
    full = oracle.Operator(pts, cfg.kernel, cfg.leaf_size, cfg.tol, box_lo=cfg.box_lo,
                           box_side=cfg.box_side)
    kappa = full.kappa
    _, perm, _ = oracle.tree(pts, cfg.box_lo, cfg.box_side, kappa)
    x = W.config_x(cfg, 7)
    yref = full.matvec(x[perm], order="tree")
    assert np.array_equal(y, yref)


def test_partition_covers_all_leaves_contiguously():
    import oracle
    import paper_2204_05536_b200 as h2d
    import workloads as W
    cfg = W.CONFIGS["c3"]
    pts = W.config_points(cfg)
    kappa = oracle.depth(cfg.n, cfg.leaf_size)
    _, _, ls = oracle.tree(pts, cfg.box_lo, cfg.box_side, kappa)
    for world in (1, 2, 4, 8):
        ranges = [h2d.partition(ls, kappa, world, r) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == 1 << (2 * kappa)
        assert all(ranges[r][1] == ranges[r + 1][0] for r in range(world - 1))
        # equal shares of the per-leaf load w(L) = |L| (1 + sum over L's ancestors X of |I_X|)
        # up to the coarse-box snap (each cut moves by <= 4 % of a share) and one leaf;
        # |I_X| from the oracle's literal lists (Defs 4.1-4.5), not the library's closed form
        sz = np.diff(ls).astype(np.float64)
        s = np.ones(1 << (2 * kappa))
        for l in range(1, kappa + 1):
            off, _ = oracle.level_lists(l)
            s += np.repeat(np.diff(off), 1 << (2 * (kappa - l)))
        w = sz * s
        loads = [w[a:b].sum() for a, b in ranges]
        assert max(loads) - min(loads) <= 0.08 * w.sum() / world + 2 * w.max()
        rows = [int(ls[b]) - int(ls[a]) for a, b in ranges]
        assert max(rows) <= 1.15 * cfg.n / world        # still close to equal point shares
