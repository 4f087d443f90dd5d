"""S11 behind the C ABI: the multi-GPU matvec as one library call (H2D_ORDER_LOCAL).

Each rank passes only its TREE-order slice of x; the library all-gathers the slices itself
(the paper's distributed matvec, §6, load model Eq. eq:par P:1259-1266)
and overlaps the gather with the stage-A items whose column box is local.

  * NCCL communicator (options.nccl_id): a world of 1 on cuda:0 (one GPU per rank is NCCL's
    rule; this pool gives one GPU) runs the NCCL code path end to end — unique id,
    ncclCommInitRank, ncclMemAlloc'd + registered gather buffer, ncclAllGather — and must
    equal the TREE-order matvec bitwise.
  * Host-staged communicator (options.allgather over a gloo group): worlds of 2 and 3
    processes sharing cuda:0 run the same split (local items, exchange, unpad, remaining
    items); with the oracle's factors loaded the reassembled y matches the oracle matvec to
    rel-l2 <= 1e-12, and with GPU-built factors the single-rank handle to 1e-13.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def h2d():
    import paper_2204_05536_b200 as m
    m.lib()
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def build(h2d, cfg, pts, **kw):
    return h2d.Hodlr2d.build(dev(pts), cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale,
                             shift=cfg.shift, box_lo=cfg.box_lo, box_side=cfg.box_side, **kw)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_nccl_world1_local_order(h2d, name):
    cfg = W.CONFIGS[name]
    pts = W.config_points(cfg)
    ref = build(h2d, cfg, pts)
    op = build(h2d, cfg, pts, nccl_id=h2d.comm_unique_id())
    inf = op.info()
    assert inf["comm_kind"] == 1 and inf["world"] == 1
    perm, _ = op.tree()
    for k in range(3):
        xt = dev(W.config_x(cfg, k)[perm])
        y = op.matvec(xt, order="local").cpu().numpy()
        y_ref = ref.matvec(xt, order="tree").cpu().numpy()
        assert np.array_equal(y, y_ref)
    # host pointers through the same entry point
    xh = W.config_x(cfg, 0)[perm].copy()
    assert np.array_equal(op.matvec(xh, order="local"), ref.matvec(dev(xh), order="tree").cpu().numpy())
    # LOCAL needs a communicator
    with pytest.raises(h2d.Hodlr2dError):
        ref.matvec(xt, order="local")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, cfg_name, factor_path, q):
    try:
        import torch
        import torch.distributed as dist
        import paper_2204_05536_b200 as m
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        cfg = W.CONFIGS[cfg_name]
        pts = W.config_points(cfg)
        op = m.Hodlr2d.build(torch.from_numpy(pts).cuda(), cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c,
                             scale=cfg.scale, shift=cfg.shift, box_lo=cfg.box_lo, box_side=cfg.box_side,
                             group=dist.group.WORLD, skip_aca=factor_path is not None)
        if factor_path is not None:
            op.load_factors(factor_path)
        inf = op.info()
        perm, _ = op.tree()
        rb, re_ = inf["row_begin"], inf["row_end"]
        ys = []
        for k in range(2):
            xl = torch.from_numpy(W.config_x(cfg, k)[perm][rb:re_].copy()).cuda()
            ys.append(op.matvec(xl, order="local").cpu().numpy())
        q.put((rank, rb, re_, inf["comm_kind"], inf["local_items"], ys))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001 - reported to the parent
        q.put((rank, None, None, None, None, repr(e)))


def run_world(world, cfg_name, factor_path=None):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, cfg_name, factor_path, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[1] is not None, r[5]
    res.sort(key=lambda r: r[1])
    assert res[0][1] == 0 and all(res[i][2] == res[i + 1][1] for i in range(world - 1))
    assert all(r[3] == 2 for r in res)                      # host-staged communicator
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_host_staged_world_oracle_factors(h2d, world, tmp_path):
    cfg = W.CONFIGS["c2"]
    pts = W.config_points(cfg)
    orc = oracle.Operator(pts, cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale, shift=cfg.shift,
                          box_lo=cfg.box_lo, box_side=cfg.box_side)
    path = str(tmp_path / "c2.h2df")
    orc.save_factors(path)
    perm, _ = orc.tree()
    res = run_world(world, "c2", path)
    for k in range(2):
        y = np.concatenate([r[5][k] for r in res])
        assert y.shape == (cfg.n,)
        assert rel(y, orc.matvec(W.config_x(cfg, k))[perm]) <= 1e-12
    # the overlap is real: some stage-A items are local, some wait for the gather
    for r in res:
        assert r[4][0] + r[4][1] > 0


def test_host_staged_world2_gpu_factors(h2d):
    cfg = W.CONFIGS["c1"]
    pts = W.config_points(cfg)
    full = build(h2d, cfg, pts)
    perm, _ = full.tree()
    res = run_world(2, "c1")
    for k in range(2):
        y = np.concatenate([r[5][k] for r in res])
        yf = full.matvec(dev(W.config_x(cfg, k)[perm]), order="tree").cpu().numpy()
        assert rel(y, yf) <= 1e-13
