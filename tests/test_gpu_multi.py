"""GPU parity of the multi-RHS matvec (NEXT N2, hodlr2d_matvec_multi) through the C ABI.

Bars: with the oracle's factors loaded, every column of Y = A X matches the oracle matvec
of that column to rel-l2 <= 1e-12 (the single-vector bar); with GPU-built factors, every
column matches the single-vector GPU matvec to <= 1e-13 (same operator, different
summation order).  Chunks of 16 / 8 / 4 / 2 and a trailing single vector are all exercised
(nrhs = 1, 2, 3, 5, 8, 11, 16, 19, 31), as are TREE order on a row-restricted handle, host pointers,
every kernel, leaves > 128 points (row blocks of the near field) and empty leaves.
"""
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


def cfg_build(h2d, cfg, pts=None, **kw):
    pts = W.config_points(cfg) if pts is None else pts
    args = dict(c=cfg.c, scale=cfg.scale, shift=cfg.shift, box_lo=cfg.box_lo, box_side=cfg.box_side)
    args.update(kw)
    return pts, h2d.Hodlr2d.build(dev(pts), cfg.kernel, cfg.leaf_size, cfg.tol, **args)


@pytest.mark.parametrize("nrhs", [1, 2, 3, 5, 8, 11, 16, 19])
def test_multi_oracle_factors_c1(h2d, nrhs, tmp_path):
    cfg = W.CONFIGS["c1"]
    pts = W.config_points(cfg)
    orc = oracle.Operator(pts, cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale,
                          shift=cfg.shift, box_lo=cfg.box_lo, box_side=cfg.box_side)
    path = str(tmp_path / "f.bin")
    orc.save_factors(path)
    _, op = cfg_build(h2d, cfg, pts)
    op.load_factors(path)
    X = np.stack([W.config_x(cfg, k) for k in range(nrhs)])
    Y = op.matvec_multi(dev(X)).cpu().numpy()
    for k in range(nrhs):
        assert rel(Y[k], orc.matvec(X[k])) <= 1e-12, k


@pytest.mark.parametrize("name", ["c2", "c1"])
def test_multi_matches_single_gpu(h2d, name):
    cfg = W.CONFIGS[name]
    pts, op = cfg_build(h2d, cfg)
    X = np.stack([W.config_x(cfg, k) for k in range(31)])   # chunks of 16, 8, 4, 2, 1
    Y = op.matvec_multi(dev(X)).cpu().numpy()
    for k in range(31):
        y1 = op.matvec(dev(X[k])).cpu().numpy()
        assert rel(Y[k], y1) <= 1e-13, k
    # host pointers give the same result (deterministic)
    Yh = op.matvec_multi(X.copy())
    assert np.array_equal(Yh, Y)


@pytest.mark.parametrize("kernel,c,scale,shift", [("imq", 0.1, 1.0, 0.0), ("one_over_r", 1.0, 1.0, 0.0),
                                                  ("rbf_phi1", 1e-3, 1.0, 4096.0),
                                                  ("rbf_phi2", 1e-3, 1.0, 4096.0),
                                                  ("test_lowrank", 1.0, 1.0, 0.5)])
def test_multi_kernels(h2d, kernel, c, scale, shift):
    pts = W.uniform_points(4096, 91)
    op = h2d.Hodlr2d.build(dev(pts), kernel, 64, 1e-10, c=c, scale=scale, shift=shift,
                           box_lo=(-1, -1), box_side=2.0, test_rank=5)
    X = np.stack([W.random_vector(4096, 200 + k) for k in range(20)])
    Y = op.matvec_multi(dev(X)).cpu().numpy()
    for k in range(20):
        assert rel(Y[k], op.matvec(dev(X[k])).cpu().numpy()) <= 1e-13


def test_multi_big_and_empty_leaves(h2d):
    # Chebyshev grid with N_max 500: corner leaves far above 128 points; clustered points:
    # empty leaves
    for pts, leaf in ((W.chebyshev_grid(60), 500), (W.uniform_points(5000, 78, (-1.0, -1.0), 0.9), 64)):
        op = h2d.Hodlr2d.build(dev(pts), "log", leaf, 1e-10, box_lo=(-1, -1), box_side=2.0)
        n = pts.shape[0]
        X = np.stack([W.random_vector(n, 300 + k) for k in range(16)])
        Y = op.matvec_multi(dev(X)).cpu().numpy()
        for k in range(16):
            yd = oracle.dense_matvec(pts, X[k], 0)
            assert rel(Y[k], op.matvec(dev(X[k])).cpu().numpy()) <= 1e-13
            assert rel(Y[k], yd) <= 1e-9


def test_multi_tree_order_row_partition(h2d):
    cfg = W.CONFIGS["c1"]
    pts = W.config_points(cfg)
    full = h2d.Hodlr2d.build(dev(pts), cfg.kernel, cfg.leaf_size, cfg.tol, box_lo=cfg.box_lo,
                             box_side=cfg.box_side)
    perm, _ = full.tree()
    X = np.stack([W.config_x(cfg, k)[perm] for k in range(22)])
    for rank in range(2):
        part = h2d.Hodlr2d.build(dev(pts), cfg.kernel, cfg.leaf_size, cfg.tol, box_lo=cfg.box_lo,
                                 box_side=cfg.box_side, world=2, rank=rank)
        Y = part.matvec_multi(dev(X), order="tree").cpu().numpy()
        for k in range(22):
            y1 = part.matvec(dev(X[k]), order="tree").cpu().numpy()
            assert rel(Y[k], y1) <= 1e-13


def test_multi_clustered_chebyshev(h2d):
    """The paper's clustered workload (Chebyshev grid, depth rule, phi_1 system): the multi-RHS
    kernels stream every item through their rings (the single-vector path routes the tiny
    ones to warp kernels); 16 + 2 + 1 vectors equal their single-vector matvecs to 1e-13."""
    pts = W.chebyshev_grid(120)
    n = pts.shape[0]
    op = h2d.Hodlr2d.build(dev(pts), "rbf_phi1", 100, 1e-12, c=1e-3, shift=float(n), box_lo=(-1, -1),
                           box_side=2.0, depth=-2)
    X = np.stack([W.random_vector(n, 700 + k) for k in range(19)])
    Y = op.matvec_multi(dev(X)).cpu().numpy()
    for k in range(19):
        assert rel(Y[k], op.matvec(dev(X[k])).cpu().numpy()) <= 1e-13, k


def test_multi_gathered_order(h2d):
    """GATHERED order (one padded all-gather buffer per vector, NaN padding never read):
    19 vectors on each rank of a world-2 partition equal the TREE-order multi-RHS matvec."""
    cfg = W.CONFIGS["c1"]
    pts, full = cfg_build(h2d, cfg)
    perm, ls = full.tree()
    kappa = full.info()["kappa"]
    Xt = np.stack([W.config_x(cfg, k)[perm] for k in range(19)])
    world = 2
    ranges = [h2d.partition(ls, kappa, world, r) for r in range(world)]
    rows = [(int(ls[a]), int(ls[b])) for a, b in ranges]
    stride = max(b - a for a, b in rows)
    Xg = np.full((19, world * stride), np.nan)
    for r, (a, b) in enumerate(rows):
        Xg[:, r * stride: r * stride + (b - a)] = Xt[:, a:b]
    for r in range(world):
        _, op = cfg_build(h2d, cfg, pts, world=world, rank=r)
        Yg = op.matvec_multi(dev(Xg), order="gathered").cpu().numpy()
        Yt = op.matvec_multi(dev(Xt), order="tree").cpu().numpy()
        assert np.array_equal(Yg, Yt)


@pytest.mark.parametrize("name", ["c2", "c1"])
def test_multi_stored_near_field(h2d, name):
    """16-vector chunks read the stored dense near-field blocks (Alg. 1 l.5) through
    DMMA; the on-the-fly near field (multi_stored_near = 0) gives the same columns to 1e-13,
    and both match the single-vector matvec."""
    cfg = W.CONFIGS[name]
    pts, op = cfg_build(h2d, cfg)
    X = np.stack([W.config_x(cfg, k) for k in range(16)])
    Ys = op.matvec_multi(dev(X)).cpu().numpy()
    op.set_diag("multi_stored_near", 0)
    Yf = op.matvec_multi(dev(X)).cpu().numpy()
    op.set_diag("multi_stored_near", 1)
    assert np.array_equal(op.matvec_multi(dev(X)).cpu().numpy(), Ys)   # deterministic
    for k in range(16):
        y1 = op.matvec(dev(X[k])).cpu().numpy()
        assert rel(Ys[k], Yf[k]) <= 1e-13, k
        assert rel(Ys[k], y1) <= 1e-13, k


def test_multi_log_table_variants(h2d):
    """The on-the-fly multi-RHS log near field on the replicated 64-bin table (default) and on
    the 512-bin table (set_diag multi_log_table 0): the same columns to rounding, both equal to
    the single-vector matvec to 1e-13; on a grid (C4 geometry) and on uniform points."""
    for pts in (W.grid_points(128), W.uniform_points(16384, 5180)):
        op = h2d.Hodlr2d.build(dev(pts), "log", 64, 1e-10, box_lo=(-1, -1), box_side=2.0)
        X = np.stack([W.random_vector(pts.shape[0], 5181 + k) for k in range(8)])
        Yr = op.matvec_multi(dev(X)).cpu().numpy()
        op.set_diag("multi_log_table", 0)
        Yt = op.matvec_multi(dev(X)).cpu().numpy()
        op.set_diag("multi_log_table", 1)
        for k in (0, 7):
            y1 = op.matvec(dev(X[k])).cpu().numpy()
            assert rel(Yr[k], Yt[k]) <= 1e-14, k
            assert rel(Yr[k], y1) <= 1e-13, k
