"""GPU parity of the symmetric build (NEXT N1, options.symmetric, R23): one ACA per
unordered pair, block (Y, X) := V U^T.

Bars: with the oracle's symmetric factors loaded <= 1e-12 vs the oracle matvec; GPU-built
factors <= 10 tol vs the dense product; (Y, X) blocks hold exactly the swapped factors of
(X, Y); the GPU operator is symmetric to rounding; a world-2 symmetric partition
reassembles the full matvec.
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


def build(h2d, cfg, pts, **kw):
    return h2d.Hodlr2d.build(dev(pts), cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale,
                             shift=cfg.shift, box_lo=cfg.box_lo, box_side=cfg.box_side, symmetric=True, **kw)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_symmetric_oracle_factors_and_dense(h2d, name, tmp_path):
    cfg = W.CONFIGS[name]
    pts = W.config_points(cfg)
    orc = oracle.Operator(pts, cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale, shift=cfg.shift,
                          box_lo=cfg.box_lo, box_side=cfg.box_side, symmetric=True)
    op = build(h2d, cfg, pts)
    x = W.config_x(cfg, 0)
    yd = oracle.dense_matvec(pts, x, cfg.kernel, cfg.c, cfg.scale, cfg.shift)
    y = op.matvec(dev(x)).cpu().numpy()
    assert rel(y, yd) <= 10 * cfg.tol
    path = str(tmp_path / "f.bin")
    orc.save_factors(path)
    op.load_factors(path)
    assert rel(op.matvec(dev(x)).cpu().numpy(), orc.matvec(x)) <= 1e-12


def test_symmetric_blocks_mirrored_and_operator_symmetric(h2d):
    cfg = W.CONFIGS["c1"]
    pts = W.config_points(cfg)
    op = build(h2d, cfg, pts)
    kappa = op.info()["kappa"]
    for l in range(1, kappa + 1):
        off, col = op.lists(l)
        r = op.ranks(l)
        for X in range(len(off) - 1):
            for e in range(off[X], off[X + 1]):
                Y = col[e]
                if Y < X:
                    continue
                t = off[Y] + int(np.searchsorted(col[off[Y]:off[Y + 1]], X))
                assert r[e] == r[t]
                if l <= 2:     # bitwise mirror (copying every block is slow)
                    U, V = op.block(l, e)
                    U2, V2 = op.block(l, t)
                    assert np.array_equal(U, V2) and np.array_equal(V, U2)
    x, y = W.config_x(cfg, 0), W.random_vector(cfg.n, 17)
    Ax = op.matvec(dev(x)).cpu().numpy()
    Ay = op.matvec(dev(y)).cpu().numpy()
    asym = abs(y @ Ax - x @ Ay) / (np.linalg.norm(y) * np.linalg.norm(Ax))
    assert asym < 1e-14


def test_symmetric_partition_union(h2d):
    cfg = W.CONFIGS["c1"]
    pts = W.config_points(cfg)
    full = build(h2d, cfg, pts)
    perm, _ = full.tree()
    x = W.config_x(cfg, 3)[perm]
    yfull = full.matvec(dev(x), order="tree").cpu().numpy()
    parts = []
    for rank in range(2):
        p = build(h2d, cfg, pts, world=2, rank=rank)
        parts.append(p.matvec(dev(x), order="tree").cpu().numpy())
    assert rel(np.concatenate(parts), yfull) <= 1e-13


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_symmetric_apply_matches_directed_panels(h2d, name):
    """The symmetric apply (A' / B' / C', single-rank symmetric handles) and the directed
    panels (H2D_SYMAPPLY=0) run the same symmetric operator: equal to rounding; multi-RHS
    on a symmetric-apply handle equals its single-vector matvecs."""
    import os
    cfg = W.CONFIGS[name]
    pts = W.config_points(cfg)
    op = build(h2d, cfg, pts)
    os.environ["H2D_SYMAPPLY"] = "0"
    try:
        ref = build(h2d, cfg, pts)
    finally:
        os.environ.pop("H2D_SYMAPPLY")
    X = np.stack([W.config_x(cfg, k) for k in range(3)])
    for k in range(3):
        assert rel(op.matvec(dev(X[k])).cpu().numpy(), ref.matvec(dev(X[k])).cpu().numpy()) <= 1e-13
    Y = op.matvec_multi(dev(X)).cpu().numpy()
    for k in range(3):
        assert np.array_equal(Y[k], op.matvec(dev(X[k])).cpu().numpy())
