"""GPU parity of the near-field paths (S9): the warp-per-leaf kernel for <= 32-point leaves,
the CTA fast kernel and the generic kernel (info p2p_leaves = [warp, fast, generic]); the
side-stream schedule of the classes against the one-stream schedule (bit-identical).

Bars: the matvec vs the dense product <= 10 tol-level bounds; with the warp path disabled
(H2D_P2P_NOWARP=1: the same leaves on the CTA paths, different summation order) equal to
1e-14; a world-2 partition (leaves next to the cut go generic) reassembles the full matvec.
Inputs: the paper's Chebyshev grids at the depth rule (most interior leaves hold a few
points, the corner leaves hundreds), tiny uniform leaves, every distance kernel.
"""
import os

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

KID = {"log": 0, "imq": 1, "one_over_r": 2, "rbf_phi1": 3, "rbf_phi2": 4}


@pytest.fixture(scope="module")
def h2d():
    import paper_2204_05536_b200 as m
    m.lib()
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def build(h2d, pts, kernel, leaf, tol, nowarp=False, **kw):
    args = dict(box_lo=(-1, -1), box_side=2.0)
    args.update(kw)
    if nowarp:
        os.environ["H2D_P2P_NOWARP"] = "1"
    try:
        return h2d.Hodlr2d.build(dev(pts), kernel, leaf, tol, **args)
    finally:
        os.environ.pop("H2D_P2P_NOWARP", None)


CASES = [
    ("cheb_phi1", lambda: W.chebyshev_grid(120), "rbf_phi1", 500, 1e-12, {"c": 1e-3, "shift": 14400.0, "depth": -2}),
    ("cheb_phi2", lambda: W.chebyshev_grid(100), "rbf_phi2", 300, 1e-12, {"c": 1e-3, "shift": 10000.0, "depth": -2}),
    ("cheb_log", lambda: W.chebyshev_grid(90), "log", 200, 1e-12, {"depth": -2}),
    ("tiny_uniform_imq", lambda: W.uniform_points(6000, 5150), "imq", 12, 1e-10, {"c": 0.1}),
    ("tiny_uniform_1r", lambda: W.uniform_points(6000, 5151), "one_over_r", 20, 1e-10, {}),
]


@pytest.mark.parametrize("name,gen,kernel,leaf,tol,kw", CASES, ids=[c[0] for c in CASES])
def test_warp_path_vs_dense_and_cta_paths(h2d, name, gen, kernel, leaf, tol, kw):
    pts = gen()
    n = pts.shape[0]
    op = build(h2d, pts, kernel, leaf, tol, **kw)
    ref = build(h2d, pts, kernel, leaf, tol, nowarp=True, **kw)
    pw, pf, pg = op.info()["p2p_leaves"]
    assert pw > 0, (pw, pf, pg)
    assert ref.info()["p2p_leaves"][0] == 0 and sum(ref.info()["p2p_leaves"]) == pw + pf + pg
    x = W.random_vector(n, 5200)
    y = op.matvec(dev(x)).cpu().numpy()
    assert rel(y, ref.matvec(dev(x)).cpu().numpy()) <= 1e-14
    yd = oracle.dense_matvec(pts, x, KID[kernel], kw.get("c", 1.0), 1.0, kw.get("shift", 0.0))
    assert rel(y, yd) <= max(10 * tol, 1e-12)


def test_warp_path_oracle_factors(h2d, tmp_path):
    """With the oracle's factors loaded the whole matvec (near field included) matches the
    oracle matvec to 1e-12 on a Chebyshev grid whose interior leaves go to the warp path."""
    pts = W.chebyshev_grid(64)
    kw = dict(c=1e-3, scale=1.0, shift=4096.0, box_lo=(-1, -1), box_side=2.0, depth=-2)
    orc = oracle.Operator(pts, KID["rbf_phi1"], 100, 1e-12, **kw)
    path = str(tmp_path / "f.bin")
    orc.save_factors(path)
    op = h2d.Hodlr2d.build(dev(pts), "rbf_phi1", 100, 1e-12, **kw)
    assert op.info()["p2p_leaves"][0] > 0
    op.load_factors(path)
    x = W.random_vector(pts.shape[0], 5300)
    assert rel(op.matvec(dev(x)).cpu().numpy(), orc.matvec(x)) <= 1e-12


def test_warp_path_partition_union(h2d):
    pts = W.chebyshev_grid(80)
    kw = dict(depth=-2)
    full = build(h2d, pts, "log", 150, 1e-12, **kw)
    perm, _ = full.tree()
    x = W.random_vector(pts.shape[0], 5400)[perm]
    yfull = full.matvec(dev(x), order="tree").cpu().numpy()
    parts = []
    for rank in range(2):
        p = build(h2d, pts, "log", 150, 1e-12, world=2, rank=rank, **kw)
        assert p.info()["p2p_leaves"][0] > 0
        parts.append(p.matvec(dev(x), order="tree").cpu().numpy())
    assert rel(np.concatenate(parts), yfull) <= 1e-14


@pytest.mark.parametrize("symmetric", [False, True])
def test_small_item_kernels(h2d, symmetric):
    """Clustered Chebyshev grid at the depth rule: hundreds of boxes <= 32 rows and leaves
    <= 8 rows run on the warp-per-item stage A / B kernels (info small_items; the default
    threshold of 4 per SM lowered to 1 by H2D_SMALL_MIN).  Equal to the
    all-ring build (H2D_SMALL_ITEMS=0) to 1e-13 and to the dense product to 1e-10;
    symmetric builds route A' / C' the same way."""
    pts = W.chebyshev_grid(150)
    kw = dict(c=1e-3, shift=22500.0, depth=-2, symmetric=symmetric)
    os.environ["H2D_SMALL_MIN"] = "1"   # this size has fewer than 4 per SM of them
    try:
        op = build(h2d, pts, "rbf_phi1", 100, 1e-12, **kw)
    finally:
        os.environ.pop("H2D_SMALL_MIN")
    sa, sb = op.info()["small_items"]
    assert sa > 0 and sb > 0, (sa, sb)
    os.environ["H2D_SMALL_ITEMS"] = "0"
    try:
        ref = build(h2d, pts, "rbf_phi1", 100, 1e-12, **kw)
    finally:
        os.environ.pop("H2D_SMALL_ITEMS")
    assert ref.info()["small_items"] == [0, 0]
    x = W.random_vector(pts.shape[0], 5500)
    y = op.matvec(dev(x)).cpu().numpy()
    assert rel(y, ref.matvec(dev(x)).cpu().numpy()) <= 1e-13
    yd = oracle.dense_matvec(pts, x, KID["rbf_phi1"], 1e-3, 1.0, 22500.0)
    assert rel(y, yd) <= 1e-10
    # every padded leaf height of the stage-B small kernel (2 / 4 / 8: the fixed row-pair
    # path; 6: the selected-multiplier path) is present and correct on its own rows
    perm, ls = op.tree()
    sizes = np.diff(ls)
    yt, rt = y[perm], ref.matvec(dev(x)).cpu().numpy()[perm]
    for hp in (2, 4, 6, 8):
        leaves = np.nonzero((sizes + 1) // 2 * 2 == hp)[0]
        leaves = leaves[sizes[leaves] > 0]
        assert leaves.size > 0, hp
        rows = np.concatenate([np.arange(ls[i], ls[i + 1]) for i in leaves])
        assert rel(yt[rows], rt[rows]) <= 1e-12, hp


def test_p2p_side_streams_bit_identical(h2d):
    """The near-field classes (generic CTA leaves, warp leaves of 1 / 2 / 3 rows per lane) run
    on their own low-priority streams; every slot value has one writer and a fixed summation
    order, so the result equals the one-stream schedule (set_diag("p2p_onestream", 1)) bit for bit.
    Chebyshev 300^2 at the depth rule with N_max 500: corner leaves of hundreds of points
    (generic kernel) beside thousands of small ones."""
    pts = W.chebyshev_grid(300)
    op = build(h2d, pts, "rbf_phi1", 500, 1e-12, c=1e-3, shift=90000.0, depth=-2)
    warp, _, generic = op.info()["p2p_leaves"]
    assert warp > 0 and generic > 0, op.info()["p2p_leaves"]
    x = W.random_vector(pts.shape[0], 5600)
    y = op.matvec(dev(x)).cpu().numpy()
    op.set_diag("p2p_onestream", 1)
    y1 = op.matvec(dev(x)).cpu().numpy()
    op.set_diag("p2p_onestream", 0)
    assert np.array_equal(y, y1)
    yd = oracle.dense_matvec(pts, x, KID["rbf_phi1"], 1e-3, 1.0, 90000.0)
    assert rel(y, yd) <= 1e-10


@pytest.mark.parametrize("path", ["warp", "cta", "generic"])
def test_log_kernel_subnormal_distances(h2d, path):
    """Points closer than ~1.5e-154 have a subnormal r^2; the near field's table log
    (hlog_r2) normalises it instead of reading a zero exponent field.
    Pairs 1e-160 apart (r^2 = 1e-320, K = 0.5 log r^2 ~ -368) inside leaves of every
    near-field path: the warp kernel (<= 96 points), the CTA kernel (warp path off) and the
    generic kernel (> 96 points), plus the multi-RHS near field; vs the oracle's dense
    product (libm log)."""
    base = W.uniform_points(3000, 4160)
    t = np.linspace(-0.95, 0.95, 40)
    extra = [np.stack([np.zeros(40), t], 1), np.stack([1e-160 * np.arange(1, 41), t], 1),   # |dx| <= 4e-159
             np.stack([t[:20], np.zeros(20)], 1), np.stack([t[:20], np.full(20, 3e-155)], 1)]   # dy = 3e-155
    pts = np.concatenate([base] + extra)
    d = pts[3000:3040] - pts[3040:3080]
    assert np.all((d ** 2).sum(1) < 2.2250738585072014e-308) and np.all((d ** 2).sum(1) > 0)
    leaf = {"warp": 64, "cta": 64, "generic": 200}[path]
    op = build(h2d, pts, "log", leaf, 1e-10, nowarp=(path == "cta"))
    warp, fast, generic = op.info()["p2p_leaves"]
    assert {"warp": warp, "cta": fast, "generic": generic}[path] > 0, op.info()["p2p_leaves"]
    x = W.random_vector(pts.shape[0], 4161)
    yd = oracle.dense_matvec(pts, x, 0)
    assert rel(op.matvec(dev(x)).cpu().numpy(), yd) <= 1e-9
    X = np.stack([W.random_vector(pts.shape[0], 4170 + k) for k in range(8)])
    Y = op.matvec_multi(dev(X)).cpu().numpy()
    for k in (0, 7):
        assert rel(Y[k], oracle.dense_matvec(pts, X[k], 0)) <= 1e-9


@pytest.mark.parametrize("gen", ["grid", "uniform"])
def test_log_table_variants(h2d, gen):
    """The warp near field's two log tables (H2D_P2P_TABLE=0: 512 bins; 1: 64 bins stored 8
    times, degree-5 polynomial; unset: the build times both and keeps the faster) give the
    same matvec to rounding, and each matches the dense product; on a regular grid (64-point
    leaves, the C4 geometry at 128^2) and on uniform points (C3 geometry at 16384)."""
    pts = W.grid_points(128) if gen == "grid" else W.uniform_points(16384, 5160)
    n = pts.shape[0]
    ops = []
    for t in ("0", "1", None):
        if t is not None:
            os.environ["H2D_P2P_TABLE"] = t
        try:
            ops.append(h2d.Hodlr2d.build(dev(pts), "log", 64, 1e-10, box_lo=(-1, -1), box_side=2.0))
        finally:
            os.environ.pop("H2D_P2P_TABLE", None)
    assert ops[0].info()["p2p_leaves"][0] > 0
    assert (ops[0].info()["p2p_log_table"], ops[1].info()["p2p_log_table"]) == (0, 1)
    assert ops[2].info()["p2p_log_table"] in (0, 1)
    x = W.random_vector(n, 5161)
    ys = [o.matvec(dev(x)).cpu().numpy() for o in ops]
    assert rel(ys[1], ys[0]) <= 1e-14
    assert rel(ys[2], ys[0]) <= 1e-14
    yd = oracle.dense_matvec(pts, x, 0)
    for y in ys:
        assert rel(y, yd) <= 1e-9
