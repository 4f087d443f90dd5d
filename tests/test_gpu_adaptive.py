"""GPU parity of the adaptive (non-balanced) quadtree (NEXT N4, options.depth = -3, DESIGN.md
R24; the paper's "non-balanced or adaptive quadtree").

Bars: leaves, permutation and per-level interaction lists bit-exact against the oracle; with
the oracle's factors loaded rel-l2 <= 1e-12 against the oracle matvec; GPU-built factors
<= 10 tol against the dense product; the balanced operator when every leaf is deepest.
Inputs: clustered points, the paper's Chebyshev grids with small N_max, a curve.
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


def clustered(n, seed):
    rng = np.random.default_rng(seed)
    a = np.clip(rng.normal((-0.7, -0.6), 0.03, (n // 2, 2)), -1, 1)
    b = rng.uniform(-1, 1, (n - n // 2, 2))
    return np.ascontiguousarray(np.concatenate([a, b]))


CASES = {
    "clustered_6000": (lambda: clustered(6000, 1), 48),
    "chebyshev_120sq": (lambda: W.chebyshev_grid(120), 64),
    "chebyshev_60sq_nmax300": (lambda: W.chebyshev_grid(60), 300),
    "curve_5000": (lambda: np.ascontiguousarray(np.stack([np.linspace(-0.9, 0.9, 5000),
                                                          0.3 * np.sin(3 * np.linspace(-0.9, 0.9, 5000))], 1)), 32),
}

KERNELS = [("log", 0, 1.0, 0.0), ("imq", 1, 0.1, 0.0), ("rbf_phi1", 3, 1e-3, 1.0), ("one_over_r", 2, 1.0, 0.0)]


def gpu(h2d, pts, kernel, nmax, tol, **kw):
    return h2d.Hodlr2d.build(dev(pts), kernel, nmax, tol, box_lo=(-1, -1), box_side=2.0, depth=-3, **kw)


def orc(pts, kid, nmax, tol, **kw):
    return oracle.Operator(pts, kid, nmax, tol, box_lo=(-1, -1), box_side=2.0, depth=-3, **kw)


@pytest.mark.parametrize("name", list(CASES))
def test_adaptive_structure_bit_exact(h2d, name):
    gen, nmax = CASES[name]
    pts = gen()
    op = gpu(h2d, pts, "log", nmax, 1e-10, skip_aca=True)
    o = orc(pts, 0, nmax, 1e-10)
    inf = op.info()
    assert inf["adaptive"] == 1 and inf["kappa"] == o.kappa
    perm, ls = op.tree()
    operm, ols = o.tree()
    assert np.array_equal(perm, operm) and np.array_equal(ls, ols)
    lv, bx = op.leaves()
    olv, obx = o.leaves()
    assert np.array_equal(lv, olv) and np.array_equal(bx, obx)
    assert inf["n_leaves"] == len(olv) and len(set(lv.tolist())) > 1
    for l in range(1, o.kappa + 1):
        off, col = op.lists(l)
        ooff, ocol = o.op_lists(l)
        assert np.array_equal(off, ooff) and np.array_equal(col, ocol), l


@pytest.mark.parametrize("name", list(CASES))
def test_adaptive_oracle_factors(h2d, name, tmp_path):
    gen, nmax = CASES[name]
    pts = gen()
    o = orc(pts, 0, nmax, 1e-10)
    path = tmp_path / "ad.h2df"
    o.save_factors(path)
    op = gpu(h2d, pts, "log", nmax, 1e-10, skip_aca=True)
    op.load_factors(path)
    for k in range(2):
        x = W.random_vector(pts.shape[0], 300 + k)
        assert rel(op.matvec(dev(x)).cpu().numpy(), o.matvec(x)) <= 1e-12
    perm, _ = op.tree()
    x = W.random_vector(pts.shape[0], 310)
    assert rel(op.matvec(dev(x[perm]), order="tree").cpu().numpy(), o.matvec(x)[perm]) <= 1e-12
    for l in range(1, o.kappa + 1):
        assert np.array_equal(op.ranks(l), o.ranks(l)[0])
    # a balanced handle refuses an adaptive factor file
    bal = h2d.Hodlr2d.build(dev(pts), "log", nmax, 1e-10, box_lo=(-1, -1), box_side=2.0, depth=o.kappa, skip_aca=True)
    with pytest.raises(h2d.Hodlr2dError):
        bal.load_factors(path)


@pytest.mark.parametrize("name", ["clustered_6000", "chebyshev_120sq", "curve_5000"])
@pytest.mark.parametrize("kernel,kid,c,shift_per_n", KERNELS)
def test_adaptive_gpu_factors_vs_dense(h2d, name, kernel, kid, c, shift_per_n):
    gen, nmax = CASES[name]
    pts = gen()
    n = pts.shape[0]
    tol = 1e-10
    shift = shift_per_n * n
    op = gpu(h2d, pts, kernel, nmax, tol, c=c, shift=shift)
    x = W.random_vector(n, 77)
    yd = oracle.dense_matvec(pts, x, kid, c, 1.0, shift)
    y = op.matvec(dev(x)).cpu().numpy()
    assert np.linalg.norm(y - yd) / np.linalg.norm(yd - shift * x) <= 10 * tol
    # multi-RHS on an adaptive handle: one vector at a time, same result
    X = np.stack([x, W.random_vector(n, 78)])
    Y = op.matvec_multi(dev(X)).cpu().numpy()
    assert np.array_equal(Y[0], y)


def test_adaptive_equals_balanced_when_every_leaf_is_deepest(h2d):
    pts = W.grid_points(128)             # N_max 64: every level-4 box holds 64 points
    ad = gpu(h2d, pts, "imq", 64, 1e-10, c=0.1)
    ba = h2d.Hodlr2d.build(dev(pts), "imq", 64, 1e-10, c=0.1, box_lo=(-1, -1), box_side=2.0, depth=-2)
    assert ad.info()["kappa"] == ba.info()["kappa"] == 4
    assert np.all(ad.leaves()[0] == 4)
    for l in range(1, 5):
        assert np.array_equal(ad.ranks(l), ba.ranks(l))
    x = W.random_vector(pts.shape[0], 5)
    assert rel(ad.matvec(dev(x)).cpu().numpy(), ba.matvec(dev(x)).cpu().numpy()) <= 1e-14


def test_adaptive_gmres_rbf(h2d):
    """The paper's RBF system on a Chebyshev grid with the adaptive tree:
    GMRES recovers lambda to the paper's accuracy."""
    pts = W.chebyshev_grid(150)
    n = pts.shape[0]
    op = gpu(h2d, pts, "rbf_phi1", 64, 1e-12, c=1e-3, shift=float(n))
    lam = np.random.default_rng(1048).uniform(-1, 1, n)
    f = oracle.dense_matvec(pts, lam, 3, 1e-3, 1.0, float(n))
    x, its, rr = op.gmres(dev(f), tol=1e-10)
    assert rr < 1e-10
    assert rel(x.cpu().numpy(), lam) < 1e-9


SMALL_ENVS = [{}, {"H2D_SMALL_MIN": "1"}, {"H2D_SMALL_MIN": "1", "H2D_SMALL_A_AFTER": "1"},
              {"H2D_SMALL_ITEMS": "0"}]


@pytest.mark.parametrize("env", SMALL_ENVS, ids=["default", "small_min1", "small_a_after", "all_ring"])
def test_adaptive_symmetric_three_pass_apply(h2d, tmp_path, env):
    """Symmetric adaptive handles run the three-pass symmetric apply (A' / B' / C' over the
    adaptive leaves and existing boxes): oracle symmetric adaptive factors <= 1e-12, GPU factors
    vs dense <= 10 tol, and the directed panels of the same build to 1e-13.  Each item
    routing: default, every small box on the warp-per-box A' / B' kernels (H2D_SMALL_MIN=1:
    stageA_small before or after the ring, stageB1_small after the B' ring), all in the rings."""
    import os
    pts = W.chebyshev_grid(130)
    n = pts.shape[0]
    kw = dict(c=1e-3, shift=float(n), symmetric=True)
    os.environ.update(env)
    try:
        _symmetric_three_pass(h2d, tmp_path, pts, n, kw, env)
    finally:
        for k in env:
            os.environ.pop(k)


def _symmetric_three_pass(h2d, tmp_path, pts, n, kw, env):
    import os
    op = gpu(h2d, pts, "rbf_phi1", 64, 1e-12, **kw)
    if env.get("H2D_SMALL_MIN") == "1":
        assert op.info()["small_items"][0] > 0
    inf = op.info()
    assert inf["symmetric_apply"] == 1 and inf["adaptive"] == 1
    x = W.random_vector(n, 21)
    y = op.matvec(dev(x)).cpu().numpy()
    yd = oracle.dense_matvec(pts, x, 3, 1e-3, 1.0, float(n))
    assert np.linalg.norm(y - yd) / np.linalg.norm(yd - n * x) <= 1e-11
    os.environ["H2D_SYMAPPLY"] = "0"
    try:
        ref = gpu(h2d, pts, "rbf_phi1", 64, 1e-12, **kw)
    finally:
        os.environ.pop("H2D_SYMAPPLY")
    assert ref.info()["symmetric_apply"] == 0
    assert rel(y, ref.matvec(dev(x)).cpu().numpy()) <= 1e-13
    o = orc(pts, 3, 64, 1e-12, c=1e-3, shift=float(n), symmetric=True)
    path = tmp_path / "sym.h2df"
    o.save_factors(path)
    op.load_factors(path)
    assert rel(op.matvec(dev(x)).cpu().numpy(), o.matvec(x)) <= 1e-12


@pytest.mark.parametrize("kernel,kid,c,shift", [("log", 0, 1.0, 0.0), ("rbf_phi1", 3, 1e-3, 14400.0)])
def test_adaptive_log_table_variants(h2d, kernel, kid, c, shift):
    """The adaptive list near field on the 512-bin and on the replicated 64-bin log table
    (H2D_P2P_TABLE=0 / 1; unset: timed at build): the same matvec to rounding, each within
    the dense product's bar; info p2p_log_table names the table."""
    import os
    pts = W.chebyshev_grid(120)
    ops = []
    for t in ("0", "1", None):
        if t is not None:
            os.environ["H2D_P2P_TABLE"] = t
        try:
            ops.append(gpu(h2d, pts, kernel, 64, 1e-12, c=c, shift=shift))
        finally:
            os.environ.pop("H2D_P2P_TABLE", None)
    assert [o.info()["p2p_log_table"] for o in ops[:2]] == [0, 1]
    assert ops[2].info()["p2p_log_table"] in (0, 1)
    x = W.random_vector(pts.shape[0], 5170)
    ys = [o.matvec(dev(x)).cpu().numpy() for o in ops]
    assert rel(ys[1], ys[0]) <= 1e-14 and rel(ys[2], ys[0]) <= 1e-14
    yd = oracle.dense_matvec(pts, x, kid, c, 1.0, shift)
    for y in ys:
        assert rel(y, yd) <= 1e-10
