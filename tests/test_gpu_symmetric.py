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


@pytest.mark.parametrize("name,world", [("c1", 2), ("c1", 3), ("c2", 2), ("c2", 4)])
def test_symmetric_partition_union(h2d, name, world):
    """Multi-rank symmetric handles run the three-pass symmetric apply (A' / B' over the whole
    boxes of every pair that touches the rank's rows, C' over its leaves) and store each pair
    ~once instead of both directed blocks: the ranks reassemble the single-rank operator."""
    cfg = W.CONFIGS[name]
    pts = W.config_points(cfg)
    full = build(h2d, cfg, pts)
    perm, _ = full.tree()
    x = W.config_x(cfg, 3)[perm]
    yfull = full.matvec(dev(x), order="tree").cpu().numpy()
    parts, dev_bytes = [], 0
    import os
    os.environ["H2D_SYMAPPLY"] = "0"
    try:
        directed = [build(h2d, cfg, pts, world=world, rank=r).info()["device_bytes"] for r in range(world)]
    finally:
        os.environ.pop("H2D_SYMAPPLY")
    for rank in range(world):
        p = build(h2d, cfg, pts, world=world, rank=rank)
        assert p.info()["symmetric_apply"] == 1
        dev_bytes += p.info()["device_bytes"]
        parts.append(p.matvec(dev(x), order="tree").cpu().numpy())
    assert rel(np.concatenate(parts), yfull) <= 1e-13
    assert dev_bytes < 0.97 * sum(directed)


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
    os.environ["H2D_PAIRAPPLY"] = "0"
    try:
        ref = build(h2d, cfg, pts)
    finally:
        os.environ.pop("H2D_SYMAPPLY")
        os.environ.pop("H2D_PAIRAPPLY")
    X = np.stack([W.config_x(cfg, k) for k in range(3)])
    for k in range(3):
        assert rel(op.matvec(dev(X[k])).cpu().numpy(), ref.matvec(dev(X[k])).cpu().numpy()) <= 1e-13
    Y = op.matvec_multi(dev(X)).cpu().numpy()
    for k in range(3):   # (single vectors take the pair apply, the 8-vector chunks B' / C')
        assert rel(Y[k], op.matvec(dev(X[k])).cpu().numpy()) <= 1e-13


def _sym_pair(h2d, pts, kernel, leaf, tol, **kw):
    """(symmetric-apply handle, directed-panel handle) of the same symmetric build."""
    import os
    args = dict(box_lo=(-1, -1), box_side=2.0, symmetric=True)
    args.update(kw)
    os.environ["H2D_PAIRAPPLY"] = "1"   # (both applies on one handle: set_diag switches)
    try:
        op = h2d.Hodlr2d.build(dev(pts), kernel, leaf, tol, **args)
    finally:
        os.environ.pop("H2D_PAIRAPPLY")
    os.environ["H2D_SYMAPPLY"] = "0"
    os.environ["H2D_PAIRAPPLY"] = "0"
    try:
        ref = h2d.Hodlr2d.build(dev(pts), kernel, leaf, tol, **args)
    finally:
        os.environ.pop("H2D_SYMAPPLY")
        os.environ.pop("H2D_PAIRAPPLY")
    assert op.info()["symmetric_apply"] == 1 and ref.info()["symmetric_apply"] == 0
    assert ref.info()["pair_apply"] == 0
    return op, ref


def both_applies(op, x):
    """(pair apply, three-pass apply) of one symmetric handle on x."""
    yp = op.matvec(dev(x)).cpu().numpy() if op.info()["pair_apply"] else None
    if yp is not None:
        op.set_diag("pair_apply", 0)
    y3 = op.matvec(dev(x)).cpu().numpy()
    if yp is not None:
        op.set_diag("pair_apply", 1)
    return yp, y3


def test_symmetric_apply_multichunk_items(h2d):
    """N = 2^18: level-1 boxes hold ~65K rows > 16384, so stage A' and B' split them into
    row chunks whose partial column sums are reduced by the last chunk (RItem path)."""
    n = 1 << 18
    pts = W.uniform_points(n, 4242)
    op, ref = _sym_pair(h2d, pts, "log", 64, 1e-8)
    for k in range(2):
        x = W.random_vector(n, 900 + k)
        yr = ref.matvec(dev(x)).cpu().numpy()
        for y in both_applies(op, x):
            if y is not None:
                assert rel(y, yr) <= 1e-13


def test_symmetric_apply_wide_panels(h2d, capfd):
    """IMQ with c = 0.05, 256-point leaves and tol 1e-13 makes first-side panels up to ~500
    columns wide (tools/probe_first_side_R.py): B' takes its two-pass (column pass +
    row-dot pass) path for those wider than 256 (share reported by H2D_VERBOSE).  Ranks hit
    the cap there, so the bar is the directed-panel apply of the same factors."""
    import os
    import re
    n = 1 << 14
    pts = W.uniform_points(n, 4343)
    os.environ["H2D_VERBOSE"] = "1"
    try:
        op, ref = _sym_pair(h2d, pts, "imq", 256, 1e-13, c=0.05)
    finally:
        os.environ.pop("H2D_VERBOSE")
    err = capfd.readouterr().err
    share = [float(m) for m in re.findall(r"wide \(R > \d+\) share ([0-9.]+)", err)]
    assert share and share[0] > 0.0, err
    for k in range(2):
        x = W.random_vector(n, 910 + k)
        yr = ref.matvec(dev(x)).cpu().numpy()
        for y in both_applies(op, x):
            if y is not None:
                assert rel(y, yr) <= 1e-13


@pytest.mark.parametrize("case", ["clustered_empty_leaves", "chebyshev_big_leaves", "rbf_phi1", "imq_depth_rule"])
def test_symmetric_apply_cases(h2d, case):
    if case == "clustered_empty_leaves":
        pts, kernel, leaf, kw = W.uniform_points(6000, 77, (-1.0, -1.0), 0.9), "log", 64, {}
    elif case == "chebyshev_big_leaves":
        pts, kernel, leaf, kw = W.chebyshev_grid(70), "log", 500, {}
    elif case == "rbf_phi1":
        pts, kernel, leaf, kw = W.chebyshev_grid(60), "rbf_phi1", 100, {"c": 1e-3, "shift": 3600.0}
    else:
        pts, kernel, leaf, kw = W.uniform_points(9000, 79), "imq", 50, {"c": 0.1, "depth": -2}
    n = pts.shape[0]
    op, ref = _sym_pair(h2d, pts, kernel, leaf, 1e-10, **kw)
    x = W.random_vector(n, 920)
    yr = ref.matvec(dev(x)).cpu().numpy()
    yp, y = both_applies(op, x)
    assert rel(y, yr) <= 1e-13 and (yp is None or rel(yp, yr) <= 1e-13)
    kid = {"log": 0, "imq": 1, "rbf_phi1": 3}[kernel]
    yd = oracle.dense_matvec(pts, x, kid, kw.get("c", 1.0), 1.0, kw.get("shift", 0.0))
    assert rel(y, yd) <= 1e-8


@pytest.mark.parametrize("name", ["c1", "c2"])
@pytest.mark.parametrize("nrhs", [8, 11, 16])
def test_symmetric_multi_rhs(h2d, name, nrhs):
    """Symmetric handles run 8-vector chunks through A' / B' / C' multi (DMMA B' fusing
    T2 = U^T X with Y1 = U T1) and the remainder one vector at a time: every column equals
    its single-vector matvec to 1e-13, in ORIGINAL and TREE order."""
    cfg = W.CONFIGS[name]
    pts = W.config_points(cfg)
    op = build(h2d, cfg, pts)
    X = np.stack([W.config_x(cfg, k) for k in range(nrhs)])
    Y = op.matvec_multi(dev(X)).cpu().numpy()
    for k in range(nrhs):
        assert rel(Y[k], op.matvec(dev(X[k])).cpu().numpy()) <= 1e-13, k
    perm, _ = op.tree()
    Xt = np.ascontiguousarray(X[:, perm])
    Yt = op.matvec_multi(dev(Xt), order="tree").cpu().numpy()
    assert rel(Yt, Y[:, perm]) <= 1e-13


def test_symmetric_multi_rhs_oracle_factors(h2d, tmp_path):
    cfg = W.CONFIGS["c1"]
    pts = W.config_points(cfg)
    orc = oracle.Operator(pts, cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale, shift=cfg.shift,
                          box_lo=cfg.box_lo, box_side=cfg.box_side, symmetric=True)
    path = str(tmp_path / "f.bin")
    orc.save_factors(path)
    op = build(h2d, cfg, pts)
    op.load_factors(path)
    X = np.stack([W.config_x(cfg, k) for k in range(8)])
    Y = op.matvec_multi(dev(X)).cpu().numpy()
    for k in range(8):
        assert rel(Y[k], orc.matvec(X[k])) <= 1e-12, k


def test_symmetric_multi_rhs_wide_panels_fallback(h2d):
    """First-side panels wider than one 448-column tile (IMQ c = 0.05, 256-point leaves,
    tol 1e-13): the handle keeps one vector at a time; results still equal."""
    n = 1 << 14
    pts = W.uniform_points(n, 4343)
    op = h2d.Hodlr2d.build(dev(pts), "imq", 256, 1e-13, c=0.05, box_lo=(-1, -1), box_side=2.0, symmetric=True)
    X = np.stack([W.random_vector(n, 950 + k) for k in range(8)])
    Y = op.matvec_multi(dev(X)).cpu().numpy()
    for k in range(8):
        assert rel(Y[k], op.matvec(dev(X[k])).cpu().numpy()) <= 1e-13


def test_symmetric_gmres(h2d):
    """GMRES on a symmetric-apply handle (the paper's phi_1 system on a Chebyshev grid):
    converges to 1e-10 and recovers the directed handle's solution to the ACA tolerance."""
    pts = W.chebyshev_grid(80)
    n = pts.shape[0]
    kw = dict(c=1e-3, shift=float(n), box_lo=(-1, -1), box_side=2.0, depth=-2)
    sym = h2d.Hodlr2d.build(dev(pts), "rbf_phi1", 100, 1e-12, symmetric=True, **kw)
    dirh = h2d.Hodlr2d.build(dev(pts), "rbf_phi1", 100, 1e-12, **kw)
    assert sym.info()["symmetric_apply"] == 1
    lam = np.random.default_rng(5).uniform(-1.0, 1.0, n)
    f = oracle.dense_matvec(pts, lam, 3, 1e-3, 1.0, float(n))
    xs, its, rr = sym.gmres(dev(f), tol=1e-10)
    xd, _, _ = dirh.gmres(dev(f), tol=1e-10)
    assert rr <= 1e-10 and its < 40
    assert rel(xs.cpu().numpy(), lam) <= 1e-9
    assert rel(xs.cpu().numpy(), xd.cpu().numpy()) <= 1e-9


def test_symmetric_partitioned_multi_rhs(h2d):
    """A symmetric build on a world-2 partition runs the symmetric apply; its multi-RHS path
    (one vector at a time on multi-rank symmetric handles, TREE order) equals its
    single-vector matvecs, and the two ranks reassemble the single-rank symmetric operator."""
    cfg = W.CONFIGS["c1"]
    pts = W.config_points(cfg)
    full = build(h2d, cfg, pts)
    perm, _ = full.tree()
    X = np.stack([W.config_x(cfg, k)[perm] for k in range(21)])
    Yfull = full.matvec_multi(dev(X), order="tree").cpu().numpy()
    parts = []
    for rank in range(2):
        p = build(h2d, cfg, pts, world=2, rank=rank)
        assert p.info()["symmetric_apply"] == 1
        Y = p.matvec_multi(dev(X), order="tree").cpu().numpy()
        for k in (0, 15, 16, 20):
            assert rel(Y[k], p.matvec(dev(X[k]), order="tree").cpu().numpy()) <= 1e-13, k
        parts.append(Y)
    assert rel(np.concatenate(parts, axis=1), Yfull) <= 1e-12


# ------------------------------------------------------------------ pair-local apply

@pytest.mark.parametrize("name,lag", [("c1", None), ("c2", None), ("c2", "0")])
def test_pair_apply_matches_three_pass_and_oracle(h2d, name, lag, tmp_path, monkeypatch):
    """The pair-local apply (opt-in on symmetric single-rank handles: each factor read once;
    small pairs one warp each, medium pairs one CTA, big pairs in row chunks per phase with
    flag-published t1 / t2) computes the same operator as the three-pass apply and, with the
    oracle's symmetric factors, the oracle matvec to <= 1e-12.  lag 0 puts every phase-2 / 3
    chunk right behind its inputs in the queue (the flag waits actually happen)."""
    cfg = W.CONFIGS[name]
    pts = W.config_points(cfg)
    monkeypatch.setenv("H2D_PAIRAPPLY", "1")
    if lag is not None:
        monkeypatch.setenv("H2D_PAIR_LAG", lag)
    op = build(h2d, cfg, pts)
    assert op.info()["pair_apply"] == 1
    for k in range(3):
        x = W.config_x(cfg, k)
        y = op.matvec(dev(x)).cpu().numpy()
        op.set_diag("pair_apply", 0)
        y3 = op.matvec(dev(x)).cpu().numpy()
        op.set_diag("pair_apply", 1)
        assert rel(y, y3) <= 1e-13
        y2 = op.matvec(dev(x)).cpu().numpy()          # accumulation order varies: not bitwise
        assert rel(y2, y) <= 1e-14
    orc = oracle.Operator(pts, cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale, shift=cfg.shift,
                          box_lo=cfg.box_lo, box_side=cfg.box_side, symmetric=True)
    path = str(tmp_path / "s.bin")
    orc.save_factors(path)
    op.load_factors(path)
    assert op.info()["pair_apply"] == 1
    x = W.config_x(cfg, 5)
    assert rel(op.matvec(dev(x)).cpu().numpy(), orc.matvec(x)) <= 1e-12


def test_pair_apply_adaptive_tree(h2d, tmp_path, monkeypatch):
    """Symmetric adaptive handles (R24) run the pair apply too: oracle symmetric adaptive
    factors <= 1e-12, GPU factors <= 10 tol vs dense."""
    pts = W.chebyshev_grid(110)
    monkeypatch.setenv("H2D_PAIRAPPLY", "1")
    kw = dict(box_lo=(-1, -1), box_side=2.0, depth=-3)
    op = h2d.Hodlr2d.build(dev(pts), "rbf_phi1", 48, 1e-12, c=1e-3, shift=12100.0, symmetric=True, **kw)
    assert op.info()["pair_apply"] == 1 and op.info()["adaptive"] == 1
    x = W.random_vector(pts.shape[0], 3)
    yd = oracle.dense_matvec(pts, x, 3, 1e-3, 1.0, 12100.0)
    assert np.linalg.norm(op.matvec(dev(x)).cpu().numpy() - yd) / np.linalg.norm(yd - 12100.0 * x) <= 1e-11
    orc = oracle.Operator(pts, 3, 48, 1e-12, c=1e-3, shift=12100.0, symmetric=True, **kw)
    path = str(tmp_path / "a.bin")
    orc.save_factors(path)
    op.load_factors(path)
    assert rel(op.matvec(dev(x)).cpu().numpy(), orc.matvec(x)) <= 1e-12
