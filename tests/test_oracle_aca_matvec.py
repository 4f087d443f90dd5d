"""Pins for the oracle's kernels, ACA (R7), matvec (Alg. 2) and dense product (R10).

Independent anchors: hand values of the kernels, exact recovery of synthetic rank-r
matrices, SVD truncation, the kappa = 0 special case (single dense block), the
scatter / linearity properties, error falling as the tolerance tightens, the paper's own
Table tab:1byr rows (tests/golden/), and the bitwise union of row-restricted operators.
"""
import math
import os
import struct

import numpy as np
import pytest

import oracle
import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


# ---------------------------------------------------------------- kernels (hand values)

def test_kernel_hand_values():
    assert oracle.kernel(0, (0, 0), (1, 0)) == 0.0                 # log 1 = 0
    assert oracle.kernel(0, (0.3, 0.2), (0.3, 0.2)) == 0.0         # K(0) = 0
    assert oracle.kernel(0, (0, 0), (math.e, 0)) == pytest.approx(1.0, abs=1e-15)
    assert oracle.kernel(0, (0, 0), (3, 4)) == pytest.approx(math.log(5.0), abs=1e-15)
    assert oracle.kernel(1, (0, 0), (0, 0), c=0.1) == 1.0          # IMQ(0) = 1
    assert oracle.kernel(1, (0, 0), (0.1, 0), c=0.1) == pytest.approx(2 ** -0.5, abs=1e-15)
    assert oracle.kernel(1, (0, 0), (0, 0.3), c=0.1) == pytest.approx(10 ** -0.5, abs=1e-15)
    assert oracle.kernel(2, (0, 0), (2, 0)) == 0.5                 # 1/r, S:183 example
    assert oracle.kernel(2, (0, 0), (0, 0)) == 0.0
    # symmetry
    for kid in (0, 1, 2, 100):
        a, b = (0.1, -0.7), (0.45, 0.3)
        assert oracle.kernel(kid, a, b, c=0.1, test_rank=4) == oracle.kernel(kid, b, a, c=0.1, test_rank=4)


# ---------------------------------------------------------------- ACA (R7)

@pytest.mark.parametrize("m,n,r", [(64, 64, 1), (64, 64, 3), (64, 64, 8), (64, 64, 15),
                                   (256, 1024, 1), (256, 1024, 8), (200, 75, 15)])
def test_aca_exact_rank_recovery(m, n, r):
    G, H = W.lowrank_gh(m, n, r, seed=100 + r + m)
    A = G @ H.T
    U, V, trunc = oracle.aca_dense(A, 1e-10)
    assert U.shape[1] == r and not trunc                           # exact rank with 2 hits + trim
    assert rel(U @ V.T, A) <= 1e-13                                # rounding of r pivoted steps


def test_aca_untrimmed_rank_is_r_plus_hits():
    G, H = W.lowrank_gh(64, 64, 5, seed=5)
    A = G @ H.T
    U, V, _ = oracle.aca_dense(A, 1e-10, consecutive=2, trim=0)
    assert U.shape[1] == 7
    U, V, _ = oracle.aca_dense(A, 1e-10, consecutive=1, trim=0)
    assert U.shape[1] == 6


def test_aca_zero_and_degenerate_blocks():
    U, V, _ = oracle.aca_dense(np.zeros((50, 50)), 1e-10)
    assert U.shape[1] == 0
    a = np.random.default_rng(1).standard_normal((1, 40))
    U, V, _ = oracle.aca_dense(a, 1e-10)                            # 1-row block: rank <= 1, exact
    assert U.shape[1] == 1 and np.allclose(U @ V.T, a, rtol=0, atol=1e-15)
    # exactly-zero rows are skipped (zero pivots, R7 step 3) and the next row is tried ...
    A = np.zeros((10, 12)); A[2, :] = np.arange(1, 13)
    U, V, _ = oracle.aca_dense(A, 1e-10)
    assert U.shape[1] == 1 and rel(U @ V.T, A) <= 1e-15
    # ... but three consecutive zero pivots stop the iteration (S:247 rule, R7)
    A = np.zeros((10, 12)); A[7, :] = np.arange(1, 13)
    U, V, _ = oracle.aca_dense(A, 1e-10)
    assert U.shape[1] == 0


def test_aca_truncation_flag():
    A = np.random.default_rng(3).standard_normal((40, 40))
    U, V, trunc = oracle.aca_dense(A, 1e-12, max_rank=5)
    assert trunc and U.shape[1] == 5


def kernel_block(kid, P, Q, c=1.0):
    return np.array([[oracle.kernel(kid, p, q, c=c) for q in Q] for p in P])


@pytest.mark.parametrize("kid,c,tol", [(0, 1.0, 1e-8), (0, 1.0, 1e-12), (1, 0.1, 1e-10), (2, 1.0, 1e-12)])
def test_aca_kernel_block_vs_svd(kid, c, tol):
    # two well-separated clusters (offset class (2,0)) and a vertex-sharing pair (1,1)
    rng = np.random.default_rng(7)
    P = rng.uniform(0, 1, (120, 2))
    for off in [(2.0, 0.0), (1.0, 1.0)]:
        Q = rng.uniform(0, 1, (150, 2)) + np.array(off)
        A = kernel_block(kid, P, Q, c)
        U, V, _ = oracle.aca_dense(A, tol)
        s = np.linalg.svd(A, compute_uv=False)
        r_eps = int(np.sum(s / s[0] > tol))                        # eps-rank
        assert rel(U @ V.T, A) <= 10 * tol
        assert U.shape[1] <= r_eps + 10


# ---------------------------------------------------------------- matvec (Alg. 2)

def test_kappa0_is_dense():
    pts = W.uniform_points(50, 9)
    x = W.random_vector(50, 1)
    for kid, c, sc, sh in [(0, 1.0, 1.0, 0.0), (1, 0.1, 1.0, 0.0), (0, 1.0, 0.25, 1.0)]:
        op = oracle.Operator(pts, kid, 64, 1e-10, c=c, scale=sc, shift=sh, box_lo=(-1, -1), box_side=2.0)
        assert op.kappa == 0
        assert rel(op.matvec(x), oracle.dense_matvec(pts, x, kid, c, sc, sh)) <= 1e-14


def test_dense_matvec_shift_and_scale_definition():
    pts = W.uniform_points(40, 2)
    x = W.random_vector(40, 2)
    y0 = oracle.dense_matvec(pts, x, 0)
    y1 = oracle.dense_matvec(pts, x, 0, scale=0.25, shift=1.0)
    assert np.allclose(y1, 0.25 * y0 + x, rtol=0, atol=1e-14)      # A = shift I + scale K
    y = oracle.dense_matvec(pts[:2], np.array([1.0, 0.0]), 1, c=0.1)
    d = np.hypot(*(pts[0] - pts[1]))
    assert y[0] == 1.0 and y[1] == pytest.approx(1 / math.sqrt(1 + (d / 0.1) ** 2), rel=1e-15)


@pytest.mark.parametrize("kid,c,scale,shift", [(0, 1.0, 1.0, 0.0), (1, 0.05, 1.0, 0.0), (2, 1.0, 1.0, 0.0),
                                               (3, 1e-3, 1.0, 4096.0), (4, 1e-3, 1.0, 4096.0),
                                               (0, 1.0, 2.0 ** -22, 1.0), (1, 0.3, -0.5, 2.0),
                                               (100, 1.0, 1.0, 0.0)])
def test_dense_rows_pinned_to_dense_matvec(kid, c, scale, shift):
    """oracle_dense_rows is the reference of every full-size GPU check (sampled rows at
    N = 2^20 .. 2^24, R10).  Pinned here to the full dense product (itself pinned to hand
    values, the kappa = 0 operator and the shift/scale definition) at N = 4096 with coincident
    points (K(0) := K0 by distance, R8): every row, in seeded random order and with repeats,
    must equal the corresponding entry of dense_matvec up to summation rounding, and a few
    rows must equal an independent numpy evaluation of A_ij = scale K(|p_i - p_j|) + shift
    delta_ij."""
    pts = W.uniform_points(4096, 404)
    pts[4000:4010] = pts[100:110]                                   # coincident points
    x = W.random_vector(4096, 405)
    y = oracle.dense_matvec(pts, x, kid, c, scale, shift, test_rank=3)
    rows = np.random.default_rng(406).permutation(np.concatenate([np.arange(4096), [5, 5, 4095]]))
    yr = oracle.dense_rows(pts, x, rows, kid, c, scale, shift, test_rank=3)
    assert np.max(np.abs(yr - y[rows])) <= 1e-13 * np.max(np.abs(y))
    # independent evaluation of a few rows straight from the kernel definitions
    some = np.array([0, 100, 4000, 4095, 2048])
    d = pts[some, None, :] - pts[None, :, :]
    r = np.hypot(d[..., 0], d[..., 1])
    safe = np.where(r > 0, r, 1.0)
    if kid == 0:
        K = np.where(r > 0, np.log(safe), 0.0)
    elif kid == 1:
        K = 1.0 / np.sqrt(1.0 + (r / c) ** 2)
    elif kid == 2:
        K = np.where(r > 0, 1.0 / safe, 0.0)
    elif kid == 3:   # phi_1
        K = np.where(r >= c, np.log(safe) / math.log(c), (safe * np.log(safe) - 1) / (c * math.log(c) - 1))
        K = np.where(r > 0, K, 0.0)
    elif kid == 4:   # phi_2
        K = np.where(r >= c, c / safe, r / c)
        K = np.where(r > 0, K, 0.0)
    else:            # test kernel: sum_s cos((s+1) p.x + 0.5 s p.y) cos(...) (hodlr2d.h)
        s = np.arange(3)
        fp = np.cos((s[None, :] + 1) * pts[some, 0:1] + 0.5 * s[None, :] * pts[some, 1:2])
        fq = np.cos((s[None, :] + 1) * pts[:, 0:1] + 0.5 * s[None, :] * pts[:, 1:2])
        K = fp @ fq.T
    A = scale * K
    A[np.arange(len(some)), some] += shift
    ref = A @ x
    assert np.max(np.abs(oracle.dense_rows(pts, x, some, kid, c, scale, shift, test_rank=3) - ref)) \
        <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_scatter_and_linearity():
    n = 600
    pts = W.uniform_points(n, 21)
    op = oracle.Operator(pts, 0, 64, 1e-10, box_lo=(-1, -1), box_side=2.0)
    assert op.kappa == 2
    # scatter test on e_j: each column reproduced -> each pair counted exactly once
    for j in range(0, n, 7):
        e = np.zeros(n); e[j] = 1.0
        col = op.matvec(e)
        ref = oracle.dense_matvec(pts, e)
        assert np.max(np.abs(col - ref)) <= 100 * 1e-10 * np.max(np.abs(ref))
    x, z = W.random_vector(n, 1), W.random_vector(n, 2)                 # linearity
    assert rel(op.matvec(x + 2.0 * z), op.matvec(x) + 2.0 * op.matvec(z)) <= 1e-13


@pytest.mark.parametrize("cfg_name", ["c1"])
def test_config_vs_dense(cfg_name):
    cfg = W.CONFIGS[cfg_name]
    pts = W.config_points(cfg)
    op = oracle.Operator(pts, cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale,
                         shift=cfg.shift, box_lo=cfg.box_lo, box_side=cfg.box_side)
    for k in range(3):
        x = W.config_x(cfg, k)
        assert rel(op.matvec(x), oracle.dense_matvec(pts, x, cfg.kernel, cfg.c, cfg.scale, cfg.shift)) <= 10 * cfg.tol


def test_error_falls_as_tol_tightens():
    # north_star: "matvec error falls as aca_tol is tightened"; C1 geometry
    cfg = W.CONFIGS["c1"]
    pts = W.config_points(cfg)
    x = W.config_x(cfg, 0)
    yd = oracle.dense_matvec(pts, x)
    errs, sizes = [], []
    for tol in (1e-4, 1e-6, 1e-8, 1e-10, 1e-12):
        op = oracle.Operator(pts, 0, 64, tol, box_lo=cfg.box_lo, box_side=cfg.box_side)
        e = rel(op.matvec(x), yd)
        assert e <= 10 * tol
        errs.append(e)
        sizes.append(op.factor_values())
    assert all(errs[i + 1] < errs[i] for i in range(len(errs) - 1))
    assert all(sizes[i + 1] > sizes[i] for i in range(len(sizes) - 1))


def test_imq_grid_vs_dense_and_congruent_blocks():
    # 64x64 cell-centre grid, IMQ c=0.1 (C2 geometry at 1/16 size), kappa = 3
    pts = W.grid_points(64)
    tol = 1e-10
    op = oracle.Operator(pts, 1, 64, tol, c=0.1, box_lo=(-1, -1), box_side=2.0)
    assert op.kappa == 3
    x = W.random_vector(pts.shape[0], 4)
    assert rel(op.matvec(x), oracle.dense_matvec(pts, x, 1, 0.1)) <= 10 * tol
    # congruent blocks (same level, same signed offset) are exact translates -> same rank
    for l in range(1, op.kappa + 1):
        off, col = oracle.level_lists(l)
        r, _ = op.ranks(l)
        by_off = {}
        for X in range(1 << (2 * l)):
            for e in range(off[X], off[X + 1]):
                Y = int(col[e])
                cx = sum(((X >> (2 * b)) & 1) << b for b in range(l)); cy = sum(((X >> (2 * b + 1)) & 1) << b for b in range(l))
                dx = sum(((Y >> (2 * b)) & 1) << b for b in range(l)); dy = sum(((Y >> (2 * b + 1)) & 1) << b for b in range(l))
                by_off.setdefault((dx - cx, dy - cy), set()).add(int(r[e]))
        assert all(len(v) == 1 for v in by_off.values()), by_off


def test_operator_near_symmetric():
    cfg = W.CONFIGS["c1"]
    pts = W.config_points(cfg)
    op = oracle.Operator(pts, 0, 64, 1e-10, box_lo=cfg.box_lo, box_side=cfg.box_side)
    x, y = W.random_vector(cfg.n, 5), W.random_vector(cfg.n, 6)
    v = W.random_vector(cfg.n, 7)
    for _ in range(20):                                      # power iteration for ||A||
        v = op.matvec(v); v /= np.linalg.norm(v)
    nrm = np.linalg.norm(op.matvec(v))
    asym = abs(x @ op.matvec(y) - y @ op.matvec(x)) / (np.linalg.norm(x) * np.linalg.norm(y) * nrm)
    assert asym <= 10 * 1e-10


def test_row_restricted_union_is_bitwise_full():
    # multi-GPU emulation: rows served by contiguous Morton ranges
    cfg = W.CONFIGS["c1"]
    pts = W.config_points(cfg)
    full = oracle.Operator(pts, 0, 64, 1e-10, box_lo=cfg.box_lo, box_side=cfg.box_side)
    x = W.config_x(cfg, 1)
    yf = full.matvec(x, order="tree")
    n = cfg.n
    cuts = [0, 1000, 1024, 2500, 4096]
    acc = np.zeros(n)
    for a, b in zip(cuts[:-1], cuts[1:]):
        part = oracle.Operator(pts, 0, 64, 1e-10, box_lo=cfg.box_lo, box_side=cfg.box_side, row_range=(a, b))
        yp = part.matvec(x, order="tree")
        assert np.all(yp[:a] == 0) and np.all(yp[b:] == 0)
        acc[a:b] = yp[a:b]
    assert np.array_equal(acc, yf)


def test_factor_file_roundtrip(tmp_path):
    cfg = W.CONFIGS["c1"]
    pts = W.config_points(cfg)
    op = oracle.Operator(pts, 0, 64, 1e-10, box_lo=cfg.box_lo, box_side=cfg.box_side)
    path = tmp_path / "c1.h2df"
    op.save_factors(path)
    perm, ls = op.tree()
    buf = open(path, "rb").read()
    assert buf[:8] == b"H2DFAC01"
    o = 8
    N, = struct.unpack_from("<q", buf, o); o += 8
    kappa, kid = struct.unpack_from("<ii", buf, o); o += 8
    o += 56 + 8
    fperm = np.frombuffer(buf, np.int32, N, o); o += 4 * N
    assert N == cfg.n and kappa == op.kappa and np.array_equal(fperm, perm)
    # rebuild the low-rank part of the matvec from the file alone (TREE order)
    x = W.config_x(cfg, 2)
    xt = x[perm]
    y_lr = np.zeros(N)
    for l in range(1, kappa + 1):
        nb, = struct.unpack_from("<q", buf, o); o += 8
        off, col = oracle.level_lists(l)
        assert nb == off[-1]
        sh = 2 * (kappa - l)
        ranks, _ = op.ranks(l)
        for X in range(1 << (2 * l)):
            for e in range(off[X], off[X + 1]):
                Y = int(col[e])
                r0, r1 = ls[X << sh], ls[(X + 1) << sh]
                c0, c1 = ls[Y << sh], ls[(Y + 1) << sh]
                r, = struct.unpack_from("<i", buf, o); o += 4
                assert r == ranks[e]
                U = np.frombuffer(buf, np.float64, (r1 - r0) * r, o).reshape(r, r1 - r0).T; o += 8 * (r1 - r0) * r
                V = np.frombuffer(buf, np.float64, (c1 - c0) * r, o).reshape(r, c1 - c0).T; o += 8 * (c1 - c0) * r
                y_lr[r0:r1] += U @ (V.T @ xt[c0:c1])
    assert o == len(buf)
    # the dense part is what remains; compare the total against the oracle within rounding
    y_dense = np.zeros(N)
    noff, ncol = oracle.near_lists(kappa)
    P = pts[perm]
    for X in range(1 << (2 * kappa)):
        for Y in ncol[noff[X]:noff[X + 1]]:
            d = P[ls[X]:ls[X + 1], None, :] - P[None, ls[Y]:ls[Y + 1], :]
            rr = np.hypot(d[..., 0], d[..., 1])
            K = np.where(rr > 0, np.log(np.where(rr > 0, rr, 1.0)), 0.0)
            y_dense[ls[X]:ls[X + 1]] += K @ xt[ls[Y]:ls[Y + 1]]
    assert rel(y_lr + y_dense, op.matvec(xt, order="tree")) <= 1e-13
    assert rel(y_lr + y_dense, op.matvec(x)[perm]) <= 1e-13


# ---------------------------------------------------------------- paper anchor

def load_golden(name):
    d = {}
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        k, v = line.split(None, 1)
        d[k] = v
    return d


def test_paper_table_1byr_row_10000():
    g = load_golden("paper_tab_1byr_n10000.txt")
    m = int(g["grid_m"])
    pts = W.chebyshev_grid(m)
    n = pts.shape[0]
    assert n == int(g["N"])
    op = oracle.Operator(pts, oracle.KERNELS[g["kernel"]], int(g["n_max"]), float(g["tol"]),
                         box_lo=(-1, -1), box_side=2.0)
    r_m = max(int(op.ranks(l)[0].max()) for l in range(1, op.kappa + 1))
    perm, ls = op.tree()
    sz = np.diff(ls)
    off, col = oracle.near_lists(op.kappa)
    dense = sum(int(sz[X]) * int(sz[col[e]]) for X in range(len(sz)) for e in range(off[X], off[X + 1]))
    mem_gb = (op.factor_values() + dense) * 8 / 1e9
    assert abs(r_m - int(g["r_m"])) <= 0.2 * int(g["r_m"])
    assert abs(mem_gb - float(g["memory_gb"])) <= 0.2 * float(g["memory_gb"])
    # eps_r = max_i |b^ - b|_i / |b|_i over ten input vectors; psi ~ U(0,1) (R17)
    eps_r = 0.0
    for k in range(10):
        x = np.random.default_rng(1000 + k).uniform(0.0, 1.0, n)
        b = oracle.dense_matvec(pts, x, 2)
        eps_r = max(eps_r, float(np.max(np.abs(op.matvec(x) - b) / np.abs(b))))
    assert eps_r <= 10 * float(g["eps_r"])


# ---------------------------------------------------------------- symmetric mode (NEXT N1, R23)

def test_symmetric_mode_oracle():
    """One ACA per unordered pair: (Y, X) holds exactly the swapped factors of (X, Y); the
    operator is then symmetric to rounding (the directed one only to O(tol)); accuracy vs
    the dense product stays within the 10 tol bar; row-restricted symmetric operators union
    bitwise to the full one."""
    cfg = W.CONFIGS["c1"]
    pts = W.config_points(cfg)
    kw = dict(box_lo=cfg.box_lo, box_side=cfg.box_side)
    op = oracle.Operator(pts, cfg.kernel, cfg.leaf_size, cfg.tol, symmetric=True, **kw)
    for l in range(1, op.kappa + 1):
        off, col = oracle.level_lists(l)
        for X in range(len(off) - 1):
            for e in range(off[X], off[X + 1]):
                Y = col[e]
                t = off[Y] + int(np.searchsorted(col[off[Y]:off[Y + 1]], X))
                U, V = op.block(l, e)
                U2, V2 = op.block(l, t)
                assert np.array_equal(U, V2) and np.array_equal(V, U2)
    x, y = W.config_x(cfg, 0), W.random_vector(cfg.n, 17)
    Ax, Ay = op.matvec(x), op.matvec(y)
    norm_a = np.linalg.norm(Ax) / np.linalg.norm(x)
    asym = abs(y @ Ax - x @ Ay) / (np.linalg.norm(x) * np.linalg.norm(y) * norm_a)
    assert asym < 1e-14
    assert rel(Ax, oracle.dense_matvec(pts, x, cfg.kernel)) <= 10 * cfg.tol
    # IMQ on the C2 grid geometry (smaller)
    g = W.grid_points(64)
    op2 = oracle.Operator(g, 1, 64, 1e-10, c=0.1, box_lo=(-1, -1), box_side=2.0, symmetric=True)
    xg = W.random_vector(g.shape[0], 3)
    assert rel(op2.matvec(xg), oracle.dense_matvec(g, xg, 1, c=0.1)) <= 1e-9
    # row-restricted symmetric operators (two halves) union bitwise to the full operator
    perm, ls = op.tree()
    half = int(ls[len(ls) // 2])
    y_full = op.matvec(x[perm], order="tree")
    parts = [oracle.Operator(pts, cfg.kernel, cfg.leaf_size, cfg.tol, symmetric=True, row_range=r, **kw)
             for r in ((0, half), (half, cfg.n))]
    y0 = parts[0].matvec(x[perm], order="tree")
    y1 = parts[1].matvec(x[perm], order="tree")
    assert np.array_equal(np.concatenate([y0[:half], y1[half:]]), y_full)
