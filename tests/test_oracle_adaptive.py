"""Pins for the oracle's adaptive (non-balanced) quadtree operator (NEXT N4, R24).

The paper: "the algorithm can also be adapted to a non-balanced or adaptive quadtree with
little modifications" (§4.4).  Reading R24 (options depth = -3): a box is subdivided
iff it holds more than N_max points; a box exists iff its parent is subdivided; at every
level the interaction lists are Eq. eq:ilist restricted to existing boxes, and
the dense blocks are the pairs Y in {X} u E_X of existing boxes at that level of which at
least one is a leaf (an edge-sharing pair of two subdivided boxes recurses, as in Alg. 1).

Independent anchors: every ordered pair (i, j) is covered exactly once (brute force); the
operator equals the balanced one bitwise when every leaf sits at the deepest level; the
dense product within the ACA tolerance; error falling with tol; the scatter test.
"""
import numpy as np
import pytest

import oracle
import workloads as W


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def clustered(n, seed):
    rng = np.random.default_rng(seed)
    a = np.clip(rng.normal((-0.7, -0.6), 0.03, (n // 2, 2)), -1, 1)
    b = rng.uniform(-1, 1, (n - n // 2, 2))
    return np.ascontiguousarray(np.concatenate([a, b]))


def build(pts, nmax, tol=1e-10, kid=0, **kw):
    return oracle.Operator(pts, kid, nmax, tol, box_lo=(-1, -1), box_side=2.0, depth=-3, **kw)


CASES = {
    "clustered_1500": (lambda: clustered(1500, 1), 32),
    "chebyshev_40sq": (lambda: W.chebyshev_grid(40), 25),
    "line_1200": (lambda: np.ascontiguousarray(np.stack([np.linspace(-0.9, 0.9, 1200),
                                                         0.2 * np.linspace(-0.9, 0.9, 1200) ** 2], 1)), 20),
}


@pytest.mark.parametrize("name", list(CASES))
def test_adaptive_tree_invariants(name):
    gen, nmax = CASES[name]
    pts = gen()
    op = build(pts, nmax)
    perm, ls = op.tree()
    k = op.kappa
    lv, bx = op.leaves()
    # leaves tile the points in Morton order, each holds <= N_max points, and every box that
    # holds more is subdivided (a leaf's parent holds more than N_max)
    starts = [int(ls[b << (2 * (k - l))]) for l, b in zip(lv, bx)]
    ends = [int(ls[(b + 1) << (2 * (k - l))]) for l, b in zip(lv, bx)]
    assert starts[0] == 0 and ends[-1] == pts.shape[0]
    assert all(ends[i] == starts[i + 1] for i in range(len(lv) - 1))
    assert max(e - s for s, e in zip(starts, ends)) <= nmax
    for l, b in zip(lv, bx):
        if l > 0:
            p = b >> 2
            cnt = int(ls[(p + 1) << (2 * (k - l + 1))] - ls[p << (2 * (k - l + 1))])
            assert cnt > nmax
    assert len(set(lv.tolist())) > 1            # genuinely non-balanced


@pytest.mark.parametrize("name", list(CASES))
def test_adaptive_blocks_tile_matrix_exactly_once(name):
    gen, nmax = CASES[name]
    pts = gen()
    n = pts.shape[0]
    op = build(pts, nmax)
    perm, ls = op.tree()
    k = op.kappa
    cover = np.zeros((n, n), np.int16)

    def rng(l, b):
        return int(ls[b << (2 * (k - l))]), int(ls[(b + 1) << (2 * (k - l))])

    for l, X, Y in zip(*op.dense_pairs()):
        (a, b), (c, d) = rng(l, X), rng(l, Y)
        cover[a:b, c:d] += 1
    for l in range(1, k + 1):
        off, col = op.op_lists(l)
        for X in range(len(off) - 1):
            for e in range(off[X], off[X + 1]):
                (a, b), (c, d) = rng(l, X), rng(l, int(col[e]))
                cover[a:b, c:d] += 1
    assert cover.min() == 1 and cover.max() == 1


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("kid,c", [(0, 1.0), (1, 0.1), (3, 1e-3)])
def test_adaptive_matvec_vs_dense(name, kid, c):
    gen, nmax = CASES[name]
    pts = gen()
    tol = 1e-10
    op = build(pts, nmax, tol, kid, c=c, shift=float(pts.shape[0]) if kid == 3 else 0.0)
    x = W.random_vector(pts.shape[0], 11)
    yd = oracle.dense_matvec(pts, x, kid, c, 1.0, float(pts.shape[0]) if kid == 3 else 0.0)
    assert rel(op.matvec(x), yd) <= 10 * tol


def test_adaptive_equals_balanced_when_every_leaf_is_deepest():
    # 64 x 64 cell-centre grid, N_max 64: every level-2 box holds 256 points, every level-3
    # box 64 -> all leaves at level 3, the balanced tree of the paper's depth rule (R22)
    pts = W.grid_points(64)
    ad = oracle.Operator(pts, 1, 64, 1e-10, c=0.1, box_lo=(-1, -1), box_side=2.0, depth=-3)
    ba = oracle.Operator(pts, 1, 64, 1e-10, c=0.1, box_lo=(-1, -1), box_side=2.0, depth=-2)
    assert ad.kappa == ba.kappa == 3
    lv, _ = ad.leaves()
    assert np.all(lv == 3)
    for l in range(1, 4):
        assert all(np.array_equal(a, b) for a, b in zip(ad.op_lists(l), ba.op_lists(l)))
    x = W.random_vector(pts.shape[0], 5)
    assert np.array_equal(ad.matvec(x), ba.matvec(x))


def test_adaptive_error_falls_with_tol_and_scatter():
    pts = clustered(1200, 7)
    x = W.random_vector(1200, 8)
    yd = oracle.dense_matvec(pts, x)
    errs = [rel(build(pts, 24, tol).matvec(x), yd) for tol in (1e-4, 1e-7, 1e-10)]
    assert errs[0] > errs[1] > errs[2] and errs[2] <= 1e-9
    op = build(pts, 24, 1e-10)
    for j in range(0, 1200, 97):          # every column reproduced
        e = np.zeros(1200); e[j] = 1.0
        ref = oracle.dense_matvec(pts, e)
        assert np.max(np.abs(op.matvec(e) - ref)) <= 1e-8 * np.max(np.abs(ref))


def test_adaptive_symmetric_mode():
    pts = clustered(1500, 3)
    op = build(pts, 32, 1e-10, symmetric=True)
    x, y = W.random_vector(1500, 1), W.random_vector(1500, 2)
    Ax, Ay = op.matvec(x), op.matvec(y)
    assert abs(y @ Ax - x @ Ay) / (np.linalg.norm(y) * np.linalg.norm(Ax)) < 1e-14
    assert rel(Ax, oracle.dense_matvec(pts, x)) <= 1e-9


def test_adaptive_row_restricted_union():
    pts = clustered(1500, 4)
    full = build(pts, 32)
    perm, ls = full.tree()
    x = W.random_vector(1500, 3)
    yf = full.matvec(x, order="tree")
    lv, bx = full.leaves()
    k = full.kappa
    cut = int(ls[int(bx[len(bx) // 2]) << (2 * (k - int(lv[len(lv) // 2])))])   # a leaf boundary
    acc = np.zeros(1500)
    for a, b in ((0, cut), (cut, 1500)):
        part = build(pts, 32, row_range=(a, b))
        acc[a:b] = part.matvec(x, order="tree")[a:b]
    assert np.array_equal(acc, yf)
