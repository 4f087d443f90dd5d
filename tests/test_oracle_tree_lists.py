"""Pins for the oracle's quadtree (R1-R4) and relation / interaction lists (Defs 4.1-4.5).

Every check here is independent of the oracle's own code path: brute force over all box
pairs with a different formulation (shared-corner counting), the closed form of the
interaction list, the paper's printed counts (|I_C| <= 15, <= 5 dense blocks), the
partition identity and SPEC's small worked examples.
"""
import itertools

import numpy as np
import pytest

import oracle
import workloads as W


def morton(ix, iy):
    c = 0
    for b in range(16):
        c |= ((ix >> b) & 1) << (2 * b)
        c |= ((iy >> b) & 1) << (2 * b + 1)
    return c


def coords(code):
    x = y = 0
    for b in range(16):
        x |= ((code >> (2 * b)) & 1) << b
        y |= ((code >> (2 * b + 1)) & 1) << b
    return x, y


# ---------------------------------------------------------------- tree (R1-R4)

def test_depth_rule_configs():
    # R1: smallest kappa with N <= leaf_size * 4^kappa -> 3/5/7/8/9
    exp = {"c1": 3, "c2": 5, "c3": 7, "c4": 8, "c5": 9}
    for k, cfg in W.CONFIGS.items():
        assert oracle.depth(cfg.n, cfg.leaf_size) == exp[k]
    assert oracle.depth(1, 500) == 0          # S:61 degenerate tree
    assert oracle.depth(64, 64) == 0
    assert oracle.depth(65, 64) == 1


def test_four_points_one_per_quadrant():
    # 4 points, one per quadrant of [-1,1]^2, one per leaf at kappa=1.
    pts = np.array([[0.5, 0.5], [-0.5, 0.5], [-0.5, -0.5], [0.5, -0.5]])  # TR, TL, BL, BR
    codes, perm, ls = oracle.tree(pts, (-1.0, -1.0), 2.0, 1)
    assert list(np.diff(ls)) == [1, 1, 1, 1]
    # Morton children: 0 BL, 1 BR, 2 TL, 3 TR (R4)
    assert list(perm) == [2, 3, 1, 0]
    assert list(codes) == [0, 1, 2, 3]


def test_split_lines_and_top_boundary():
    # half-open boxes, closed global top/right edge (R3)
    pts = np.array([[0.0, 0.0], [1.0, 1.0], [-1.0, -1.0], [0.5, -1.0], [1.0, -1.0]])
    codes, perm, ls = oracle.tree(pts, (-1.0, -1.0), 2.0, 2)
    by_orig = {int(p): int(c) for p, c in zip(perm, codes)}
    assert coords(by_orig[0]) == (2, 2)      # split line x=0 -> upper box
    assert coords(by_orig[1]) == (3, 3)      # top-right corner clamped
    assert coords(by_orig[2]) == (0, 0)
    assert coords(by_orig[3]) == (3, 0)      # x = 0.5 lies on the level-2 split x=0.5
    assert coords(by_orig[4]) == (3, 0)


def test_out_of_box_and_nonfinite_rejected():
    with pytest.raises(ValueError, match="outside"):
        oracle.tree(np.array([[0.0, 0.0], [1.5, 0.0]]), (-1.0, -1.0), 2.0, 2)
    with pytest.raises(ValueError, match="non-finite"):
        oracle.tree(np.array([[0.0, np.nan]]), (-1.0, -1.0), 2.0, 2)
    with pytest.raises(ValueError):
        oracle.Operator(np.zeros((0, 2)))


@pytest.mark.parametrize("n,kappa,seed", [(1000, 3, 1), (4096, 3, 2), (20000, 5, 3)])
def test_tree_invariants_random(n, kappa, seed):
    lo, side = (-1.0, -1.0), 2.0
    pts = W.uniform_points(n, seed, lo, side)
    codes, perm, ls = oracle.tree(pts, lo, side, kappa)
    # index conservation
    assert sorted(perm.tolist()) == list(range(n))
    assert ls[0] == 0 and ls[-1] == n and np.all(np.diff(ls) >= 0)
    # codes nondecreasing; ties keep input order (stable sort)
    assert np.all(np.diff(codes.astype(np.int64)) >= 0)
    same = np.diff(codes.astype(np.int64)) == 0
    assert np.all(np.diff(perm)[same] > 0)
    # leaf ranges agree with codes
    for b in range(1 << (2 * kappa)):
        assert np.all(codes[ls[b]:ls[b + 1]] == b)
    # geometric containment, independent of the quantisation formula
    h = side / (1 << kappa)
    cx = np.array([coords(int(c))[0] for c in codes])
    cy = np.array([coords(int(c))[1] for c in codes])
    P = pts[perm]
    assert np.all(lo[0] + cx * h <= P[:, 0] + 1e-15) and np.all(P[:, 0] <= lo[0] + (cx + 1) * h + 1e-15)
    assert np.all(lo[1] + cy * h <= P[:, 1] + 1e-15) and np.all(P[:, 1] <= lo[1] + (cy + 1) * h + 1e-15)
    # parent range = union of child ranges at every level
    for l in range(kappa):
        sh = 2 * (kappa - l)
        for b in range(1 << (2 * l)):
            s, e = ls[b << sh], ls[(b + 1) << sh]
            assert np.all((codes[s:e] >> sh) == b)
            kids = [(ls[(4 * b + c) << (sh - 2)], ls[(4 * b + c + 1) << (sh - 2)]) for c in range(4)]
            assert kids[0][0] == s and kids[-1][1] == e
            assert all(kids[i][1] == kids[i + 1][0] for i in range(3))


def test_grid_configs_exactly_64_per_leaf():
    cfg = W.CONFIGS["c2"]
    pts = W.config_points(cfg)
    k = oracle.depth(cfg.n, cfg.leaf_size)
    _, _, ls = oracle.tree(pts, cfg.box_lo, cfg.box_side, k)
    assert np.all(np.diff(ls) == 64)


# ---------------------------------------------------------------- relations (Defs 4.1-4.5)

def brute_relation(a, b):
    """Independent formulation: count shared corners of two same-level unit boxes."""
    if a == b:
        return "self"
    ca = {(a[0] + dx, a[1] + dy) for dx in (0, 1) for dy in (0, 1)}
    cb = {(b[0] + dx, b[1] + dy) for dx in (0, 1) for dy in (0, 1)}
    s = len(ca & cb)
    return {2: "edge", 1: "vertex", 0: "wellsep"}[s]


def brute_sets(level):
    side = 1 << level
    boxes = [morton(x, y) for y in range(side) for x in range(side)]
    rel = {}
    for c in boxes:
        E, V, Wl = set(), set(), set()
        for d in boxes:
            r = brute_relation(coords(c), coords(d))
            {"edge": E, "vertex": V, "wellsep": Wl}.get(r, set()).add(d)
        rel[c] = (E, V, Wl)
    return boxes, rel


@pytest.mark.parametrize("level", [1, 2, 3, 4])
def test_literal_definitions_bruteforce(level):
    boxes, rel = brute_sets(level)
    _, prel = brute_sets(level - 1) if level >= 2 else (None, None)
    off, col = oracle.level_lists(level)
    for c in boxes:
        E, V, Wl = rel[c]
        # partition identity P:684: {C} ∪ E ∪ V ∪ W = all clusters of the level, disjoint
        assert len(E) + len(V) + len(Wl) + 1 == len(boxes)
        assert len(E) <= 4 and len(V) <= 4               # Defs 4.1, 4.2
        parent = c >> 2
        clan = {(parent << 2) | k for k in range(4)} - {c}
        if level >= 2:
            for e in prel[parent][0]:
                clan |= {(e << 2) | k for k in range(4)}
        il = sorted((clan & V) | (clan & Wl))               # Eq. eq:ilist
        oE, oclan, oil = oracle.box_sets(level, c)
        assert sorted(E) == sorted(oE)
        assert sorted(clan) == sorted(oclan)
        assert il == list(oil)
        assert il == list(col[off[c]:off[c + 1]])
        # closed form: manhattan(parents) <= 1 and manhattan >= 2
        cx, cy = coords(c)
        cf = []
        for d in boxes:
            dx, dy = coords(d)
            px, py = coords(parent)
            qx, qy = coords(d >> 2)
            if abs(px - qx) + abs(py - qy) <= 1 and abs(cx - dx) + abs(cy - dy) >= 2:
                cf.append(d)
        assert sorted(cf) == il


@pytest.mark.parametrize("level", range(1, 8))
def test_list_counts_and_bounds(level):
    off, col = oracle.level_lists(level)
    deg = np.diff(off)
    # directed block count 15*4^l - 28*2^l and max 15
    assert off[-1] == 15 * 4 ** level - 28 * 2 ** level
    assert deg.max() <= 15
    if level >= 3:
        assert deg.max() == 15
    # symmetry: D in I_C <=> C in I_D
    pairs = set()
    for c in range(len(deg)):
        for d in col[off[c]:off[c + 1]]:
            pairs.add((c, int(d)))
    assert all((d, c) in pairs for (c, d) in pairs)
    # lists ascending
    for c in range(len(deg)):
        seg = col[off[c]:off[c + 1]]
        assert np.all(np.diff(seg) > 0)


def test_level1_diagonal_sibling():
    # level-1 node 0 -> interaction list {2} in the paper's numbering = Morton child 3
    off, col = oracle.level_lists(1)
    assert [list(col[off[b]:off[b + 1]]) for b in range(4)] == [[3], [2], [1], [0]]
    E, clan, il = oracle.box_sets(1, 0)
    assert sorted(E) == [1, 2] and sorted(clan) == [1, 2, 3] and il == [3]


@pytest.mark.parametrize("kappa", [0, 1, 2, 5, 7])
def test_near_field_counts(kappa):
    off, col = oracle.near_lists(kappa)
    deg = np.diff(off)
    assert off[-1] == 5 * 4 ** kappa - 4 * 2 ** kappa    # self + edge sharers
    assert deg.max() <= 5                                # P:871 "maximum of five dense matrices"
    for b in range(len(deg)):
        assert b in col[off[b]:off[b + 1]]


def tiling_count(n, kappa, seed):
    pts = W.uniform_points(n, seed)
    _, _, ls = oracle.tree(pts, (-1.0, -1.0), 2.0, kappa)
    cover = np.zeros((n, n), np.int32)
    for l in range(1, kappa + 1):
        off, col = oracle.level_lists(l)
        sh = 2 * (kappa - l)
        for X in range(1 << (2 * l)):
            for Y in col[off[X]:off[X + 1]]:
                cover[ls[X << sh]:ls[(X + 1) << sh], ls[int(Y) << sh]:ls[(int(Y) + 1) << sh]] += 1
    off, col = oracle.near_lists(kappa)
    for X in range(1 << (2 * kappa)):
        for Y in col[off[X]:off[X + 1]]:
            cover[ls[X]:ls[X + 1], ls[Y]:ls[Y + 1]] += 1
    return cover


@pytest.mark.parametrize("n,kappa", [(300, 2), (1024, 3), (700, 4)])
def test_blocks_tile_matrix_exactly_once(n, kappa):
    # every ordered pair (i, j) covered exactly once (north_star)
    cover = tiling_count(n, kappa, 11 + kappa)
    assert cover.min() == 1 and cover.max() == 1
