"""Oracle pins for the paper's application (NEXT N3): the RBF kernels phi_1 / phi_2 of
§5.2, GMRES and the RBF interpolation solve.

Pins (none of them re-types the oracle's own formula):
  * kernel hand values at points where the piecewise definitions reduce to closed numbers,
    and continuity at r = a;
  * GMRES against numpy's dense LU solve (the plain definition of the solution);
  * Table tab:ker1_init row N = 10000 (r_m, CR) for phi_1 (tests/golden/);
  * phi_2 = a * (1/r) for r >= a: a relative ACA tolerance is scale invariant, so the phi_2
    operator has exactly the ranks of the 1/r operator on the same tree (R21;
    the paper's 78 vs 113 for 1/r is not reproducible under that reading) and its CR is
    checked against Table tab:ker2_init;
  * the paper's solution accuracy ||lambda - lambda_hat|| / ||lambda|| ~ 1e-10.
"""
import math
import os

import numpy as np
import pytest

import oracle
import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")
A_RBF = 1e-3          # a = 0.001


def load_golden(name):
    d = {}
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            k, v = line.split(None, 1)
            d[k] = v
    return d


def test_rbf_kernel_hand_values():
    a = A_RBF
    k1 = lambda r: oracle.kernel(3, (0.0, 0.0), (r, 0.0), c=a)   # noqa: E731
    k2 = lambda r: oracle.kernel(4, (0.0, 0.0), (0.0, r), c=a)   # noqa: E731
    assert k1(1.0) == 0.0                                  # log 1 = 0
    assert k1(a) == pytest.approx(1.0, abs=1e-15)          # log a / log a
    assert k1(0.5 * a) == pytest.approx((0.5 * a * math.log(0.5 * a) - 1) / (a * math.log(a) - 1), abs=1e-15)
    assert k1(a * (1 - 1e-9)) == pytest.approx(1.0, abs=1e-8)   # continuous at r = a
    assert k1(0.1) == pytest.approx(1.0 / 3.0, abs=1e-15)  # log 0.1 / log 0.001
    assert k2(2 * a) == pytest.approx(0.5, abs=1e-15)
    assert k2(0.5 * a) == pytest.approx(0.5, abs=1e-15)
    assert k2(a) == pytest.approx(1.0, abs=1e-15)
    assert k1(0.0) == 0.0 and k2(0.0) == 0.0               # diagonal excluded (Eq. eq:ker)
    for kid in (3, 4):
        p, q = (0.1, -0.7), (0.45, 0.3)
        assert oracle.kernel(kid, p, q, c=a) == oracle.kernel(kid, q, p, c=a)


def test_oracle_gmres_matches_dense_solve():
    rng = np.random.default_rng(7)
    n = 300
    A = n * np.eye(n) + rng.standard_normal((n, n)) * 3.0
    b = rng.standard_normal(n)
    x_ref = np.linalg.solve(A, b)
    for restart in (5, 30, 400):
        x, its, rr = oracle.gmres(lambda v: A @ v, b, tol=1e-12, restart=restart)
        assert rr < 1e-12
        assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) < 1e-11
        assert its <= 400
    # the true residual it reports is the residual of the returned x
    x, its, rr = oracle.gmres(lambda v: A @ v, b, tol=1e-6, restart=3, max_iter=4)
    assert rr == pytest.approx(np.linalg.norm(b - A @ x) / np.linalg.norm(b), rel=1e-12)
    assert its == 4
    # b = 0 -> x = 0 without iterations
    x, its, rr = oracle.gmres(lambda v: A @ v, np.zeros(n))
    assert its == 0 and not x.any()


def rbf_operator(kernel_name, m, tol, n_max=500):
    pts = W.chebyshev_grid(m)
    n = pts.shape[0]
    return pts, oracle.Operator(pts, oracle.KERNELS[kernel_name], n_max, tol, c=A_RBF, scale=1.0,
                                shift=float(n), box_lo=(-1, -1), box_side=2.0)


def cr_of(op, n):
    perm, ls = op.tree()
    sz = np.diff(ls)
    off, col = oracle.near_lists(op.kappa)
    dense = sum(int(sz[X]) * int(sz[col[e]]) for X in range(len(sz)) for e in range(off[X], off[X + 1]))
    return (op.factor_values() + dense) / n ** 2


def test_paper_table_rbf_phi1_row_10000():
    g = load_golden("paper_tab_rbf_phi1_n10000.txt")
    pts, op = rbf_operator(g["kernel"], int(g["grid_m"]), float(g["tol"]), int(g["n_max"]))
    n = pts.shape[0]
    assert n == int(g["N"])
    r_m = max(int(op.ranks(l)[0].max()) for l in range(1, op.kappa + 1))
    assert abs(r_m - int(g["r_m"])) <= 0.25 * int(g["r_m"]), r_m
    cr = cr_of(op, n)
    assert abs(cr - float(g["cr"])) <= 0.25 * float(g["cr"]), cr


def test_rbf_phi2_scale_invariance_and_cr_row_10000():
    g = load_golden("paper_tab_rbf_phi2_n10000.txt")
    pts, op2 = rbf_operator(g["kernel"], int(g["grid_m"]), float(g["tol"]), int(g["n_max"]))
    n = pts.shape[0]
    op_r = oracle.Operator(pts, oracle.KERNELS["one_over_r"], int(g["n_max"]), float(g["tol"]),
                           box_lo=(-1, -1), box_side=2.0)
    same = tot = 0
    rm1 = rm2 = 0
    for l in range(1, op2.kappa + 1):
        r2, _ = op2.ranks(l)
        r1, _ = op_r.ranks(l)
        assert np.all(np.abs(r2 - r1) <= 3)              # rounding near-ties of the stop at 1e-12
        same += int(np.sum(r2 == r1))
        tot += r2.size
        rm1, rm2 = max(rm1, int(r1.max())), max(rm2, int(r2.max()))
    assert same >= 0.98 * tot, (same, tot)               # ranks of a/r == ranks of 1/r
    assert abs(rm1 - rm2) <= 2
    cr = cr_of(op2, n)
    assert abs(cr - float(g["cr"])) <= 0.25 * float(g["cr"]), cr


@pytest.mark.parametrize("kernel_name", ["rbf_phi1", "rbf_phi2"])
def test_paper_rbf_solution_error(kernel_name):
    """random lambda, f = A lambda by the explicit (dense) product, HODLR2D-GMRES
    (ACA 1e-12, residual 1e-10) recovers lambda to ~1e-10 relative."""
    pts, op = rbf_operator(kernel_name, 50, 1e-12)
    n = pts.shape[0]
    lam = np.random.default_rng(1048).uniform(-1.0, 1.0, n)
    f = oracle.dense_matvec(pts, lam, oracle.KERNELS[kernel_name], c=A_RBF, scale=1.0, shift=float(n))
    lam_hat, its, rr = oracle.gmres(op.matvec, f, tol=1e-10, restart=30)
    assert rr < 1e-10
    err = np.linalg.norm(lam - lam_hat) / np.linalg.norm(lam)
    assert err < 1e-9, err                                 # "of the order of 1e-10"
    assert its < 60


# ---------------------------------------------------------------- the paper's depth rule (R22)

def test_paper_depth_rule_definition():
    """depth = -2: the smallest kappa whose fullest leaf holds <= N_max points."""
    for pts, n_max in ((W.chebyshev_grid(100), 500), (W.uniform_points(5000, 3), 64),
                       (W.uniform_points(3000, 4, (-1.0, -1.0), 0.3), 100)):
        op = oracle.Operator(pts, 0, n_max, 1e-6, box_lo=(-1, -1), box_side=2.0, depth=-2)
        k = op.kappa
        _, _, ls = oracle.tree(pts, (-1, -1), 2.0, k)
        assert int(np.diff(ls).max()) <= n_max
        if k > 0:
            _, _, ls1 = oracle.tree(pts, (-1, -1), 2.0, k - 1)
            assert int(np.diff(ls1).max()) > n_max


def test_paper_depth_rule_reproduces_tables():
    """With the paper's own depth rule the N = 10000 rows are reproduced closely: kappa = 4
    (R1 gives 3); phi_1 CR 0.1536 vs 0.154 and r_m 41 vs 42 (Table tab:ker1_init);
    1/r memory 0.215 vs 0.23 GB and r_m 103 vs 113 (Table tab:1byr_init)."""
    g = load_golden("paper_tab_rbf_phi1_n10000.txt")
    pts = W.chebyshev_grid(int(g["grid_m"]))
    n = pts.shape[0]
    op = oracle.Operator(pts, oracle.KERNELS["rbf_phi1"], int(g["n_max"]), float(g["tol"]), c=A_RBF,
                         scale=1.0, shift=float(n), box_lo=(-1, -1), box_side=2.0, depth=-2)
    assert op.kappa == 4
    r_m = max(int(op.ranks(l)[0].max()) for l in range(1, op.kappa + 1))
    assert abs(r_m - int(g["r_m"])) <= 2, r_m
    assert abs(cr_of(op, n) - float(g["cr"])) <= 0.03 * float(g["cr"]), cr_of(op, n)
    g1 = load_golden("paper_tab_1byr_n10000.txt")
    op1 = oracle.Operator(pts, oracle.KERNELS["one_over_r"], int(g1["n_max"]), float(g1["tol"]),
                          box_lo=(-1, -1), box_side=2.0, depth=-2)
    r_m1 = max(int(op1.ranks(l)[0].max()) for l in range(1, op1.kappa + 1))
    mem = cr_of(op1, n) * n * n * 8 / 1e9
    assert abs(r_m1 - int(g1["r_m"])) <= 0.1 * int(g1["r_m"]), r_m1
    assert abs(mem - float(g1["memory_gb"])) <= 0.1 * float(g1["memory_gb"]), mem
