"""GPU parity of the paper's application (NEXT N3) through the C ABI: the RBF kernels
phi_1 / phi_2 in the build and the matvec, and hodlr2d_gmres (P:917-920,
P:1020-1048) against the oracle and the dense solution.

Bars: oracle factors loaded -> rel-l2 <= 1e-12 vs the oracle matvec; GPU factors ->
<= 10 * aca_tol vs the dense product; GMRES -> the paper's ~1e-10 solution accuracy
(bar 1e-9) and the oracle GMRES's iteration count +-2.  The Chebyshev grids cluster points
in the corners: pairs closer than a = 0.001 (the second branch of phi_1 / phi_2) and leaves
> 96 points (the generic P2P path) both occur.
"""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

A_RBF = 1e-3


@pytest.fixture(scope="module")
def h2d():
    import paper_2204_05536_b200 as m
    m.lib()
    return m


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def build_pair(h2d, kernel_name, m, tol, n_max=500):
    pts = W.chebyshev_grid(m)
    n = pts.shape[0]
    kid = oracle.KERNELS[kernel_name]
    orc = oracle.Operator(pts, kid, n_max, tol, c=A_RBF, scale=1.0, shift=float(n),
                          box_lo=(-1, -1), box_side=2.0)
    gpu = h2d.Hodlr2d.build(dev(pts), kid, n_max, tol, c=A_RBF, scale=1.0, shift=float(n),
                            box_lo=(-1, -1), box_side=2.0)
    return pts, orc, gpu


def test_chebyshev_grid_exercises_both_branches():
    pts = W.chebyshev_grid(100)           # used by test_rbf_oracle_factors_parity[100]
    d = np.hypot(pts[0, 0] - pts[1, 0], pts[0, 1] - pts[1, 1])
    assert d < A_RBF                      # corner neighbours closer than a


@pytest.mark.parametrize("kernel_name", ["rbf_phi1", "rbf_phi2"])
@pytest.mark.parametrize("m", [50, 100])
def test_rbf_oracle_factors_parity(h2d, kernel_name, m, tmp_path):
    pts, orc, gpu = build_pair(h2d, kernel_name, m, 1e-12)
    path = str(tmp_path / "f.bin")
    orc.save_factors(path)
    gpu.load_factors(path)
    x = W.random_vector(pts.shape[0], 31 + m)
    y = gpu.matvec(dev(x)).cpu().numpy()
    assert rel(y, orc.matvec(x)) <= 1e-12


@pytest.mark.parametrize("kernel_name", ["rbf_phi1", "rbf_phi2"])
def test_rbf_gpu_factors_vs_dense(h2d, kernel_name):
    tol = 1e-10
    pts, orc, gpu = build_pair(h2d, kernel_name, 64, tol, n_max=64)
    n = pts.shape[0]
    x = W.random_vector(n, 77)
    y = gpu.matvec(dev(x)).cpu().numpy()
    yd = oracle.dense_matvec(pts, x, oracle.KERNELS[kernel_name], c=A_RBF, scale=1.0, shift=float(n))
    assert rel(y, yd) <= 10 * tol
    # the kernel part alone (the beta = N shift dominates ||A x||)
    ys = y - n * x
    yds = yd - n * x
    assert rel(ys, yds) <= 10 * tol


@pytest.mark.parametrize("kernel_name", ["rbf_phi1", "rbf_phi2"])
def test_gpu_gmres_rbf_paper_accuracy(h2d, kernel_name):
    pts, orc, gpu = build_pair(h2d, kernel_name, 50, 1e-12)
    n = pts.shape[0]
    lam = np.random.default_rng(1048).uniform(-1.0, 1.0, n)
    f = oracle.dense_matvec(pts, lam, oracle.KERNELS[kernel_name], c=A_RBF, scale=1.0, shift=float(n))
    lam_hat, its, rr = gpu.gmres(dev(f), tol=1e-10, restart=30)
    lam_hat = lam_hat.cpu().numpy()
    assert gpu.gmres_converged and rr < 1e-10
    assert rel(lam_hat, lam) < 1e-9                       # P:1048 "of the order of 1e-10"
    _, its_o, _ = oracle.gmres(orc.matvec, f, tol=1e-10, restart=30)
    assert abs(its - its_o) <= 2
    # the reported residual is the true one of the returned x (GPU matvec)
    r = f - gpu.matvec(dev(lam_hat)).cpu().numpy()
    assert np.linalg.norm(r) / np.linalg.norm(f) == pytest.approx(rr, rel=1e-3, abs=1e-14)


def test_gpu_gmres_host_pointers_restart_and_edges(h2d):
    pts, orc, gpu = build_pair(h2d, "rbf_phi1", 40, 1e-12)
    n = pts.shape[0]
    rng = np.random.default_rng(5)
    f = rng.standard_normal(n)
    x_dev, its_d, rr_d = gpu.gmres(dev(f), tol=1e-11, restart=30)
    x_host, its_h, rr_h = gpu.gmres(f.copy(), tol=1e-11, restart=30)       # numpy = host pointers
    assert its_d == its_h and np.array_equal(x_dev.cpu().numpy(), x_host)  # deterministic
    x_r, its_r, rr_r = gpu.gmres(dev(f), tol=1e-11, restart=4)             # many restarts
    assert rr_r < 1e-11 and rel(x_r.cpu().numpy(), x_host) < 1e-9
    # dense solution of the HODLR2D system (oracle operator as a dense matrix, small N)
    x_ref, _, _ = oracle.gmres(orc.matvec, f, tol=1e-13, restart=200)
    assert rel(x_host, x_ref) < 1e-9
    # b = 0 -> x = 0 with no iterations
    z, its0, rr0 = gpu.gmres(dev(np.zeros(n)))
    assert its0 == 0 and rr0 == 0.0 and not z.any()
    # not converged -> warning status, residual still reported
    x2, its2, rr2 = gpu.gmres(dev(f), tol=1e-14, restart=3, max_iter=2)
    assert its2 == 2 and not gpu.gmres_converged and rr2 > 1e-14


def test_paper_depth_rule_gpu_matches_oracle(h2d):
    """depth = -2 (the paper's max-occupancy rule, R22): same depth and bit-identical tree."""
    for pts, n_max in ((W.chebyshev_grid(100), 500), (W.uniform_points(3000, 4, (-1.0, -1.0), 0.3), 100)):
        orc = oracle.Operator(pts, 0, n_max, 1e-8, box_lo=(-1, -1), box_side=2.0, depth=-2)
        gpu = h2d.Hodlr2d.build(dev(pts), "log", n_max, 1e-8, box_lo=(-1, -1), box_side=2.0, depth=-2)
        assert gpu.info()["kappa"] == orc.kappa
        p_g, ls_g = gpu.tree()
        p_o, ls_o = orc.tree()
        assert np.array_equal(p_g, p_o) and np.array_equal(ls_g, ls_o)
        x = W.random_vector(pts.shape[0], 9)
        yd = oracle.dense_matvec(pts, x, 0)
        assert rel(gpu.matvec(dev(x)).cpu().numpy(), yd) <= 1e-7


def test_paper_table_rbf_phi1_row_250000_gpu(h2d):
    """Table tab:ker1_init, row N = 250000: r_m 59, CR 0.013 — reproduced by the GPU
    build with the paper's depth rule (R22) to r_m 57, CR 0.0127; the GMRES solve of the
    paper's system converges to its 1e-10 residual in a handful of iterations."""
    pts = W.chebyshev_grid(500)
    n = pts.shape[0]
    op = h2d.Hodlr2d.build(dev(pts), "rbf_phi1", 500, 1e-12, c=A_RBF, scale=1.0, shift=float(n),
                           box_lo=(-1, -1), box_side=2.0, depth=-2)
    inf = op.info()
    assert abs(inf["rank_max"] - 59) <= 4, inf["rank_max"]
    assert abs(inf["compression_ratio"] - 0.013) <= 0.05 * 0.013, inf["compression_ratio"]
    lam = dev(np.random.default_rng(3).uniform(-1.0, 1.0, n))
    lam_hat, its, rr = op.gmres(op.matvec(lam), tol=1e-10)
    assert rr < 1e-10 and its < 30
    assert float(torch.linalg.norm(lam_hat - lam) / torch.linalg.norm(lam)) < 1e-9


def test_gpu_gmres_argument_errors(h2d):
    """GMRES needs a single-rank handle and positive tol / restart / max_iter: H2D_EINVAL,
    and the handle stays usable."""
    pts = W.uniform_points(3000, 61)
    kw = dict(box_lo=(-1, -1), box_side=2.0, shift=3000.0)
    part = h2d.Hodlr2d.build(dev(pts), "log", 64, 1e-10, world=2, rank=0, **kw)
    b = dev(W.random_vector(3000, 62))
    with pytest.raises(h2d.Hodlr2dError) as e:
        part.gmres(b, tol=1e-10)
    assert e.value.code == h2d.H2D_EINVAL
    op = h2d.Hodlr2d.build(dev(pts), "log", 64, 1e-10, **kw)
    for kwargs in (dict(tol=0.0), dict(tol=1e-10, restart=0), dict(tol=1e-10, max_iter=0)):
        with pytest.raises(h2d.Hodlr2dError) as e:
            op.gmres(b, **kwargs)
        assert e.value.code == h2d.H2D_EINVAL
    x, its, rr = op.gmres(b, tol=1e-10)
    assert rr <= 1e-10
