"""Binding and ABI error paths on the GPU: vector lengths checked before the C
call, stream ordering when torch's current stream differs from the handle's, GMRES restart
bound, diagnostics switches by name, pageable host buffers staged by the library."""
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


@pytest.fixture(scope="module")
def op(h2d):
    pts = W.uniform_points(3000, 12)
    return h2d.Hodlr2d.build(torch.from_numpy(pts).cuda(), "log", 64, 1e-10, box_lo=(-1, -1), box_side=2.0,
                             shift=3000.0), pts


def test_vector_lengths_checked(h2d, op):
    o, pts = op
    with pytest.raises(ValueError):
        o.matvec(torch.zeros(2999, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        o.matvec(torch.zeros(3000, dtype=torch.float64, device="cuda"),
                 out=torch.zeros(10, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        o.matvec_multi(torch.zeros(3, 2999, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        o.gmres(torch.zeros(5, dtype=torch.float64, device="cuda"))


def test_other_stream_ordering(h2d, op):
    """x produced on a side stream, matvec called under it: the binding orders the handle's
    stream after torch's current stream and back (same result as on the default stream)."""
    o, pts = op
    x = W.random_vector(3000, 4)
    ref = o.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        xd = torch.from_numpy(x).cuda(non_blocking=False) * 1.0
        y = o.matvec(xd)
        y2 = y * 1.0
    torch.cuda.synchronize()
    assert np.array_equal(y2.cpu().numpy(), ref)


def test_gmres_restart_bound_and_diag_names(h2d, op):
    o, pts = op
    b = torch.ones(3000, dtype=torch.float64, device="cuda")
    with pytest.raises(h2d.Hodlr2dError) as e:
        o.gmres(b, restart=70000)
    assert e.value.code == h2d.H2D_EINVAL
    with pytest.raises(h2d.Hodlr2dError):
        o.set_diag("no_such_switch", 1)
    with pytest.raises(h2d.Hodlr2dError):      # directed handle: no pair apply built
        o.set_diag("pair_apply", 1)
    o.set_diag("p2p_serial", 1)
    x = W.random_vector(3000, 5)
    y1 = o.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    o.set_diag("p2p_serial", 0)
    o.set_diag("p2p_place", 1)   # near field beside stage B
    y2 = o.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    o.set_diag("p2p_place", 0)   # beside stage A
    y0 = o.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(y0, y1)
    assert np.array_equal(y0, y2)
    with pytest.raises(h2d.Hodlr2dError):
        o.set_diag("p2p_place", 2)
    o.set_diag("p2p_place", -1)  # timed placement: calls 1-2 beside A, 3-4 beside B, then the faster
    for _ in range(8):
        assert np.array_equal(o.matvec(torch.from_numpy(x).cuda()).cpu().numpy(), y0)
    o.set_diag("p2p_place", 0)


def test_pageable_host_buffers(h2d, op):
    """numpy (pageable) x / y go through the library's pinned staging: same bits as device
    buffers, for matvec, matvec_multi and gmres."""
    o, pts = op
    x = W.random_vector(3000, 6)
    yd = o.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(o.matvec(x.copy()), yd)
    X = np.stack([x, W.random_vector(3000, 7)])
    Yd = o.matvec_multi(torch.from_numpy(X).cuda()).cpu().numpy()
    assert np.array_equal(o.matvec_multi(X.copy()), Yd)
    xs, its, rr = o.gmres(yd.copy(), tol=1e-12)
    assert rr < 1e-12 and np.linalg.norm(xs - x) / np.linalg.norm(x) < 1e-9
    assert np.linalg.norm(yd - oracle.dense_matvec(pts, x, 0, 1.0, 1.0, 3000.0)) <= 1e-9 * np.linalg.norm(yd)
