"""Stream-ordered host-buffer matvec (hodlr2d_matvec_async / hodlr2d_wait, include/hodlr2d.h):
the same operation as hodlr2d_matvec_ex (Alg. 2) with the host copies
pipelined under the kernels of neighbouring calls.

Bars: every result bitwise equal to hodlr2d_matvec_ex on the same x (same kernels, same
schedule); many calls in flight on distinct pinned buffers each land in their own y; TREE
order and device pointers; symmetric handles; pageable buffers and LOCAL order refused with
H2D_EINVAL before anything is enqueued; synchronous calls unaffected afterwards.
"""

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def h2d():
    import paper_2204_05536_b200 as m
    m.lib()
    return m


def build(h2d, cfg, **kw):
    pts = torch.from_numpy(np.ascontiguousarray(W.config_points(cfg))).cuda()
    return h2d.Hodlr2d.build(pts, cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale, shift=cfg.shift,
                             box_lo=cfg.box_lo, box_side=cfg.box_side, **kw)


@pytest.mark.parametrize("symmetric", [False, True])
def test_async_pipeline_bitwise_equal_to_sync(h2d, symmetric):
    cfg = W.CONFIGS["c2"]
    op = build(h2d, cfg, symmetric=symmetric)
    n = cfg.n
    K = 7   # more calls in flight than staging slots
    xs = [torch.from_numpy(W.random_vector(n, 900 + k)).pin_memory() for k in range(K)]
    ys = [torch.full((n,), np.nan, dtype=torch.float64).pin_memory() for _ in range(K)]
    torch.cuda.synchronize()
    for k in range(K):
        op.matvec_async(xs[k], ys[k])
    op.wait()
    for k in range(K):
        ref = op.matvec(xs[k].cuda()).cpu()
        assert torch.equal(ys[k], ref), k
    # reusing two y buffers alternately (the bench pattern): the last two results stand
    y2 = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
    for k in range(K):
        op.matvec_async(xs[k], y2[k % 2])
    op.wait()
    assert torch.equal(y2[(K - 1) % 2], ys[K - 1]) and torch.equal(y2[(K - 2) % 2], ys[K - 2])
    # synchronous host-buffer calls afterwards still work (separate staging)
    yp = np.empty(n)
    op.matvec_raw(xs[0].numpy().ctypes.data, yp.ctypes.data, h2d.ORDER_ORIGINAL)
    assert np.array_equal(yp, ys[0].numpy())


def test_async_tree_order_and_device_pointers(h2d):
    cfg = W.CONFIGS["c1"]
    op = build(h2d, cfg)
    perm, _ = op.tree()
    n = cfg.n
    xt = torch.from_numpy(W.random_vector(n, 31)[perm].copy())
    ref = op.matvec(xt.cuda(), order="tree").cpu()
    yh = torch.empty(n, dtype=torch.float64).pin_memory()
    op.matvec_async(xt.pin_memory(), yh, order="tree")
    xd, yd = xt.cuda(), torch.empty(n, dtype=torch.float64, device="cuda")
    op.matvec_async(xd, yd, order="tree")            # device x and y
    yh2 = torch.empty(n, dtype=torch.float64).pin_memory()
    op.matvec_async(xd, yh2, order="tree")           # device x, host y
    op.wait()
    assert torch.equal(yh, ref) and torch.equal(yd.cpu(), ref) and torch.equal(yh2, ref)


def test_async_rejects_pageable_and_local(h2d):
    cfg = W.CONFIGS["c1"]
    op = build(h2d, cfg)
    n = cfg.n
    L = h2d.lib()
    xp, yp = np.zeros(n), np.zeros(n)
    assert L.hodlr2d_matvec_async(op._h, xp.ctypes.data, yp.ctypes.data, h2d.ORDER_ORIGINAL) == h2d.H2D_EINVAL
    assert "pinned" in L.hodlr2d_last_error().decode()
    xh = torch.zeros(n, dtype=torch.float64).pin_memory()
    yh = torch.zeros(n, dtype=torch.float64).pin_memory()
    assert L.hodlr2d_matvec_async(op._h, xh.data_ptr(), yh.data_ptr(), h2d.ORDER_LOCAL) == h2d.H2D_EINVAL
    assert L.hodlr2d_matvec_async(op._h, None, yh.data_ptr(), h2d.ORDER_ORIGINAL) == h2d.H2D_EINVAL
    assert L.hodlr2d_matvec_async(None, xh.data_ptr(), yh.data_ptr(), h2d.ORDER_ORIGINAL) == h2d.H2D_EINVAL
    assert L.hodlr2d_wait(None) == h2d.H2D_EINVAL
    with pytest.raises(ValueError):
        op.matvec_async(torch.zeros(n, dtype=torch.float64), yh)
    assert L.hodlr2d_wait(op._h) == 0
