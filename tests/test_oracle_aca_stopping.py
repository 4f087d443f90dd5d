"""The ACA stopping rule (R7: stop after 3 consecutive tolerance hits, drop those 3
terms) on the geometries where a weaker rule nearly failed.

SURVEY §8(c) A7 measured SPEC's one-hit rule at 9.3 x tol on 16384 uniform points with the
IMQ kernel c = 0.05 at tol 1e-6 (the C5 geometry at 1/1024 of its size) — a near-failure
of the north star's 10 x tol bar.  The oracle's operator under R7 is pinned here against
the EXACT dense product on that geometry and on scaled-down C2 (IMQ grid) and C4
(I + h^2 log on the unit-square grid, where the kernel part alone is checked, SURVEY §8(c)
"C4 error check is weak as stated") geometries, asserting a margin below the bar.
"""
import numpy as np
import pytest

import oracle
import workloads as W


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


CASES = {
    # name: (points, kernel id, c, scale, shift, leaf, tol, margin: max err / tol asserted)
    "c5_geometry_16384_imq": (lambda: W.uniform_points(16384, 20220405), 1, 0.05, 1.0, 0.0, 64, 1e-6, 3.0),
    "c2_geometry_64sq_imq_1e-6": (lambda: W.grid_points(64), 1, 0.1, 1.0, 0.0, 64, 1e-6, 3.0),
    "c2_geometry_64sq_imq_1e-8": (lambda: W.grid_points(64), 1, 0.1, 1.0, 0.0, 64, 1e-8, 3.0),
    "c4_geometry_128sq_ie": (lambda: W.grid_points(128, (0.0, 0.0), 1.0), 0, 1.0, 2.0 ** -14, 1.0, 64, 1e-8, 3.0),
}


@pytest.mark.parametrize("name", list(CASES))
def test_r7_stopping_rule_error_margin(name):
    gen, kid, c, scale, shift, leaf, tol, margin = CASES[name]
    pts = gen()
    n = pts.shape[0]
    box = ((0.0, 0.0), 1.0) if name.startswith("c4") else ((-1.0, -1.0), 2.0)
    op = oracle.Operator(pts, kid, leaf, tol, c=c, scale=scale, shift=shift, box_lo=box[0], box_side=box[1])
    worst = 0.0
    for k in range(3):
        x = W.random_vector(n, 7100 + k)
        yd = oracle.dense_matvec(pts, x, kid, c, scale, shift)
        y = op.matvec(x)
        # the kernel part alone (identical to the full error when shift = 0)
        worst = max(worst, float(np.linalg.norm(y - yd) / np.linalg.norm(yd - shift * x)))
    print(f"{name}: max rel-l2 error / tol = {worst / tol:.3f}")
    assert worst <= margin * tol, worst / tol


def test_one_hit_rule_is_weaker_on_the_c5_geometry():
    """The reading R7 exists because fewer hits stop early: on the C5 geometry the one-hit
    untrimmed rule (SPEC's) has a larger error than R7 (the survey measured 9.3 x tol)."""
    gen, kid, c, scale, shift, leaf, tol, _ = CASES["c5_geometry_16384_imq"]
    pts = gen()
    x = W.random_vector(pts.shape[0], 7200)
    yd = oracle.dense_matvec(pts, x, kid, c)
    errs = {}
    for hits, trim in ((1, 0), (3, 3)):
        op = oracle.Operator(pts, kid, leaf, tol, c=c, box_lo=(-1, -1), box_side=2.0, consecutive=hits, trim=trim)
        errs[hits] = rel(op.matvec(x), yd)
    print(f"one hit: {errs[1] / tol:.2f} x tol, R7: {errs[3] / tol:.2f} x tol")
    assert errs[3] < errs[1]
