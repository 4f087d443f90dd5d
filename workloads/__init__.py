"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the HODLR2D method (no tree, no lists, no kernel
evaluation, no ACA).  It only draws points and right-hand sides, exactly as stated in
SURVEY.md §8(d) ("Configs as concrete synthetic inputs"):

* numpy ``default_rng(seed)`` (PCG64), fp64, points interleaved ``(x, y)`` in ORIGINAL order;
* points seed ``20220400 + config#``; k-th x seed ``20220500 + 1000*config# + k``;
* grid configs use cell centres, point k = (i, j) with x fastest, ``k = j*G + i``
  (reading R13).

The paper's own workloads are Chebyshev grids (§5.1 "Chebyshev grid");
BASELINE.json replaces them by uniform random points and cell-centre grids; no public
dataset is involved.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

KERNEL_LOG = 0
KERNEL_IMQ = 1
KERNEL_TEST_LOWRANK = 100


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config as data (no method arithmetic)."""
    num: int                 # config number 1..5 (seed offset)
    name: str
    n: int
    points: str              # "uniform" | "grid"
    grid: int                # G for grid configs (N = G*G), else 0
    box_lo: tuple            # root square lower-left corner
    box_side: float          # root square side
    kernel: int              # KERNEL_LOG | KERNEL_IMQ
    c: float                 # IMQ shape parameter
    scale: float             # A = shift*I + scale*K
    shift: float
    leaf_size: int
    tol: float
    x_dist: str              # "uniform" (U(-1,1)) | "normal" (N(0,1))
    matvecs: int             # matvecs the config asks for
    extra: dict = field(default_factory=dict)


CONFIGS = {
    "c1": Config(1, "C1", 4096, "uniform", 0, (-1.0, -1.0), 2.0, KERNEL_LOG, 1.0, 1.0, 0.0,
                 64, 1e-10, "uniform", 10),
    "c2": Config(2, "C2", 65536, "grid", 256, (-1.0, -1.0), 2.0, KERNEL_IMQ, 0.1, 1.0, 0.0,
                 64, 1e-10, "normal", 10),
    "c3": Config(3, "C3", 1 << 20, "uniform", 0, (-1.0, -1.0), 2.0, KERNEL_LOG, 1.0, 1.0, 0.0,
                 64, 1e-8, "uniform", 100),
    # h = 1/2048 cell side; h^2 = 2^-22 quadrature weight
    "c4": Config(4, "C4", 1 << 22, "grid", 2048, (0.0, 0.0), 1.0, KERNEL_LOG, 1.0, 2.0 ** -22, 1.0,
                 64, 1e-8, "normal", 100),
    "c5": Config(5, "C5", 1 << 24, "uniform", 0, (-1.0, -1.0), 2.0, KERNEL_IMQ, 0.05, 1.0, 0.0,
                 128, 1e-6, "normal", 50),
}


def uniform_points(n: int, seed: int, lo=(-1.0, -1.0), side: float = 2.0) -> np.ndarray:
    """n points i.i.d. uniform in the square [lo, lo+side]^2, shape (n, 2), fp64, C order."""
    rng = np.random.default_rng(seed)
    u = rng.uniform(0.0, 1.0, size=(n, 2))
    pts = np.empty((n, 2), dtype=np.float64)
    pts[:, 0] = lo[0] + side * u[:, 0]
    pts[:, 1] = lo[1] + side * u[:, 1]
    # keep every point inside the closed root square despite rounding of lo + side*u
    np.clip(pts[:, 0], lo[0], lo[0] + side, out=pts[:, 0])
    np.clip(pts[:, 1], lo[1], lo[1] + side, out=pts[:, 1])
    return pts


def grid_points(g: int, lo=(-1.0, -1.0), side: float = 2.0) -> np.ndarray:
    """Cell centres of a g x g grid over [lo, lo+side]^2; point k=(i,j) with x fastest."""
    h = side / g
    i = np.arange(g, dtype=np.float64)
    xs = lo[0] + (i + 0.5) * h
    ys = lo[1] + (i + 0.5) * h
    pts = np.empty((g * g, 2), dtype=np.float64)
    pts[:, 0] = np.tile(xs, g)
    pts[:, 1] = np.repeat(ys, g)
    return pts


def config_points(cfg: Config) -> np.ndarray:
    if cfg.points == "grid":
        return grid_points(cfg.grid, cfg.box_lo, cfg.box_side)
    return uniform_points(cfg.n, 20220400 + cfg.num, cfg.box_lo, cfg.box_side)


def config_x(cfg: Config, k: int, n: int | None = None) -> np.ndarray:
    """k-th right-hand side of a config (ORIGINAL point order)."""
    n = cfg.n if n is None else n
    rng = np.random.default_rng(20220500 + 1000 * cfg.num + k)
    if cfg.x_dist == "uniform":
        return rng.uniform(-1.0, 1.0, size=n)
    return rng.standard_normal(size=n)


def random_vector(n: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal(size=n)


def lowrank_gh(m: int, n: int, r: int, seed: int):
    """Seeded Gaussian factors G (m x r), H (n x r) for an exactly rank-r test matrix G H^T."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((m, r)), rng.standard_normal((n, r))


def chebyshev_grid(m: int, lo=(-1.0, -1.0), side: float = 2.0) -> np.ndarray:
    """m x m tensor grid of first-kind Chebyshev nodes cos((2k+1)pi/(2m)) mapped to the box,
    x fastest (the paper's sqrt(N) x sqrt(N) Chebyshev grid; first kind per
    SPEC's stated choice)."""
    k = np.arange(m, dtype=np.float64)
    t = np.cos((2.0 * k + 1.0) * np.pi / (2.0 * m))        # in (-1, 1)
    xs = lo[0] + (t + 1.0) * 0.5 * side
    ys = lo[1] + (t + 1.0) * 0.5 * side
    pts = np.empty((m * m, 2), dtype=np.float64)
    pts[:, 0] = np.tile(xs, m)
    pts[:, 1] = np.repeat(ys, m)
    return pts
