"""ctypes harness over the HODLR2D CPU oracle (oracle/hodlr2d_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hodlr2d_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

KERNELS = {"log": 0, "imq": 1, "one_over_r": 2, "rbf_phi1": 3, "rbf_phi2": 4, "test_lowrank": 100}


def compile_oracle(force: bool = False) -> str:
    """g++ -O2 -ffp-contract=off (no fast-math) -fopenmp; R14."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-shared", "-fPIC", "-o", tmp, _SRC]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            compile_oracle()
            L = C.CDLL(_LIB)
            d, i, i64, vp = C.c_double, C.c_int, C.c_int64, C.c_void_p
            L.oracle_last_error.restype = C.c_char_p
            L.oracle_depth.argtypes = [i64, i]
            L.oracle_kernel.argtypes = [i, d, i, d, d, d, d]
            L.oracle_kernel.restype = d
            L.oracle_tree.argtypes = [vp, i64, d, d, d, i, vp, vp, vp]
            L.oracle_box_sets.argtypes = [i, i, vp, vp, vp, vp, vp, vp]
            L.oracle_classify.argtypes = [i, i, i, i]
            L.oracle_level_lists.argtypes = [i, vp, vp]
            L.oracle_level_lists.restype = i64
            L.oracle_near_lists.argtypes = [i, vp, vp]
            L.oracle_near_lists.restype = i64
            L.oracle_aca_dense.argtypes = [vp, i, i, d, i, i, i, vp, vp, vp, vp]
            L.oracle_dense_matvec.argtypes = [vp, i64, i, d, d, d, i, vp, vp]
            L.oracle_dense_rows.argtypes = [vp, i64, i, d, d, d, i, vp, vp, i64, vp]
            L.oracle_build.argtypes = [vp, i64, i, d, d, d, i, i, d, d, d, d, i, i, i, i, i64, i64, i]
            L.oracle_build.restype = vp
            L.oracle_destroy.argtypes = [vp]
            L.oracle_kappa.argtypes = [vp]
            L.oracle_build_seconds.argtypes = [vp]
            L.oracle_build_seconds.restype = d
            L.oracle_get_tree.argtypes = [vp, vp, vp]
            L.oracle_num_blocks.argtypes = [vp, i]
            L.oracle_num_blocks.restype = i64
            L.oracle_get_ranks.argtypes = [vp, i, vp, vp]
            L.oracle_get_block.argtypes = [vp, i, i64, vp, vp, vp, vp, vp]
            L.oracle_factor_values.argtypes = [vp]
            L.oracle_factor_values.restype = i64
            L.oracle_matvec.argtypes = [vp, vp, vp, i]
            L.oracle_save_factors.argtypes = [vp, C.c_char_p]
            L.oracle_set_threads.argtypes = [i]
            L.oracle_leaves.argtypes = [vp, vp, vp]
            L.oracle_leaves.restype = i64
            L.oracle_op_level_lists.argtypes = [vp, i, vp, vp]
            L.oracle_op_level_lists.restype = i64
            L.oracle_dense_pairs.argtypes = [vp, vp, vp, vp]
            L.oracle_dense_pairs.restype = i64
            _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def set_threads(t: int) -> None:
    lib().oracle_set_threads(int(t))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def last_error() -> str:
    return lib().oracle_last_error().decode()


def depth(n: int, leaf_size: int) -> int:
    return int(lib().oracle_depth(n, leaf_size))


def kernel(kernel_id: int, p, q, c: float = 1.0, test_rank: int = 1) -> float:
    return float(lib().oracle_kernel(kernel_id, c, test_rank, p[0], p[1], q[0], q[1]))


def tree(points: np.ndarray, lo, side: float, kappa: int):
    """(codes in tree order u32, perm i32, leaf_start i32)."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    n = pts.shape[0]
    codes = np.zeros(n, np.uint32)
    perm = np.zeros(n, np.int32)
    ls = np.zeros((1 << (2 * kappa)) + 1, np.int32)
    rc = lib().oracle_tree(_p(pts), n, lo[0], lo[1], side, kappa, _p(codes), _p(perm), _p(ls))
    if rc != 0:
        raise ValueError(f"oracle_tree rc={rc}: {last_error()}")
    return codes, perm, ls


def box_sets(level: int, box: int):
    E = np.zeros(8, np.int32); clan = np.zeros(32, np.int32); il = np.zeros(32, np.int32)
    nE = C.c_int(); nc = C.c_int(); ni = C.c_int()
    lib().oracle_box_sets(level, box, _p(E), C.byref(nE), _p(clan), C.byref(nc), _p(il), C.byref(ni))
    return list(E[:nE.value]), list(clan[:nc.value]), list(il[:ni.value])


def classify(a, b) -> int:
    return int(lib().oracle_classify(a[0], a[1], b[0], b[1]))


def level_lists(level: int):
    tot = lib().oracle_level_lists(level, None, None)
    off = np.zeros((1 << (2 * level)) + 1, np.int32)
    col = np.zeros(tot, np.int32)
    lib().oracle_level_lists(level, _p(off), _p(col))
    return off, col


def near_lists(kappa: int):
    tot = lib().oracle_near_lists(kappa, None, None)
    off = np.zeros((1 << (2 * kappa)) + 1, np.int32)
    col = np.zeros(tot, np.int32)
    lib().oracle_near_lists(kappa, _p(off), _p(col))
    return off, col


def aca_dense(A: np.ndarray, tol: float, max_rank: int = 128, consecutive: int = 3, trim: int = 3):
    A = np.asfortranarray(A, dtype=np.float64)
    m, n = A.shape
    kmax = min(m, n, max_rank)
    U = np.zeros(m * kmax + 1); V = np.zeros(n * kmax + 1)
    r = C.c_int(); tr = C.c_int()
    Af = A.ravel(order="F")
    lib().oracle_aca_dense(_p(Af), m, n, tol, max_rank, consecutive, trim, _p(U), _p(V),
                           C.byref(r), C.byref(tr))
    k = r.value
    return U[: m * k].reshape(k, m).T.copy(), V[: n * k].reshape(k, n).T.copy(), bool(tr.value)


def dense_matvec(points, x, kernel_id=0, c=1.0, scale=1.0, shift=0.0, test_rank=1):
    pts = np.ascontiguousarray(points, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros_like(x)
    lib().oracle_dense_matvec(_p(pts), pts.shape[0], kernel_id, c, scale, shift, test_rank, _p(x), _p(y))
    return y


def dense_rows(points, x, rows, kernel_id=0, c=1.0, scale=1.0, shift=0.0, test_rank=1):
    pts = np.ascontiguousarray(points, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros(rows.shape[0])
    lib().oracle_dense_rows(_p(pts), pts.shape[0], kernel_id, c, scale, shift, test_rank, _p(x),
                            _p(rows), rows.shape[0], _p(out))
    return out


class Operator:
    """Oracle HODLR2D operator (Alg. 1 build, Alg. 2 matvec)."""

    def __init__(self, points, kernel_id=0, leaf_size=64, tol=1e-10, c=1.0, scale=1.0, shift=0.0,
                 test_rank=1, box_lo=(0.0, 0.0), box_side=0.0, depth=-1, max_rank=128,
                 consecutive=3, trim=3, row_range=None, symmetric=False):
        self.points = np.ascontiguousarray(points, dtype=np.float64)
        self.n = self.points.shape[0]
        lo, hi = row_range if row_range is not None else (0, 0)
        self._h = lib().oracle_build(_p(self.points), self.n, kernel_id, c, scale, shift, test_rank,
                                     leaf_size, tol, box_lo[0], box_lo[1], box_side, depth, max_rank,
                                     consecutive, trim, lo, hi, int(bool(symmetric)))
        if not self._h:
            raise ValueError(f"oracle_build failed: {last_error()}")
        self.kappa = int(lib().oracle_kappa(self._h))
        self.build_seconds = float(lib().oracle_build_seconds(self._h))

    def close(self):
        if self._h:
            lib().oracle_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def tree(self):
        perm = np.zeros(self.n, np.int32)
        ls = np.zeros((1 << (2 * self.kappa)) + 1, np.int32)
        lib().oracle_get_tree(self._h, _p(perm), _p(ls))
        return perm, ls

    def num_blocks(self, level):
        return int(lib().oracle_num_blocks(self._h, level))

    def ranks(self, level):
        nb = self.num_blocks(level)
        r = np.zeros(nb, np.int32); t = np.zeros(nb, np.int32)
        lib().oracle_get_ranks(self._h, level, _p(r), _p(t))
        return r, t

    def block(self, level, e):
        m = C.c_int(); n = C.c_int(); r = C.c_int()
        lib().oracle_get_block(self._h, level, e, C.byref(m), C.byref(n), C.byref(r), None, None)
        U = np.zeros(m.value * r.value + 1); V = np.zeros(n.value * r.value + 1)
        lib().oracle_get_block(self._h, level, e, C.byref(m), C.byref(n), C.byref(r), _p(U), _p(V))
        k = r.value
        return (U[: m.value * k].reshape(k, m.value).T.copy(), V[: n.value * k].reshape(k, n.value).T.copy())

    def factor_values(self):
        return int(lib().oracle_factor_values(self._h))

    def matvec(self, x, order="original"):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.n)
        lib().oracle_matvec(self._h, _p(x), _p(y), 0 if order == "original" else 1)
        return y

    def leaves(self):
        """(level, box) of every leaf, Morton order (adaptive tree R24; balanced: level kappa)."""
        k = int(lib().oracle_leaves(self._h, None, None))
        lv = np.zeros(max(k, 1), np.int32); bx = np.zeros(max(k, 1), np.int32)
        lib().oracle_leaves(self._h, _p(lv), _p(bx))
        return lv[:k], bx[:k]

    def op_lists(self, level):
        """The operator's interaction-list CSR of a level (adaptive: existing boxes only)."""
        tot = int(lib().oracle_op_level_lists(self._h, level, None, None))
        off = np.zeros((1 << (2 * level)) + 1, np.int32)
        col = np.zeros(max(tot, 1), np.int32)
        lib().oracle_op_level_lists(self._h, level, _p(off), _p(col))
        return off, col[:tot]

    def dense_pairs(self):
        """Dense blocks as arrays (level, X, Y), ordered by (level, X, Y)."""
        k = int(lib().oracle_dense_pairs(self._h, None, None, None))
        a, b, c = (np.zeros(max(k, 1), np.int32) for _ in range(3))
        lib().oracle_dense_pairs(self._h, _p(a), _p(b), _p(c))
        return a[:k], b[:k], c[:k]

    def save_factors(self, path):
        rc = lib().oracle_save_factors(self._h, str(path).encode())
        if rc != 0:
            raise ValueError(last_error())


def gmres(matvec, b, tol=1e-10, restart=30, max_iter=1000):
    """Restarted GMRES(m) on x -> matvec(x), x0 = 0, stopping when the true (restart) or the
    Givens-estimated (inner) relative residual ||b - A x|| / ||b|| < tol.

    The paper's solver (§5.2: "stopping criteria for GMRES is
    residual less than 1e-10 with restart after each iterations"; restart length and
    orthogonalisation unstated -> DESIGN.md R20: GMRES(30), relative residual, x0 = 0).
    Plain textbook algorithm (Saad, Iterative Methods, Alg. 6.9): Arnoldi with modified
    Gram-Schmidt, Givens rotations on the Hessenberg matrix, back substitution.
    Returns (x, total inner iterations, final relative residual ||b - A x|| / ||b||)."""
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    bnorm = float(np.linalg.norm(b))
    x = np.zeros(n)
    if bnorm == 0.0:
        return x, 0, 0.0
    its = 0
    while True:
        r = b - matvec(x)
        beta = float(np.linalg.norm(r))
        if beta / bnorm < tol or its >= max_iter:
            return x, its, beta / bnorm
        m = restart
        V = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        k = 0
        for j in range(m):
            w = matvec(V[j])
            for i in range(j + 1):                      # modified Gram-Schmidt
                H[i, j] = float(np.dot(w, V[i]))
                w = w - H[i, j] * V[i]
            H[j + 1, j] = float(np.linalg.norm(w))
            if H[j + 1, j] > 0.0:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):                          # previous rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            d = float(np.hypot(H[j, j], H[j + 1, j]))    # new rotation zeroing H[j+1, j]
            cs[j], sn[j] = (H[j, j] / d, H[j + 1, j] / d) if d > 0.0 else (1.0, 0.0)
            H[j, j] = d
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            k = j + 1
            its += 1
            if abs(g[j + 1]) / bnorm < tol or its >= max_iter:
                break
        y = np.zeros(k)                                 # back substitution H[:k,:k] y = g[:k]
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - float(np.dot(H[i, i + 1:k], y[i + 1:k]))) / H[i, i]
        x = x + V[:k].T @ y
