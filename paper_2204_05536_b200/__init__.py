"""B200-native HODLR2D fast matvec (arXiv 2204.05536) — thin ctypes binding of the C ABI.

Every entry point mirrors a function of ``include/hodlr2d.h`` (same names, argument
marshalling only).  All arithmetic of the build and the matvec runs in the CUDA kernels
of ``libhodlr2d.so``; there is no CPU fallback: if the library is missing, importing the
binding's functions raises.  PyTorch is used only for device memory and streams.

Quick use::

    import torch, paper_2204_05536_b200 as h2d
    pts = torch.rand(1 << 20, 2, dtype=torch.float64, device="cuda") * 2 - 1
    op = h2d.Hodlr2d.build(pts, kernel="log", leaf_size=64, aca_tol=1e-8,
                           box_lo=(-1, -1), box_side=2.0)
    y = op.matvec(torch.randn(1 << 20, dtype=torch.float64, device="cuda"))
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# H2D_LIBRARY: diagnostics builds of the same sources (e.g. a timing variant); default in-tree
LIB_PATH = os.environ.get("H2D_LIBRARY") or os.path.join(_HERE, "libhodlr2d.so")

H2D_OK, H2D_WTRUNC, H2D_WNOCONV = 0, 1, 2
H2D_EINVAL, H2D_EOUTOFBOX, H2D_ECOINCIDENT, H2D_ENOMEM = -1, -2, -3, -4
H2D_ECUDA, H2D_ENCCL, H2D_EFACTORS = -5, -6, -7
KERNELS = {"log": 0, "imq": 1, "one_over_r": 2, "rbf_phi1": 3, "rbf_phi2": 4, "test_lowrank": 100}
ORDER_ORIGINAL, ORDER_TREE, ORDER_GATHERED, ORDER_LOCAL = 0, 1, 2, 3
ORDERS = {"original": 0, "tree": 1, "gathered": 2, "local": 3}
COMM_ID_BYTES = 128
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
MAX_LEVELS = 16
NUM_STAGES = 6
STAGE_NAMES = ("input_permute", "stageA_VTx", "stageB_Ut", "p2p_join_wait", "combine", "p2p_near")

# Every function declared in include/hodlr2d.h (checked by tests/test_abi.py).
ABI_FUNCTIONS = (
    "hodlr2d_default_options", "hodlr2d_build", "hodlr2d_build_ex", "hodlr2d_matvec",
    "hodlr2d_matvec_ex", "hodlr2d_get_info", "hodlr2d_copy_tree", "hodlr2d_copy_lists",
    "hodlr2d_num_blocks", "hodlr2d_copy_ranks", "hodlr2d_copy_block", "hodlr2d_load_factors",
    "hodlr2d_save_factors", "hodlr2d_stage_times", "hodlr2d_set_timing", "hodlr2d_destroy",
    "hodlr2d_last_error", "hodlr2d_partition", "hodlr2d_gmres", "hodlr2d_matvec_multi", "hodlr2d_leaf_costs",
    "hodlr2d_comm_unique_id", "hodlr2d_set_diag", "hodlr2d_copy_leaves", "hodlr2d_matvec_async",
    "hodlr2d_wait",
)


class Options(C.Structure):
    """Mirror of ``hodlr2d_options``."""
    _fields_ = [
        ("c", C.c_double), ("scale", C.c_double), ("shift", C.c_double),
        ("box_lo", C.c_double * 2), ("box_side", C.c_double),
        ("depth", C.c_int), ("max_rank", C.c_int), ("aca_consecutive", C.c_int),
        ("aca_trim", C.c_int), ("test_rank", C.c_int),
        ("stream", C.c_void_p), ("world", C.c_int), ("rank", C.c_int),
        ("row_begin", C.c_int64), ("row_end", C.c_int64),
        ("aca_scratch_bytes", C.c_size_t), ("timing", C.c_int), ("skip_aca", C.c_int),
        ("symmetric", C.c_int), ("leaf_weights", C.c_void_p),
        ("nccl_id", C.c_void_p), ("allgather", ALLGATHER_FN), ("allgather_ctx", C.c_void_p),
    ]


class Info(C.Structure):
    """Mirror of ``hodlr2d_info``."""
    _fields_ = [
        ("n", C.c_int64), ("kappa", C.c_int), ("world", C.c_int), ("rank", C.c_int),
        ("row_begin", C.c_int64), ("row_end", C.c_int64),
        ("leaf_begin", C.c_int64), ("leaf_end", C.c_int64),
        ("box_lo", C.c_double * 2), ("box_side", C.c_double),
        ("blocks_per_level", C.c_int64 * (MAX_LEVELS + 1)), ("blocks_built", C.c_int64),
        ("rank_max", C.c_int), ("rank_hist", C.c_int64 * 129),
        ("u_values", C.c_int64), ("v_values", C.c_int64), ("near_pairs", C.c_int64),
        ("compression_ratio", C.c_double), ("truncated", C.c_int64),
        ("tree_seconds", C.c_double), ("aca_seconds", C.c_double), ("pack_seconds", C.c_double),
        ("build_seconds", C.c_double), ("matvec_bytes", C.c_int64),
        ("stageA_bytes", C.c_int64), ("stageB_bytes", C.c_int64), ("p2p_pairs", C.c_double),
        ("device_bytes", C.c_int64), ("gather_stride", C.c_int64), ("p2p_bytes", C.c_int64),
        ("symmetric_apply", C.c_int), ("p2p_launches", C.c_int), ("p2p_leaves", C.c_int64 * 3),
        ("apply_launches", C.c_int), ("small_items", C.c_int64 * 2),
        ("comm_kind", C.c_int), ("adaptive", C.c_int), ("pair_apply", C.c_int), ("n_leaves", C.c_int64),
        ("local_items", C.c_int64 * 2), ("stored_near_values", C.c_int64),
        ("p2p_log_table", C.c_int),
    ]

    def as_dict(self) -> dict:
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            if hasattr(v, "__len__"):
                v = list(v)
            d[name] = v
        d["blocks_per_level"] = d["blocks_per_level"][1: self.kappa + 1]
        d["rank_hist"] = {r: c for r, c in enumerate(d["rank_hist"]) if c}
        return d


_lock = threading.Lock()
_lib = None


def lib() -> C.CDLL:
    """Load libhodlr2d.so (built in-tree by ``__graft_entry__.build()``).  Raises if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2204_05536_b200.build` "
                    "(there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            vp, i, i64, d = C.c_void_p, C.c_int, C.c_int64, C.c_double
            L.hodlr2d_default_options.argtypes = [C.POINTER(Options)]
            L.hodlr2d_default_options.restype = None
            L.hodlr2d_build.argtypes = [vp, i64, i, i, d, C.POINTER(vp)]
            L.hodlr2d_build_ex.argtypes = [vp, i64, i, i, d, C.POINTER(Options), C.POINTER(vp)]
            L.hodlr2d_matvec.argtypes = [vp, vp, vp]
            L.hodlr2d_matvec_ex.argtypes = [vp, vp, vp, i]
            L.hodlr2d_matvec_async.argtypes = [vp, vp, vp, i]
            L.hodlr2d_wait.argtypes = [vp]
            L.hodlr2d_get_info.argtypes = [vp, C.POINTER(Info)]
            L.hodlr2d_copy_tree.argtypes = [vp, vp, vp]
            L.hodlr2d_copy_lists.argtypes = [vp, i, vp, vp]
            L.hodlr2d_num_blocks.argtypes = [vp, i]
            L.hodlr2d_num_blocks.restype = i64
            L.hodlr2d_copy_ranks.argtypes = [vp, i, vp]
            L.hodlr2d_copy_block.argtypes = [vp, i, i64, C.POINTER(i), C.POINTER(i), C.POINTER(i), vp, vp]
            L.hodlr2d_load_factors.argtypes = [vp, C.c_char_p]
            L.hodlr2d_save_factors.argtypes = [vp, C.c_char_p]
            L.hodlr2d_stage_times.argtypes = [vp, vp, C.POINTER(i64), i]
            L.hodlr2d_set_timing.argtypes = [vp, i]
            L.hodlr2d_destroy.argtypes = [vp]
            L.hodlr2d_last_error.restype = C.c_char_p
            L.hodlr2d_partition.argtypes = [vp, i, i, i, C.POINTER(i64), C.POINTER(i64)]
            L.hodlr2d_gmres.argtypes = [vp, vp, vp, d, i, i, C.POINTER(i), C.POINTER(d)]
            L.hodlr2d_matvec_multi.argtypes = [vp, vp, vp, i, i]
            L.hodlr2d_leaf_costs.argtypes = [vp, vp]
            L.hodlr2d_comm_unique_id.argtypes = [vp]
            L.hodlr2d_set_diag.argtypes = [vp, C.c_char_p, i]
            L.hodlr2d_copy_leaves.argtypes = [vp, vp, vp]
            L.hodlr2d_copy_leaves.restype = i64
            _lib = L
    return _lib


class Hodlr2dError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc: int) -> int:
    if rc < 0:
        raise Hodlr2dError(rc, lib().hodlr2d_last_error().decode())
    return rc


def _ptr(a) -> int:
    """Raw pointer of a torch tensor (host or CUDA) or a numpy array (host)."""
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"] or a.dtype != np.float64:
            raise ValueError("numpy arrays must be C-contiguous float64")
        return a.ctypes.data
    if not a.is_contiguous() or str(a.dtype) != "torch.float64":
        raise ValueError("tensors must be contiguous float64")
    return a.data_ptr()


def partition(leaf_start: np.ndarray, kappa: int, world: int, rank: int):
    """hodlr2d_partition (host only): leaves [begin, end) served by `rank` of `world`."""
    ls = np.ascontiguousarray(leaf_start, dtype=np.int32)
    lb, le = C.c_int64(), C.c_int64()
    _check(lib().hodlr2d_partition(ls.ctypes.data, kappa, world, rank, C.byref(lb), C.byref(le)))
    return lb.value, le.value


def comm_unique_id() -> bytes:
    """hodlr2d_comm_unique_id: a fresh NCCL unique id for options.nccl_id (one rank creates
    it, the caller broadcasts it)."""
    buf = (C.c_ubyte * COMM_ID_BYTES)()
    _check(lib().hodlr2d_comm_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def _host_allgather(group):
    """Host all-gather callback (options.allgather) over a torch.distributed CPU group (gloo):
    argument marshalling only — the library hands over host buffers it owns."""
    import torch
    import torch.distributed as dist

    def cb(send, recv, nbytes, ctx):
        try:
            world = dist.get_world_size(group)
            n = nbytes // 8
            st = torch.from_numpy(np.ctypeslib.as_array((C.c_double * n).from_address(send)))
            rt = torch.from_numpy(np.ctypeslib.as_array((C.c_double * (n * world)).from_address(recv)))
            dist.all_gather_into_tensor(rt, st, group=group)
            return 0
        except Exception:  # noqa: BLE001 - reported to the library as a failed collective
            return -1
    return ALLGATHER_FN(cb)


def default_options() -> Options:
    o = Options()
    lib().hodlr2d_default_options(C.byref(o))
    return o


class Hodlr2d:
    """Owner of a ``hodlr2d_t`` handle."""

    def __init__(self, handle: int, n: int, keepalive=None):
        self._h = C.c_void_p(handle)
        self.n = n
        self._keep = keepalive
        self.status = H2D_OK

    # -------------------------------------------------------------- build
    @classmethod
    def build(cls, points, kernel="log", leaf_size=64, aca_tol=1e-10, *, c=1.0, scale=1.0,
              shift=0.0, box_lo=(0.0, 0.0), box_side=0.0, depth=-1, max_rank=128,
              aca_consecutive=3, aca_trim=3, test_rank=1, stream=None, world=1, rank=0,
              row_range=None, aca_scratch_bytes=0, timing=False, skip_aca=False, symmetric=False,
              leaf_weights=None, group=None, nccl_id=None):
        """hodlr2d_build_ex.  ``points``: (N, 2) float64 torch tensor (CUDA or CPU) or numpy array.
        ``leaf_weights``: host float64 array of 4^kappa per-leaf loads for the world partition
        (e.g. the sum over ranks of ``leaf_costs()`` of a first build).
        ``group``: a torch.distributed process group; world / rank are taken from it and the
        handle gets a communicator for ``matvec(x_local, order="local")`` (S11): with an NCCL
        group, rank 0's NCCL unique id is broadcast over it (the library then owns an NCCL
        communicator); with a gloo group, the library's host-staged gather calls back into
        all_gather_into_tensor.  ``nccl_id``: an id from ``comm_unique_id()`` (no group)."""
        kid = KERNELS[kernel] if isinstance(kernel, str) else int(kernel)
        o = default_options()
        o.c, o.scale, o.shift = c, scale, shift
        o.box_lo[0], o.box_lo[1] = box_lo
        o.box_side = box_side
        o.depth, o.max_rank = depth, max_rank
        o.aca_consecutive, o.aca_trim, o.test_rank = aca_consecutive, aca_trim, test_rank
        if stream is None:
            try:
                import torch
                if torch.cuda.is_available():
                    stream = torch.cuda.current_stream().cuda_stream
            except Exception:
                stream = None
        o.stream = stream or None
        keep = []
        if group is not None:
            import torch.distributed as dist
            world, rank = dist.get_world_size(group), dist.get_rank(group)
            if dist.get_backend(group) == "nccl":
                obj = [comm_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0), group=group)
                nccl_id = obj[0]
            else:
                cb = _host_allgather(group)
                keep.append(cb)
                o.allgather = cb
        if nccl_id is not None:
            idbuf = (C.c_ubyte * COMM_ID_BYTES).from_buffer_copy(nccl_id)
            keep.append(idbuf)
            o.nccl_id = C.cast(idbuf, C.c_void_p)
        o.world, o.rank = world, rank
        if row_range is not None:
            o.row_begin, o.row_end = row_range
        o.aca_scratch_bytes = aca_scratch_bytes
        o.timing = int(bool(timing))
        o.skip_aca = int(bool(skip_aca))
        o.symmetric = int(bool(symmetric))
        lw = None
        if leaf_weights is not None:
            lw = np.ascontiguousarray(leaf_weights, dtype=np.float64)
            o.leaf_weights = lw.ctypes.data
        n = points.shape[0]
        h = C.c_void_p()
        rc = _check(lib().hodlr2d_build_ex(_ptr(points), n, kid, leaf_size, aca_tol, C.byref(o), C.byref(h)))
        op = cls(h.value, n, keepalive=keep)
        op.status = rc
        op._stream = stream
        return op

    @classmethod
    def build_default(cls, points, kernel_id: int, leaf_size: int, aca_tol: float):
        """hodlr2d_build (the four-argument north-star call, default options)."""
        h = C.c_void_p()
        rc = _check(lib().hodlr2d_build(_ptr(points), points.shape[0], kernel_id, leaf_size, aca_tol, C.byref(h)))
        op = cls(h.value, points.shape[0])
        op.status = rc
        return op

    def close(self):
        if self._h is not None and self._h.value:
            lib().hodlr2d_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -------------------------------------------------------------- matvec
    def _lens(self, o: int):
        """(len_x, len_y) of one vector in order o (include/hodlr2d.h orderings)."""
        if o == ORDER_ORIGINAL:
            return self.n, self.n
        inf = self.info()
        m = inf["row_end"] - inf["row_begin"]
        if o == ORDER_TREE:
            return self.n, m
        if o == ORDER_GATHERED:
            return inf["world"] * inf["gather_stride"], m
        return m, m

    def _check_vec(self, a, length: int, what: str):
        """The C side reads / writes exactly `length` values: refuse shorter buffers and
        tensors on another device than the handle's stream (marshalling checks only)."""
        numel = a.size if isinstance(a, np.ndarray) else a.numel()
        if numel != length:
            raise ValueError(f"{what} has {numel} values, expected {length}")
        if not isinstance(a, np.ndarray) and a.is_cuda:
            import torch
            if a.device.index != torch.cuda.current_device():
                raise ValueError(f"{what} is on {a.device}, the handle on cuda:{torch.cuda.current_device()}")

    def _ordered(self, *tensors):
        """Order the handle's stream (fixed at build) after torch's current stream when they
        differ, and the current stream after it on exit (a context manager)."""
        import contextlib
        if not any(getattr(t, "is_cuda", False) for t in tensors):
            return contextlib.nullcontext()
        import torch
        cur = torch.cuda.current_stream()
        if self._stream is None or cur.cuda_stream == self._stream:
            return contextlib.nullcontext()
        hs = torch.cuda.ExternalStream(self._stream)

        @contextlib.contextmanager
        def ctx():
            hs.wait_stream(cur)
            yield
            cur.wait_stream(hs)
        return ctx()

    _stream = None

    def matvec(self, x, out=None, order="original"):
        """hodlr2d_matvec / hodlr2d_matvec_ex.  Returns ``out`` (allocated like x if None).
        order="local" (handles built with a group / nccl_id): x is this rank's TREE rows
        [row_begin, row_end); every rank of the world must call it (S11 inside)."""
        o = ORDERS[order]
        lx, ly = self._lens(o)
        self._check_vec(x, lx, "x")
        if out is None:
            if isinstance(x, np.ndarray):
                out = np.empty(ly, dtype=np.float64)
            else:
                import torch
                out = torch.empty(ly, dtype=torch.float64, device=x.device)
        self._check_vec(out, ly, "out")
        with self._ordered(x, out):
            if o == ORDER_ORIGINAL:
                _check(lib().hodlr2d_matvec(self._h, _ptr(x), _ptr(out)))
            else:
                _check(lib().hodlr2d_matvec_ex(self._h, _ptr(x), _ptr(out), o))
        return out

    def gmres(self, b, x=None, tol=1e-10, restart=30, max_iter=1000):
        """hodlr2d_gmres: solve A x = b (x0 = 0) with restarted GMRES on the HODLR2D matvec.
        Returns (x, iterations, true relative residual); ``converged`` is the rc == H2D_OK."""
        if x is None:
            if isinstance(b, np.ndarray):
                x = np.empty_like(b)
            else:
                import torch
                x = torch.empty_like(b)
        self._check_vec(b, self.n, "b")
        self._check_vec(x, self.n, "x")
        its, rr = C.c_int(), C.c_double()
        with self._ordered(b, x):
            rc = _check(lib().hodlr2d_gmres(self._h, _ptr(b), _ptr(x), tol, restart, max_iter,
                                            C.byref(its), C.byref(rr)))
        self.gmres_converged = rc == H2D_OK
        return x, its.value, rr.value

    def matvec_multi(self, X, out=None, order="original"):
        """hodlr2d_matvec_multi: ``X`` is (nrhs, N) (one vector per row, C-contiguous);
        returns ``out`` of shape (nrhs, len_y)."""
        o = ORDERS[order]
        nrhs = X.shape[0]
        lx, m = self._lens(o)
        self._check_vec(X, nrhs * lx, "X")
        if out is None:
            if isinstance(X, np.ndarray):
                out = np.empty((nrhs, m), dtype=np.float64)
            else:
                import torch
                out = torch.empty((nrhs, m), dtype=torch.float64, device=X.device)
        self._check_vec(out, nrhs * m, "out")
        with self._ordered(X, out):
            _check(lib().hodlr2d_matvec_multi(self._h, _ptr(X), _ptr(out), nrhs, o))
        return out

    def matvec_multi_raw(self, x_ptr: int, y_ptr: int, nrhs: int, order: int = ORDER_ORIGINAL):
        _check(lib().hodlr2d_matvec_multi(self._h, x_ptr, y_ptr, nrhs, order))

    def matvec_raw(self, x_ptr: int, y_ptr: int, order: int = ORDER_ORIGINAL):
        _check(lib().hodlr2d_matvec_ex(self._h, x_ptr, y_ptr, order))

    def matvec_async(self, x, y, order="original"):
        """hodlr2d_matvec_async: enqueue y = A x on pinned host (or device) tensors and return;
        x must stay unmodified and y unread until wait()."""
        o = ORDERS[order] if isinstance(order, str) else order
        lx, ly = self._lens(o)
        self._check_vec(x, lx, "x")
        self._check_vec(y, ly, "y")
        for t, nm in ((x, "x"), (y, "y")):
            if t.device.type == "cpu" and not t.is_pinned():
                raise ValueError(f"matvec_async: {nm} must be pinned host or device memory")
        _check(lib().hodlr2d_matvec_async(self._h, _ptr(x), _ptr(y), o))

    def matvec_async_raw(self, x_ptr: int, y_ptr: int, order: int = ORDER_ORIGINAL):
        _check(lib().hodlr2d_matvec_async(self._h, x_ptr, y_ptr, order))

    def wait(self):
        """hodlr2d_wait: every matvec_async call so far has completed."""
        _check(lib().hodlr2d_wait(self._h))

    # -------------------------------------------------------------- inspection
    def leaf_costs(self):
        """hodlr2d_leaf_costs: per-leaf algorithmic bytes of this handle's served leaves
        (float64, 4^kappa entries, zero elsewhere)."""
        kappa = self.info()["kappa"]
        out = np.zeros(1 << (2 * kappa), dtype=np.float64)
        _check(lib().hodlr2d_leaf_costs(self._h, out.ctypes.data))
        return out

    def info(self) -> dict:
        inf = Info()
        _check(lib().hodlr2d_get_info(self._h, C.byref(inf)))
        return inf.as_dict()

    def tree(self):
        inf = self.info()
        perm = np.zeros(self.n, np.int32)
        ls = np.zeros((1 << (2 * inf["kappa"])) + 1, np.int32)
        _check(lib().hodlr2d_copy_tree(self._h, perm.ctypes.data, ls.ctypes.data))
        return perm, ls

    def leaves(self):
        """hodlr2d_copy_leaves: (level, box) of every leaf in Morton order."""
        k = lib().hodlr2d_copy_leaves(self._h, None, None)
        lv = np.zeros(max(k, 1), np.int32)
        bx = np.zeros(max(k, 1), np.int32)
        lib().hodlr2d_copy_leaves(self._h, lv.ctypes.data, bx.ctypes.data)
        return lv[:k], bx[:k]

    def lists(self, level: int):
        kappa = self.info()["kappa"]
        tot = lib().hodlr2d_num_blocks(self._h, level)
        nbox = 1 << (2 * (kappa if level == 0 else level))
        off = np.zeros(nbox + 1, np.int32)
        col = np.zeros(max(tot, 1), np.int32)
        _check(lib().hodlr2d_copy_lists(self._h, level, off.ctypes.data, col.ctypes.data))
        return off, col[:tot]

    def ranks(self, level: int):
        nb = lib().hodlr2d_num_blocks(self._h, level)
        r = np.zeros(max(nb, 1), np.int32)
        _check(lib().hodlr2d_copy_ranks(self._h, level, r.ctypes.data))
        return r[:nb]

    def block(self, level: int, e: int):
        m, n, r = C.c_int(), C.c_int(), C.c_int()
        _check(lib().hodlr2d_copy_block(self._h, level, e, C.byref(m), C.byref(n), C.byref(r), None, None))
        U = np.zeros(m.value * r.value + 1)
        V = np.zeros(n.value * r.value + 1)
        _check(lib().hodlr2d_copy_block(self._h, level, e, C.byref(m), C.byref(n), C.byref(r),
                                        U.ctypes.data, V.ctypes.data))
        k = r.value
        return (U[: m.value * k].reshape(k, m.value).T.copy(), V[: n.value * k].reshape(k, n.value).T.copy())

    def load_factors(self, path):
        _check(lib().hodlr2d_load_factors(self._h, str(path).encode()))

    def save_factors(self, path):
        _check(lib().hodlr2d_save_factors(self._h, str(path).encode()))

    def set_diag(self, name: str, value: int):
        """hodlr2d_set_diag: a diagnostics switch of this handle's matvec."""
        _check(lib().hodlr2d_set_diag(self._h, name.encode(), int(value)))

    def set_timing(self, on: bool):
        _check(lib().hodlr2d_set_timing(self._h, int(bool(on))))

    def stage_times(self, reset: bool = True):
        ms = (C.c_double * NUM_STAGES)()
        cnt = C.c_int64()
        _check(lib().hodlr2d_stage_times(self._h, C.cast(ms, C.c_void_p), C.byref(cnt), int(bool(reset))))
        return dict(zip(STAGE_NAMES, list(ms))), cnt.value
