"""CPU checks of the C ABI boundary: the library loads, exports every function that
include/hodlr2d.h declares, the ctypes mirrors match the C struct layouts, and argument
validation fails with the documented codes before any device work."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hodlr2d.h")


@pytest.fixture(scope="module")
def h2d():
    import paper_2204_05536_b200 as m
    from paper_2204_05536_b200 import build as b
    b.build()
    return m


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hodlr2d_[a-z_]+)\s*\(", src)))


def test_header_declares_binding_functions(h2d):
    assert declared_functions() == sorted(h2d.ABI_FUNCTIONS)


def test_library_exports_every_declared_symbol(h2d):
    L = h2d.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", h2d.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (\w+)", out))
    assert set(declared_functions()) <= exported
    # nothing but the ABI leaks out of the shared object
    assert all(s.startswith("hodlr2d_") for s in exported)


def test_struct_layouts_match_c(h2d, tmp_path):
    prog = tmp_path / "layout.c"
    prog.write_text(f"""
#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(hodlr2d_options),
         sizeof(hodlr2d_info), offsetof(hodlr2d_options, stream), offsetof(hodlr2d_options, aca_scratch_bytes),
         offsetof(hodlr2d_options, symmetric) + 1000000 * offsetof(hodlr2d_options, leaf_weights),
         offsetof(hodlr2d_info, rank_hist),
         offsetof(hodlr2d_info, matvec_bytes), offsetof(hodlr2d_info, device_bytes),
         offsetof(hodlr2d_info, symmetric_apply), offsetof(hodlr2d_info, p2p_launches),
         offsetof(hodlr2d_info, p2p_leaves), offsetof(hodlr2d_info, apply_launches),
         offsetof(hodlr2d_info, small_items));
  printf("%zu %zu %zu %zu %zu %zu %zu\\n", offsetof(hodlr2d_options, nccl_id), offsetof(hodlr2d_options, allgather_ctx),
         offsetof(hodlr2d_info, comm_kind), offsetof(hodlr2d_info, n_leaves), offsetof(hodlr2d_info, local_items),
         offsetof(hodlr2d_info, stored_near_values), offsetof(hodlr2d_info, p2p_log_table));
  return 0;
}}""")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-o", str(exe), str(prog)])
    vals = list(map(int, subprocess.check_output([str(exe)]).split()))
    O, I = h2d.Options, h2d.Info
    assert vals == [C.sizeof(O), C.sizeof(I), O.stream.offset, O.aca_scratch_bytes.offset,
                    O.symmetric.offset + 1000000 * O.leaf_weights.offset,
                    I.rank_hist.offset, I.matvec_bytes.offset, I.device_bytes.offset, I.symmetric_apply.offset,
                    I.p2p_launches.offset, I.p2p_leaves.offset, I.apply_launches.offset, I.small_items.offset,
                    O.nccl_id.offset, O.allgather_ctx.offset, I.comm_kind.offset, I.n_leaves.offset,
                    I.local_items.offset, I.stored_near_values.offset, I.p2p_log_table.offset]


def test_default_options(h2d):
    o = h2d.default_options()
    assert (o.c, o.scale, o.shift, o.depth, o.max_rank) == (1.0, 1.0, 0.0, -1, 128)
    assert (o.aca_consecutive, o.aca_trim, o.world, o.rank, o.timing) == (3, 3, 1, 0, 0)


def test_argument_validation_codes(h2d):
    pts = np.zeros((4, 2))
    L = h2d.lib()
    h = C.c_void_p()
    o = h2d.default_options()
    assert L.hodlr2d_build_ex(pts.ctypes.data, 0, 0, 64, 1e-8, C.byref(o), C.byref(h)) == h2d.H2D_EINVAL
    assert L.hodlr2d_build_ex(pts.ctypes.data, 4, 0, 0, 1e-8, C.byref(o), C.byref(h)) == h2d.H2D_EINVAL
    assert L.hodlr2d_build_ex(pts.ctypes.data, 4, 0, 64, 1.5, C.byref(o), C.byref(h)) == h2d.H2D_EINVAL
    assert L.hodlr2d_build_ex(pts.ctypes.data, 4, 7, 64, 1e-8, C.byref(o), C.byref(h)) == h2d.H2D_EINVAL
    assert "kernel" in L.hodlr2d_last_error().decode()
    o.world, o.rank = 2, 2
    assert L.hodlr2d_build_ex(pts.ctypes.data, 4, 0, 64, 1e-8, C.byref(o), C.byref(h)) == h2d.H2D_EINVAL
    assert h.value is None
    assert L.hodlr2d_destroy(None) == 0
    assert L.hodlr2d_num_blocks(None, 1) == -1
    assert L.hodlr2d_copy_leaves(None, None, None) == -1
    # the adaptive tree is single-rank only; depth below -3 is invalid
    o = h2d.default_options()
    o.depth, o.world, o.rank = -3, 2, 0
    assert L.hodlr2d_build_ex(pts.ctypes.data, 4, 0, 64, 1e-8, C.byref(o), C.byref(h)) == h2d.H2D_EINVAL
    o = h2d.default_options()
    o.depth = -4
    assert L.hodlr2d_build_ex(pts.ctypes.data, 4, 0, 64, 1e-8, C.byref(o), C.byref(h)) == h2d.H2D_EINVAL
    # hodlr2d_partition (host only): bad arguments are reported, not thrown across the ABI
    ls = np.zeros(17, np.int32)
    lb, le = C.c_int64(), C.c_int64()
    assert L.hodlr2d_partition(ls.ctypes.data, 2, 0, 0, C.byref(lb), C.byref(le)) == h2d.H2D_EINVAL
    assert L.hodlr2d_partition(ls.ctypes.data, 16, 1, 0, C.byref(lb), C.byref(le)) == h2d.H2D_EINVAL
    assert L.hodlr2d_partition(None, 2, 1, 0, C.byref(lb), C.byref(le)) == h2d.H2D_EINVAL
    ls = np.arange(17, dtype=np.int32) * 3
    assert L.hodlr2d_partition(ls.ctypes.data, 2, 2, 1, C.byref(lb), C.byref(le)) == 0 and le.value == 16
    # the NCCL unique id: H2D_OK where NCCL loads, else H2D_ENCCL (never a crash)
    idb = (C.c_ubyte * h2d.COMM_ID_BYTES)()
    assert L.hodlr2d_comm_unique_id(C.cast(idb, C.c_void_p)) in (0, h2d.H2D_ENCCL)
    assert L.hodlr2d_comm_unique_id(None) == h2d.H2D_EINVAL
    assert L.hodlr2d_set_diag(None, b"p2p_serial", 1) == h2d.H2D_EINVAL


def test_product_package_does_not_touch_the_oracle():
    pkg = os.path.join(ROOT, "paper_2204_05536_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "hodlr2d_oracle" not in txt and "liboracle" not in txt, f
