"""C-ABI tests that need no GPU: the library loads, exports every symbol the header
declares, and rejects malformed descriptors with the documented status codes (all
validation happens before any device call)."""
import ctypes as C
import os
import re

import numpy as np
import pytest
import torch

from bfinputs import random_butterfly, random_ranks_butterfly
import paper_2007_00202_b200 as pkg
from paper_2007_00202_b200 import bfapply as B

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "bfapply.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    L = pkg.lib()
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    assert pkg.version().startswith("bfapply")


def test_status_strings():
    L = pkg.lib()
    for code, name in B.STATUS.items():
        assert L.bf_status_string(code).decode() == name


def _create(bf, mutate=None):
    keep = B._Keep()
    d = B.make_desc(bf, keep)
    if mutate:
        mutate(d, keep)
    h = C.c_void_p()
    rc = pkg.lib().bf_create(C.byref(d), 0, C.byref(h))
    if rc == 0:
        pkg.lib().bf_destroy(h)
    return rc


def test_bad_leaf_ptr_is_shape_error():
    bf = random_butterfly(L=2, leaf=4, r=2, seed=0)

    def mut(d, keep):
        p = keep(np.array([0, 4, 3, 12, 16], dtype=np.int64))
        d.row_leaf_ptr = p.ctypes.data_as(C.POINTER(C.c_int64))
    assert _create(bf, mut) == -2


def test_bad_L_is_shape_error():
    bf = random_butterfly(L=2, leaf=4, r=2, seed=0)

    def mut(d, keep):
        d.lc = 3
    assert _create(bf, mut) == -2


def test_length_mismatch_is_rank_error():
    bf = random_butterfly(L=2, leaf=4, r=2, seed=0)

    def mut(d, keep):
        d.len_R = d.len_R - 1
    assert _create(bf, mut) == -3


def test_negative_rank_is_rank_error():
    bf = random_butterfly(L=2, leaf=4, r=2, seed=0)

    def mut(d, keep):
        rr = keep(np.array(bf.rank_row(), dtype=np.int32))
        rr[0] = -1
        d.rank_row = rr.ctypes.data_as(C.POINTER(C.c_int32))
    assert _create(bf, mut) == -3


def test_bad_perm_is_perm_error():
    bf = random_butterfly(L=2, leaf=4, r=2, seed=0)

    def mut(d, keep):
        p = keep(np.arange(bf.m, dtype=np.int64))
        p[1] = 0
        d.row_perm = p.ctypes.data_as(C.POINTER(C.c_int64))
    assert _create(bf, mut) == -4


def test_null_args():
    h = C.c_void_p()
    assert pkg.lib().bf_create(None, 0, C.byref(h)) == -1
    assert pkg.lib().bf_apply_op(None, 0, 1, None, 1, None, 1, None, 0, None) == -1
    assert pkg.lib().hodbf_apply(None, 0, 1, None, 1, None, 1, None, 0, None) == -1


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device path")
def test_no_device_fails_loudly():
    bf = random_ranks_butterfly(2, [3, 2, 4, 1], [2, 2, 3, 5], seed=0)
    assert _create(bf) == -8
    with pytest.raises(B.BFError):
        pkg.BFHandle(bf, 0)


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors of the C-ABI structs have the header's sizes and field offsets (a
    mismatch would corrupt every call silently): compile a probe against include/bfapply.h."""
    import subprocess
    from paper_2007_00202_b200 import construct as cx
    structs = {"bf_desc": B.bf_desc, "hodbf_desc": B.hodbf_desc, "bf_info_t": B.bf_info_t,
               "bf_round_info_t": B.bf_round_info_t, "bf_rmv_desc": cx.bf_rmv_desc, "bf_rmv_stats": cx.bf_rmv_stats,
               "bf_factor": cx.bf_factor, "bf_product": cx.bf_product, "bf_operator": cx.bf_operator,
               "bf_inv_opts": cx.bf_inv_opts, "bf_front": cx.bf_front}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "bfapply.h"', 'int main(void) {']
    for name, st in structs.items():
        lines.append(f'  printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in st._fields_:
            lines.append(f'  printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines.append('  return 0; }')
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    subprocess.run(["gcc", "-std=c99", "-I", inc, str(src), "-o", str(exe)], check=True)
    out = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines())
    for name, st in structs.items():
        assert int(out[name]) == C.sizeof(st), name
        for f, _ in st._fields_:
            assert int(out[f"{name}.{f}"]) == getattr(st, f).offset, (name, f)


def test_construction_calls_need_a_device():
    """bf_random_matvec / hodbf_invert / bf_mf_create have no CPU path: without a CUDA device they
    return BF_ERR_DEVICE (or BF_ERR_ARG for an obviously bad argument) instead of computing."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    from paper_2007_00202_b200 import construct as cx
    L = cx._lib()
    d = cx.bf_rmv_desc()
    lp = np.array([0, 4, 8], dtype=np.int64)
    d.dtype, d.L, d.lc, d.rank_max, d.m, d.n = 2, 1, -1, 4, 8, 8
    d.row_leaf_ptr = lp.ctypes.data_as(C.POINTER(C.c_int64))
    d.col_leaf_ptr = lp.ctypes.data_as(C.POINTER(C.c_int64))
    d.eps, d.oversample = 1e-10, 4
    h = C.c_void_p()
    st = cx.bf_rmv_stats()
    rc = L.bf_random_matvec(C.byref(d), C.cast(L.bf_operator_apply, C.c_void_p), None, 0, None, C.byref(h),
                            C.byref(st))
    assert rc == -8 and not h.value


# ---- bf_desc.level_maps ("level-by-level index permutations") and L <= 30 ----
def _create_maps(bf, maps, mutate=None, dist=False):
    keep = B._Keep()
    d = B.make_desc(bf, keep, level_maps=maps)
    if mutate:
        mutate(d, keep)
    h = C.c_void_p()
    if dist:  # host-only distributed plan (device < 0): the whole create runs, nothing uploads
        rc = pkg.lib().bf_dist_create(C.byref(d), 0, 1, -1, C.byref(h))
    else:
        rc = pkg.lib().bf_create(C.byref(d), 0, C.byref(h))
    if rc == 0:
        pkg.lib().bf_destroy(h)
    return rc


def test_level_maps_not_bijection_is_perm_error():
    from bfinputs import random_level_maps, slot_ordered
    bf = random_ranks_butterfly(3, [3, 2, 4, 1, 5, 2, 2, 3], [2, 2, 3, 5, 1, 1, 4, 2], seed=0)
    maps = random_level_maps(bf.L, seed=1)
    bad = [m.copy() for m in maps]
    bad[2][0] = bad[2][1]
    assert _create_maps(slot_ordered(bf, maps), bad) == -4
    bad = [m.copy() for m in maps]
    bad[0][3] = 1 << bf.L
    assert _create_maps(slot_ordered(bf, maps), bad) == -4


def test_level_maps_accepted_by_a_host_plan():
    """A slot-ordered descriptor with its maps passes every create-time check (ranks, lengths)
    through the canonical re-pack; the same packing without maps, with ragged ranks whose block
    sizes differ per slot, fails the rank-chain length check."""
    from bfinputs import random_level_maps, slot_ordered
    rng = np.random.default_rng(3)
    bf = random_ranks_butterfly(4, rng.integers(0, 9, 16), rng.integers(1, 9, 16), seed=3, rmin=0, rmax=7)
    for lv in (None, [0], [bf.L], [bf.lc], [1, 3]):
        maps = random_level_maps(bf.L, seed=5, levels=lv)
        assert _create_maps(slot_ordered(bf, maps), maps, dist=True) == 0
    maps = random_level_maps(bf.L, seed=5)
    assert _create_maps(slot_ordered(bf, maps), None, dist=True) in (0, -3)
    assert _create_maps(bf, [None] * (bf.L + 1), dist=True) == 0


def test_L_limit_is_30():
    bf = random_butterfly(L=2, leaf=4, r=2, seed=0)

    def mut(d, keep):
        d.L = 31
    assert _create(bf, mut) == -2


def test_create_dist_needs_a_comm_for_several_ranks():
    """bf_create_dist (library-owned NCCL): NULL communicator with nranks > 1 on a device is
    BF_ERR_ARG; a host-only plan (device < 0) needs none and has bf_dist_create's layout."""
    from paper_2007_00202_b200.dist import _lib
    L = _lib()
    assert L.bf_nccl_available() in (0, 1)
    bf = random_butterfly(L=4, leaf=8, r=4, seed=0)
    keep = B._Keep()
    d = B.make_desc(bf, keep)
    h = C.c_void_p()
    assert L.bf_create_dist(C.byref(d), 0, 2, None, 0, C.byref(h)) == -1
    assert L.bf_create_dist(C.byref(d), 1, 2, None, -1, C.byref(h)) == 0
    h2 = C.c_void_p()
    assert L.bf_dist_create(C.byref(d), 1, 2, -1, C.byref(h2)) == 0
    lay = []
    for hh in (h, h2):
        wb, so, ro = C.c_size_t(), C.c_size_t(), C.c_size_t()
        sc, rc = (C.c_int64 * 2)(), (C.c_int64 * 2)()
        assert L.bf_dist_layout(hh, 0, 8, C.byref(wb), C.byref(so), C.byref(ro), sc, rc) == 0
        lay.append((wb.value, so.value, ro.value, list(sc), list(rc)))
        L.bf_destroy(hh)
    assert lay[0] == lay[1]
    assert L.bf_apply_dist(None, 0, 1, None, 1, None, 1, None, 0, None) == -1
