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
