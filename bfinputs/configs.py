"""Config registry for BASELINE.json configs[0..4] plus scaled-down parity variants.

Each builder returns the factor object and the seeded right-hand side block:
  cfg1  random butterfly, n = 1024, L = 5, leaf 32, r = 8, nrhs 16, seed 0, c128
  cfg2  Helmholtz butterfly between two 64x64 planes (8h apart), 8 ppw, eps 1e-6,
        leaf 64 (L = 6), nrhs 64, c128
  cfg3  HOD-BF of a 128x128 planar self-interaction, 10 ppw, diag 1 + 1j kappa h,
        leaf 64 (LH = 8), eps 1e-4, nrhs 256, c128 / c64
  cfg4  HOD-BF, 160x160 grid x 2 tangential components (51200), dyadic kernel,
        10 ppw, leaf 50 (LH = 10), eps 1e-4, nrhs 512, c128
  cfg5  random butterfly, n = 2^20, L = 14, leaf 64, r = 16, nrhs 32, seed 1, c64/c128
Construction results can be cached on disk (BF_CACHE_DIR, default /tmp/bfcache): the
cache only saves time, every entry is rebuilt when missing.
"""
from __future__ import annotations

import os
import pickle
import hashlib

import numpy as np

from .factors import random_butterfly, random_rhs
from .geometry import (KernelMatrix, bisection_tree, expand_components, grid_points,
                       tree_depth_for_leaf)
from .construct import bf_entry_eval, hodbf_entry_eval

CACHE_VERSION = 3


def _cache(name, builder):
    d = os.environ.get("BF_CACHE_DIR", "/tmp/bfcache")
    key = hashlib.sha1(f"{name}-v{CACHE_VERSION}".encode()).hexdigest()[:12]
    path = os.path.join(d, f"{name}-{key}.pkl")
    if os.path.exists(path):
        try:
            with open(path, "rb") as f:
                return pickle.load(f)
        except Exception:
            pass
    obj = builder()
    try:
        os.makedirs(d, exist_ok=True)
        tmp = path + f".{os.getpid()}.tmp"
        with open(tmp, "wb") as f:
            pickle.dump(obj, f, protocol=pickle.HIGHEST_PROTOCOL)
        os.replace(tmp, path)
    except OSError:
        pass
    return obj


def cfg1(dtype=np.complex128):
    bf = random_butterfly(L=5, leaf=32, r=8, seed=0, dtype=dtype)
    X = random_rhs(bf.n, 16, seed=10, dtype=dtype)
    return bf, X


def cfg5(dtype=np.complex128, nrhs=32):
    bf = random_butterfly(L=14, leaf=64, r=16, seed=1, dtype=dtype)
    X = random_rhs(bf.n, nrhs, seed=11, dtype=dtype)
    return bf, X


def helmholtz_planes_bf(nx: int, leaf: int, ppw: float, sep: float, eps: float, seed=0,
                        proxy_cap=None):
    """Butterfly of the Helmholtz kernel between two parallel nx x nx planes."""
    h = 1.0
    kappa = 2 * np.pi / (ppw * h)
    depth = tree_depth_for_leaf(nx * nx, leaf)
    perm, ptr = bisection_tree(nx, nx, depth)
    P_O = grid_points(nx, nx, z=sep * h)
    P_S = grid_points(nx, nx, z=0.0)
    K = KernelMatrix(P_O, P_S, kappa)

    def ext(I, J):
        return K(perm[I], perm[J])

    bf = bf_entry_eval(ext, ptr, ptr, depth, eps, proxy_cap=proxy_cap, seed=seed,
                       meta={"kind": "helmholtz-planes", "nx": nx, "eps": eps, "kappa": kappa})
    bf.row_perm = perm.copy()
    bf.col_perm = perm.copy()
    bf.meta["kernel"] = K
    return bf


def cfg2(dtype=np.complex128, nx=64):
    bf = _cache(f"cfg2-nx{nx}", lambda: helmholtz_planes_bf(nx, 64, 8.0, 8.0, 1e-6))
    bf = bf if dtype == np.complex128 else bf.astype(dtype)
    X = random_rhs(bf.n, 64, seed=2, dtype=dtype)
    return bf, X


def helmholtz_plane_hodbf(nx: int, leaf: int, ppw: float, eps: float, ncomp=1, proxy_cap=None):
    h = 1.0
    kappa = 2 * np.pi / (ppw * h)
    npts = nx * nx
    depth = tree_depth_for_leaf(npts * ncomp, leaf)
    # depth counted on unknowns; the point tree has the same depth
    perm_p, ptr_p = bisection_tree(nx, nx, depth)
    P = grid_points(nx, nx)
    selfv = 1.0 + 1j * kappa * h
    if ncomp == 1:
        perm, ptr = perm_p, ptr_p
        K = KernelMatrix(P, P, kappa, "helmholtz", self_value=selfv)
    else:
        perm, ptr = expand_components(perm_p, ptr_p, ncomp)
        K = KernelMatrix(P, P, kappa, "dyadic", self_value=selfv)
    H = hodbf_entry_eval(K, perm, ptr, depth, eps, proxy_cap=proxy_cap,
                         meta={"kind": "hodbf", "nx": nx, "eps": eps, "kappa": kappa, "ncomp": ncomp})
    H.meta["kernel"] = K
    return H


def cfg3(dtype=np.complex128, nx=128, nrhs=256):
    H = _cache(f"cfg3-nx{nx}", lambda: helmholtz_plane_hodbf(nx, 64, 10.0, 1e-4))
    H = H if dtype == np.complex128 else H.astype(dtype)
    X = random_rhs(H.n, nrhs, seed=3, dtype=dtype)
    return H, X


def cfg4(dtype=np.complex128, nx=160, nrhs=512, proxy_cap=None):
    H = _cache(f"cfg4-nx{nx}-cap{proxy_cap}",
               lambda: helmholtz_plane_hodbf(nx, 64, 10.0, 1e-4, ncomp=2, proxy_cap=proxy_cap))
    H = H if dtype == np.complex128 else H.astype(dtype)
    X = random_rhs(H.n, nrhs, seed=4, dtype=dtype)
    return H, X
