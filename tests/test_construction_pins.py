"""Pins of the input-construction tooling (no GPU).

P4: butterflies / HOD-BF compressed by ID (Alg. 2) from the
oscillatory Helmholtz kernel on tiny point sets, densified by the oracle, match the
brute-force kernel matrix within 10 eps.  A wrong index anywhere in
the oracle's Eq. (3.1)-(3.2) reconstruction gives an O(1) error here.
A13: the dyadic kernel equals (I + grad grad / kappa^2) g by 4th-order differences.
"""
import numpy as np
import pytest

import oracle
from bfinputs.configs import helmholtz_planes_bf, helmholtz_plane_hodbf
from bfinputs.geometry import bisection_tree, dyadic, grid_points, helmholtz


def _brute_bf(bf):
    K = bf.meta["kernel"]
    return K(np.arange(K.shape[0]), np.arange(K.shape[1]))


@pytest.mark.parametrize("nx,leaf,eps", [(16, 16, 1e-6), (16, 8, 1e-4), (24, 16, 1e-6)])
def test_P4_helmholtz_planes_butterfly(nx, leaf, eps):
    bf = helmholtz_planes_bf(nx, leaf, ppw=8.0, sep=8.0, eps=eps)
    oracle.validate(bf)
    err = oracle.rel_err(oracle.bf_dense(bf), _brute_bf(bf))
    assert err <= 10 * eps, err


@pytest.mark.parametrize("nx,leaf,eps", [(32, 16, 1e-4), (16, 8, 1e-6)])
def test_P4_helmholtz_hodbf(nx, leaf, eps):
    H = helmholtz_plane_hodbf(nx, leaf, ppw=10.0, eps=eps)
    K = H.meta["kernel"]
    A = K(np.arange(H.n), np.arange(H.n))
    kappa = 2 * np.pi / 10.0
    np.testing.assert_allclose(np.diag(A), 1 + 1j * kappa)
    err = oracle.rel_err(oracle.hodbf_dense(H), A)
    assert err <= 10 * eps, err


def test_P4_dyadic_hodbf_small():
    H = helmholtz_plane_hodbf(8, 16, ppw=10.0, eps=1e-4, ncomp=2)
    K = H.meta["kernel"]
    A = K(np.arange(H.n), np.arange(H.n))
    assert oracle.rel_err(oracle.hodbf_dense(H), A) <= 1e-3


def test_A13_dyadic_vs_finite_differences():
    kappa = 2 * np.pi / 10.0
    rng = np.random.default_rng(0)
    P = rng.uniform(0, 20, size=(5, 3))
    P[:, 2] = 0
    Q = rng.uniform(0, 20, size=(4, 3))
    Q[:, 2] = 0
    G = dyadic(P, Q, kappa).reshape(5, 2, 4, 2)
    hstep = 1e-2

    def g(x):
        r = np.linalg.norm(x)
        return np.exp(1j * kappa * r) / (4 * np.pi * r)

    for a in range(5):
        for b in range(4):
            d = P[a] - Q[b]
            for s in range(2):
                for t in range(2):
                    es, et = np.eye(3)[s], np.eye(3)[t]
                    # 4th-order mixed/second derivative stencil
                    def f(i, j):
                        return g(d + i * hstep * es + j * hstep * et)
                    if s == t:
                        d2 = (-f(2, 0) + 16 * f(1, 0) - 30 * f(0, 0) + 16 * f(-1, 0) - f(-2, 0)) / (12 * hstep ** 2)
                    else:
                        c = np.array([1, -8, 0, 8, -1]) / (12 * hstep)
                        d2 = sum(c[i + 2] * c[j + 2] * f(i, j) for i in range(-2, 3) for j in range(-2, 3))
                    ref = (g(d) if s == t else 0) + d2 / kappa ** 2
                    assert abs(G[a, s, b, t] - ref) <= 1e-8 * abs(g(d))


def test_tree_bisection_shapes():
    perm, ptr = bisection_tree(64, 64, 6)
    assert len(ptr) == 65 and np.all(np.diff(ptr) == 64)
    assert np.array_equal(np.sort(perm), np.arange(4096))
    # first leaf is the lower-left 8x8 box
    P = grid_points(64, 64)[perm[:64]]
    assert P[:, 0].max() == 7 and P[:, 1].max() == 7
    perm, ptr = bisection_tree(160, 160, 10)
    assert np.all(np.diff(ptr) == 25)
