"""Pins of the oracle's GLL rule (2-point Gauss-Lobatto, collocated with the Q1 nodes: the
quadrature of the CEED benchmark problems BP5/BP6 the paper names, P:581, P:638, P:664-668;
SURVEY §8(c) item 1, reading R1).

Independent routes: the unit-cube element matrix of SURVEY App. A (K = (1/4)[3 on the diagonal,
-1 between edge neighbours, 0 otherwise]); Kronecker sums with the LUMPED 1-D mass h/2 diag(m)
(scipy.sparse.kron; the 1-D stiffness and the 1-D phi phi' matrix are exact under 2-point GLL);
null spaces, symmetry and rotation covariance on deformed cells (valid for any rule).
"""
from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2308_09839_b200 import inputs as I

CORNER = np.array(I.VTK_CORNERS, float)


def fe1d_gll(n, h):
    K = sp.lil_matrix((n + 1, n + 1)); M = sp.lil_matrix((n + 1, n + 1)); D = sp.lil_matrix((n + 1, n + 1))
    Ke = np.array([[1, -1], [-1, 1]]) / h
    Me = np.array([[1, 0], [0, 1]]) * h / 2          # lumped (nodal quadrature)
    De = 0.5 * np.array([[-1, 1], [-1, 1]])          # int phi_i phi_j' (exact under GLL)
    for e in range(n):
        for a in range(2):
            for b in range(2):
                K[e + a, e + b] += Ke[a, b]; M[e + a, e + b] += Me[a, b]; D[e + a, e + b] += De[a, b]
    return K.tocsr(), M.tocsr(), D.tocsr()


def kron3(Az, Ay, Ax):
    return sp.kron(Az, sp.kron(Ay, Ax)).tocsr()


def test_gll_unit_cube_element(oracle):
    diff = np.abs(CORNER[:, None, :] - CORNER[None, :, :]).sum(-1)
    Kex = np.where(diff == 0, 3.0, np.where(diff == 1, -1.0, 0.0)) / 4
    with oracle.quadrature("gll"):
        K = oracle.element_matrix("scalar", CORNER)
        K2 = oracle.element_matrix("scalar", CORNER * 0.5)
    assert np.abs(K - Kex).max() < 1e-15
    assert np.abs(K2 - 0.5 * Kex).max() < 1e-15
    # and the default rule is untouched afterwards
    assert abs(oracle.element_matrix("scalar", CORNER)[0, 0] - 1 / 3) < 1e-15


def test_gll_scalar_box_is_lumped_kronecker_sum(oracle):
    nx, ny, nz, h = 4, 3, 2, 0.3
    Kx, Mx, _ = fe1d_gll(nx, h); Ky, My, _ = fe1d_gll(ny, h); Kz, Mz, _ = fe1d_gll(nz, h)
    A = kron3(Kz, My, Mx) + kron3(Mz, Ky, Mx) + kron3(Mz, My, Kx)
    x = np.random.default_rng(0).uniform(-1, 1, A.shape[0])
    with oracle.quadrature("gll"):
        y = oracle.apply("scalar", 0, nx, ny, nz, h, x)
        yv = oracle.apply("vector", 0, nx, ny, nz, h, np.repeat(x, 3))
    assert np.abs(y - A @ x).max() < 1e-13
    assert np.abs(yv - np.repeat(A @ x, 3)).max() < 1e-13
    # interior stencil: 7 points, 6h at the centre, -h at the face neighbours
    assert np.count_nonzero(np.abs(A.toarray()[A.shape[0] // 2]) > 1e-14) <= 7


def test_gll_elastic_constant_material_kronecker(oracle):
    nx, ny, nz, h, lam, mu = 3, 2, 2, 0.5, 1.3, 0.7
    one = [fe1d_gll(nx, h), fe1d_gll(ny, h), fe1d_gll(nz, h)]

    def term(mats):
        return kron3(mats[2], mats[1], mats[0])

    nn = (nx + 1) * (ny + 1) * (nz + 1)
    A = sp.csr_matrix((3 * nn, 3 * nn))
    for k in range(3):
        for l in range(3):
            if k == l:
                B = (lam + 2 * mu) * term([one[d][0] if d == k else one[d][1] for d in range(3)])
                for j in range(3):
                    if j != k:
                        B = B + mu * term([one[d][0] if d == j else one[d][1] for d in range(3)])
            else:
                def pick(dk, dl):
                    return [one[d][2].T if d == dk else (one[d][2] if d == dl else one[d][1]) for d in range(3)]
                B = lam * term(pick(k, l)) + mu * term(pick(l, k))
            A = A + sp.kron(B, sp.csr_matrix(([1.0], ([k], [l])), shape=(3, 3)))
    x = np.random.default_rng(1).uniform(-1, 1, 3 * nn)
    with oracle.quadrature("gll"):
        y = oracle.apply("elastic", 0, nx, ny, nz, h, x, lam=lam, mu=mu)
    assert np.abs(y - A @ x).max() < 1e-13 * np.abs(A @ x).max()


@pytest.mark.parametrize("kind", ["scalar", "elastic"])
def test_gll_deformed_invariants(oracle, kind):
    g = I.rng(I.SEED_BASE + 990)
    coords, cells, _ = I.hex_box_mesh(3, 3, 2, g=g, jitter=0.2)
    lam, mu = 10 ** g.uniform(-1, 1, cells.shape[0]), 10 ** g.uniform(-1, 1, cells.shape[0])
    n = coords.shape[0]; c = I.ncomp(kind)
    with oracle.quadrature("gll"):
        if kind == "scalar":
            assert np.abs(oracle.apply_hex(kind, coords, cells, np.ones(n))).max() < 1e-13
        else:
            W = np.array([[0, -1, 0], [1, 0, 0], [0, 0, 0]])
            for m in (np.tile([1.0, 0, 0], n), (coords @ W.T).ravel()):
                assert np.abs(oracle.apply_hex(kind, coords, cells, m, None, lam, mu)).max() < 1e-12
        A = np.stack([oracle.apply_hex(kind, coords, cells, e, None, lam, mu) for e in np.eye(n * c)], 1)
        assert np.abs(A - A.T).max() < 1e-14 * np.abs(A).max()
        Q, _ = np.linalg.qr(np.random.default_rng(3).normal(size=(3, 3)))
        if np.linalg.det(Q) < 0:
            Q[:, 0] = -Q[:, 0]
        x = np.random.default_rng(4).uniform(-1, 1, n * c)
        if kind == "scalar":
            yr = oracle.apply_hex(kind, coords @ Q.T, cells, x)
            assert np.abs(yr - A @ x).max() < 1e-13 * np.abs(A @ x).max()
        else:
            yr = oracle.apply_hex(kind, coords @ Q.T, cells, (x.reshape(n, 3) @ Q.T).ravel(), None, lam, mu)
            ref = ((A @ x).reshape(n, 3) @ Q.T).ravel()
            assert np.abs(yr - ref).max() < 1e-13 * np.abs(ref).max()


def test_gll_differs_from_gauss(oracle):
    x = np.random.default_rng(5).uniform(-1, 1, 27)
    a = oracle.apply("scalar", 0, 2, 2, 2, 0.5, x)
    with oracle.quadrature("gll"):
        b = oracle.apply("scalar", 0, 2, 2, 2, 0.5, x)
    assert np.abs(a - b).max() > 1e-2
