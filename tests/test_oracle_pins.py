"""Pins of the CPU oracle (oracle/fem_oracle.c) to what the paper and the mathematics fix.

None of these tests re-types the oracle's formulas. Each pin is an independent route:
  * golden numbers printed in the paper/SPEC (tests/golden/paper_facts.txt);
  * exact rational integration of the trilinear basis (fractions.Fraction, separable 1-D
    integrals, no quadrature, no Jacobian code) -> element matrices of Eq. 4-6;
  * library identities: the assembled box operators equal Kronecker sums of 1-D FE matrices
    (scipy.sparse.kron), numpy dense solves for CG;
  * invariants: null spaces (constants, rigid-body modes), symmetry, spectra, finite termination.
A plausible mistake in the oracle (dropped term, wrong sign/index, transposed J) fails one of them.
"""
from __future__ import annotations

import math
import os
from fractions import Fraction
from itertools import product

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2308_09839_b200 import inputs as I

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CORNER = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]
SIGN = [tuple(2 * c - 1 for c in cc) for cc in CORNER]


def paper_facts():
    out = {}
    with open(os.path.join(GOLDEN, "paper_facts.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            key, val = line.split()[:2]
            out[key] = float(val)
    return out


# ------------------------------------------------------------------------------------------
# exact rational integrals R[p][q][i][j] = int_{[-1,1]^3} d_p phi_i d_q phi_j  (separable)
# ------------------------------------------------------------------------------------------
def _int1d(fa, fb):
    """int_{-1}^{1} fa(t) fb(t) dt for linear fa = (c0 + c1 t): exact rational."""
    a0, a1 = fa
    b0, b1 = fb
    # (a0 + a1 t)(b0 + b1 t) = a0 b0 + (a0 b1 + a1 b0) t + a1 b1 t^2
    return Fraction(2) * a0 * b0 + Fraction(2, 3) * a1 * b1


def _factor(i, d, deriv):
    s = SIGN[i][d]
    if deriv:
        return (Fraction(s, 2), Fraction(0))
    return (Fraction(1, 2), Fraction(s, 2))


def exact_R():
    R = [[[[None] * 8 for _ in range(8)] for _ in range(3)] for _ in range(3)]
    for p, q, i, j in product(range(3), range(3), range(8), range(8)):
        v = Fraction(1)
        for d in range(3):
            v *= _int1d(_factor(i, d, d == p), _factor(j, d, d == q))
        R[p][q][i][j] = v
    return R


R_EXACT = exact_R()
R_NP = np.array([[[[float(R_EXACT[p][q][i][j]) for j in range(8)] for i in range(8)]
                  for q in range(3)] for p in range(3)])


def exact_elem_scalar(A):
    """K_ij = |det A| sum_pq (A^-1 A^-T)_pq R_pq(i,j) for the affine map x = A xi + b."""
    Ai = np.linalg.inv(A)
    Gm = Ai @ Ai.T
    return abs(np.linalg.det(A)) * np.einsum("pq,pqij->ij", Gm, R_NP)


def exact_elem_elastic(A, lam, mu):
    """K_{3i+k,3j+l} = int lam d_k phi_i d_l phi_j + mu(delta_kl grad phi_i.grad phi_j + d_l phi_i d_k phi_j)."""
    AiT = np.linalg.inv(A).T  # d_k phi = sum_p AiT[k,p] d^_p phi^
    det = abs(np.linalg.det(A))
    K = np.zeros((24, 24))
    S = exact_elem_scalar(A)
    for k in range(3):
        for l in range(3):
            lam_t = np.einsum("p,q,pqij->ij", AiT[k], AiT[l], R_NP)
            mu_t = np.einsum("p,q,pqij->ij", AiT[l], AiT[k], R_NP)
            blk = det * (lam * lam_t + mu * mu_t) + (mu * S if k == l else 0.0)
            K[k::3, l::3] = blk
    return K


def affine_nodes(A, b0):
    return np.array([A @ np.array(s, float) + b0 for s in SIGN])


# ------------------------------------------------------------------------------------------
# 1-D assembled FE matrices for the Kronecker identities
# ------------------------------------------------------------------------------------------
def fe1d(n, h):
    K = sp.lil_matrix((n + 1, n + 1)); M = sp.lil_matrix((n + 1, n + 1)); D = sp.lil_matrix((n + 1, n + 1))
    Ke = np.array([[1, -1], [-1, 1]]) / h
    Me = np.array([[2, 1], [1, 2]]) * h / 6
    De = 0.5 * np.array([[-1, 1], [-1, 1]])  # D_ij = int phi_i phi_j'
    for e in range(n):
        for a in range(2):
            for b in range(2):
                K[e + a, e + b] += Ke[a, b]; M[e + a, e + b] += Me[a, b]; D[e + a, e + b] += De[a, b]
    return K.tocsr(), M.tocsr(), D.tocsr()


def kron3(Az, Ay, Ax):
    return sp.kron(Az, sp.kron(Ay, Ax)).tocsr()


def scalar_kron(nx, ny, nz, h):
    Kx, Mx, _ = fe1d(nx, h); Ky, My, _ = fe1d(ny, h); Kz, Mz, _ = fe1d(nz, h)
    return kron3(Kz, My, Mx) + kron3(Mz, Ky, Mx) + kron3(Mz, My, Kx)


def elastic_kron(nx, ny, nz, h, lam, mu):
    one = [fe1d(nx, h), fe1d(ny, h), fe1d(nz, h)]  # per dim (K, M, D)

    def term(mats):  # mats[d] for d = x, y, z
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
                    return [one[d][2].T if d == dk else (one[d][2] if d == dl else one[d][1])
                            for d in range(3)]
                B = lam * term(pick(k, l)) + mu * term(pick(l, k))
            E = sp.csr_matrix(([1.0], ([k], [l])), shape=(3, 3))
            A = A + sp.kron(B, E)
    return A.tocsr()


# ==========================================================================================
# 1. reference element
# ==========================================================================================
def test_reference_element_facts(oracle):
    facts = paper_facts()
    xq, wq, dphi, phi = oracle.reference_element()
    assert wq.sum() == facts["gauss_weight_sum"]
    assert np.allclose(xq[0], facts["gauss_point_0"], atol=0, rtol=1e-15)
    g0 = oracle.basis_gradients([0.0, 0.0, 0.0])
    assert np.all(g0[0] == facts["grad_node0_at_origin"])
    # partition of unity and its gradient at random points
    r = np.random.default_rng(0)
    for _ in range(20):
        xi = r.uniform(-1, 1, 3)
        assert abs(oracle.basis_values(xi).sum() - 1) < 1e-15
        assert np.abs(oracle.basis_gradients(xi).sum(axis=0)).max() < 1e-15
    # Kronecker property at the nodes
    for a, s in enumerate(SIGN):
        v = oracle.basis_values(np.array(s, float))
        assert np.array_equal(v, np.eye(8)[a])


def test_reference_gradients_finite_difference(oracle):
    r = np.random.default_rng(1)
    for _ in range(10):
        xi = r.uniform(-1, 1, 3)
        g = oracle.basis_gradients(xi)
        for d in range(3):
            e = np.zeros(3); e[d] = 1e-6
            fd = (oracle.basis_values(xi + e) - oracle.basis_values(xi - e)) / 2e-6
            assert np.abs(fd - g[:, d]).max() < 1e-8


def test_gauss_rule_exact_for_cubic_monomials(oracle):
    xq, wq, _, _ = oracle.reference_element()
    for a, b, c in product(range(4), repeat=3):
        exact = 1.0
        for p in (a, b, c):
            exact *= 0.0 if p % 2 else 2.0 / (p + 1)
        got = np.sum(wq * xq[:, 0] ** a * xq[:, 1] ** b * xq[:, 2] ** c)
        assert abs(got - exact) < 1e-14


# ==========================================================================================
# 2. element matrices vs exact rational integration (Eq. 4-6)
# ==========================================================================================
def test_scalar_unit_cube_closed_form(oracle):
    G = np.loadtxt(os.path.join(GOLDEN, "q1_laplace_unit_cube.txt"))
    # exact rational route: J = I/2 on the unit cube -> K = det(J) * 4 * sum_p R_pp
    Kex = [[sum(R_EXACT[p][p][i][j] for p in range(3)) * Fraction(1, 2) for j in range(8)]
           for i in range(8)]
    assert all(Kex[i][j] * 12 == int(G[i, j]) for i in range(8) for j in range(8))
    X = np.array(CORNER, float)
    K = oracle.element_matrix("scalar", X)
    assert np.abs(K - G / 12).max() < 1e-15
    for h in (0.25, 3.0):
        assert np.abs(oracle.element_matrix("scalar", X * h) - h * G / 12).max() < 1e-14 * h


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_element_matrices_sheared_affine(oracle, seed):
    """Non-symmetric affine map: catches transposed J / J^-T / index slips in Eq. 4-6."""
    r = np.random.default_rng(100 + seed)
    A = np.diag(r.uniform(0.5, 1.5, 3)) + 0.3 * r.uniform(-1, 1, (3, 3))
    assert np.linalg.det(A) > 0
    X = affine_nodes(A, r.uniform(-1, 1, 3))
    lam, mu = r.uniform(0.5, 3.0), r.uniform(0.2, 2.0)
    Ks = oracle.element_matrix("scalar", X)
    assert np.abs(Ks - exact_elem_scalar(A)).max() < 1e-13
    Kv = oracle.element_matrix("vector", X)
    assert np.abs(Kv - np.kron(exact_elem_scalar(A), np.eye(3))).max() < 1e-13
    Ke = oracle.element_matrix("elastic", X, lam, mu)
    Kref = exact_elem_elastic(A, lam, mu)
    assert np.abs(Ke - Kref).max() < 1e-13 * np.abs(Kref).max()


def test_elastic_unit_cube_diagonals(oracle):
    """unit cube, diag K_lambda = 1/9, diag K_mu = 4/9; spectra."""
    X = np.array(CORNER, float)
    Kl = oracle.element_matrix("elastic", X, 1.0, 0.0)
    Km = oracle.element_matrix("elastic", X, 0.0, 1.0)
    assert np.abs(np.diag(Kl) - 1 / 9).max() < 1e-15
    assert np.abs(np.diag(Km) - 4 / 9).max() < 1e-15
    el = np.sort(np.linalg.eigvalsh(Kl))
    exp_l = np.sort([0.0] * 17 + [1 / 18] * 3 + [1 / 3] * 3 + [1.5])
    assert np.abs(el - exp_l).max() < 1e-13
    em = np.sort(np.linalg.eigvalsh(Km))
    exp_m = np.sort([0.0] * 6 + [1 / 6] * 2 + [2 / 9] * 3 + [0.5] * 6 + [2 / 3] + [1.0] * 6)
    assert np.abs(em - exp_m).max() < 1e-13


# ==========================================================================================
# 3. assembled operators: Kronecker identities (library routine), dense brute force
# ==========================================================================================
def test_scalar_apply_equals_kronecker_sum(oracle):
    nx, ny, nz, h = 4, 3, 2, 0.37
    A = scalar_kron(nx, ny, nz, h)
    x = np.random.default_rng(3).uniform(-1, 1, A.shape[0])
    y = oracle.apply("scalar", 0, nx, ny, nz, h, x)
    assert np.abs(y - A @ x).max() < 1e-14 * np.abs(A @ x).max() * 10
    # interior stencil values: centre 8h/3, face 0, edge -h/6, corner -h/12
    Ad = A.toarray()
    n = 1 + 5 * (1 + 4 * 1)  # node (1,1,1)
    assert abs(Ad[n, n] - 8 * h / 3) < 1e-15
    assert abs(Ad[n, n + 1]) < 1e-16
    assert abs(Ad[n, n + 1 + 5] + h / 6) < 1e-15
    assert abs(Ad[n, n + 1 + 5 + 20] + h / 12) < 1e-15


def test_vector_apply_is_block_diagonal(oracle):
    nx, ny, nz, h = 3, 2, 2, 0.5
    A = scalar_kron(nx, ny, nz, h)
    x = np.random.default_rng(4).uniform(-1, 1, 3 * A.shape[0])
    y = oracle.apply("vector", 0, nx, ny, nz, h, x)
    for c in range(3):
        assert np.abs(y[c::3] - A @ x[c::3]).max() < 1e-14


def test_elastic_constant_material_equals_kronecker(oracle):
    nx, ny, nz, h, lam, mu = 3, 2, 2, 0.41, 1.7, 0.6
    A = elastic_kron(nx, ny, nz, h, lam, mu)
    x = np.random.default_rng(5).uniform(-1, 1, A.shape[0])
    y = oracle.apply("elastic", 0, nx, ny, nz, h, x, lam=lam, mu=mu)
    ref = A @ x
    assert np.abs(y - ref).max() < 1e-13 * np.abs(ref).max()
    # centre block 8h(lam+4mu)/9 I3 on a mesh with an interior node
    B = elastic_kron(2, 2, 2, h, lam, mu).toarray()
    n = 13
    assert np.abs(B[3 * n:3 * n + 3, 3 * n:3 * n + 3] - 8 * h * (lam + 4 * mu) / 9 * np.eye(3)).max() < 1e-14


@pytest.mark.parametrize("dims", [(2, 2, 2), (3, 2, 2)])
def test_elastic_cellwise_dense_brute_force(oracle, dims):
    """Scatter of exact (rational-integrated) element matrices with cell-wise lambda, mu."""
    nx, ny, nz = dims
    h = 0.5
    g = np.random.default_rng(6)
    lam, mu = I.lognormal_materials(g, nx, ny, nz)
    Kl = exact_elem_elastic(np.eye(3) * h / 2, 1.0, 0.0)
    Km = exact_elem_elastic(np.eye(3) * h / 2, 0.0, 1.0)
    nn = (nx + 1) * (ny + 1) * (nz + 1)
    A = np.zeros((3 * nn, 3 * nn))
    for k, j, i in product(range(nz), range(ny), range(nx)):
        e = i + nx * (j + ny * k)
        nid = [(i + c[0]) + (nx + 1) * ((j + c[1]) + (ny + 1) * (k + c[2])) for c in CORNER]
        dof = np.array([3 * n + c for n in nid for c in range(3)])
        A[np.ix_(dof, dof)] += lam[e] * Kl + mu[e] * Km
    Ad = oracle.assemble_dense("elastic", 0, nx, ny, nz, h, lam, mu)
    assert np.abs(Ad - A).max() < 1e-13 * np.abs(A).max()
    x = g.uniform(-1, 1, 3 * nn)
    y = oracle.apply("elastic", 0, nx, ny, nz, h, x, lam=lam, mu=mu)
    assert np.abs(y - A @ x).max() < 1e-13 * np.abs(A @ x).max()
    # Dirichlet: y = P A P x + (I - P) x
    bm = np.repeat(I.boundary_mask(nx, ny, nz), 3)
    P = np.diag((~bm).astype(float))
    Ac = P @ A @ P + np.diag(bm.astype(float))
    yc = oracle.apply("elastic", 1, nx, ny, nz, h, x, lam=lam, mu=mu)
    assert np.abs(yc - Ac @ x).max() < 1e-13 * np.abs(Ac @ x).max()
    assert np.array_equal(yc[bm], x[bm])


def test_dirichlet_2x2x2_spectrum(oracle):
    """2x2x2 at h = 1/2, one interior node: constrained spectrum {1, 4/3}."""
    A = oracle.assemble_dense("scalar", 1, 2, 2, 2, 0.5)
    ev = np.unique(np.round(np.linalg.eigvalsh(A), 12))
    assert np.allclose(ev, [1.0, 4.0 / 3.0])


# ==========================================================================================
# 4. invariants: null spaces, symmetry
# ==========================================================================================
def rigid_body_modes(nx, ny, nz, h):
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    X = np.stack([i.ravel() * h, j.ravel() * h, k.ravel() * h], axis=1)
    modes = []
    for d in range(3):
        m = np.zeros_like(X); m[:, d] = 1; modes.append(m.ravel())
    for W in ([[0, -1, 0], [1, 0, 0], [0, 0, 0]], [[0, 0, -1], [0, 0, 0], [1, 0, 0]],
              [[0, 0, 0], [0, 0, -1], [0, 1, 0]]):
        modes.append((X @ np.array(W, float).T).ravel())
    return modes


def test_null_spaces(oracle):
    nx, ny, nz, h = 4, 3, 5, 0.3
    nn = (nx + 1) * (ny + 1) * (nz + 1)
    y = oracle.apply("scalar", 0, nx, ny, nz, h, np.ones(nn))
    assert np.abs(y).max() < 1e-14
    y = oracle.apply("vector", 0, nx, ny, nz, h, np.ones(3 * nn))
    assert np.abs(y).max() < 1e-14
    lam, mu = I.materials(np.random.default_rng(7), nx, ny, nz)
    scale = (lam + 2 * mu).max() * h * 16
    for m in rigid_body_modes(nx, ny, nz, h):
        y = oracle.apply("elastic", 0, nx, ny, nz, h, m, lam=lam, mu=mu)
        assert np.abs(y).max() < 1e-13 * scale


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("bc", [0, 1])
def test_symmetry(oracle, kind, bc):
    nx, ny, nz, h = 5, 4, 3, 0.2
    c = I.ncomp(kind)
    g = np.random.default_rng(8)
    lam, mu = I.materials(g, nx, ny, nz)
    x = I.uniform_vector(g, nx, ny, nz, c); z = I.uniform_vector(g, nx, ny, nz, c)
    ax = oracle.apply(kind, bc, nx, ny, nz, h, x, lam=lam, mu=mu)
    az = oracle.apply(kind, bc, nx, ny, nz, h, z, lam=lam, mu=mu)
    assert abs(z @ ax - x @ az) < 1e-13 * (np.abs(z) @ np.abs(ax))


def test_paper_mesh_counts(oracle):
    def oracle_dense_elastic(m, lam, mu):
        return oracle.assemble_dense("elastic", 0, m, m, m, 1.0 / m, lam, mu)

    facts = paper_facts()
    assert I.n_nodes(100, 100, 100) == facts["nodes_1e6_hexes"]
    assert 3 * I.n_nodes(100, 100, 100) == facts["rows_mechanics_1e6"]
    assert I.boundary_mask(100, 100, 100).sum() == facts["boundary_nodes_100cube"]
    # interior-row nnz of the assembled operators (Table 1): structural 27 / 81
    # (pattern = union of the 1-D K, M couplings; the face entries cancel numerically)
    K1, M1, _ = fe1d(4, 0.25)
    pat1 = (abs(K1) + abs(M1)).tocsr()
    S = kron3(pat1, pat1, pat1)
    n = 2 + 5 * (2 + 5 * 2)
    assert S[n].count_nonzero() == facts["nnz_per_row_scalar"]
    assert 3 * S[n].count_nonzero() == facts["nnz_per_row_mechanics"]
    # elasticity: every one of the 81 structural couplings of an interior row is carried by
    # some element matrix entry (the oracle's dense assembly, random material)
    lam, mu = I.materials(np.random.default_rng(13), 4, 4, 4)
    A = np.abs(oracle_dense_elastic(4, lam, mu))
    assert A[3 * n].reshape(-1, 3).any(axis=1).sum() * 3 == facts["nnz_per_row_mechanics"]


# ==========================================================================================
# 5. dot and CG (Table 4 recurrences)
# ==========================================================================================
def test_dot(oracle):
    assert oracle.dot(np.ones(8), np.ones(8)) == 8.0
    b = np.random.default_rng(9).uniform(-1, 1, 10)
    e3 = np.zeros(10); e3[3] = 1
    assert oracle.dot(e3, b) == b[3]
    a = np.random.default_rng(10).uniform(-1, 1, 100000)
    c = np.random.default_rng(11).uniform(-1, 1, 100000)
    exact = math.fsum(float(Fraction(u) * Fraction(v)) for u, v in zip(a[:2000], c[:2000]))
    assert abs(oracle.dot(a[:2000], c[:2000]) - exact) < 1e-15


def test_cg_manufactured_solution_c1(oracle):
    nx = ny = nz = 8; h = 1 / 8
    g = I.rng(I.SEED_BASE + 0)
    xs = I.interior_rhs(g, nx, ny, nz, 1)  # x* random interior, 0 on boundary
    A = scalar_kron(nx, ny, nz, h).toarray()
    bm = I.boundary_mask(nx, ny, nz)
    P = np.diag((~bm).astype(float))
    Ac = P @ A @ P + np.diag(bm.astype(float))
    b = Ac @ xs
    res = oracle.cg("scalar", 1, nx, ny, nz, h, b, tol=0.0, maxit=50)
    assert np.abs(res.x - xs).max() < 1e-13
    assert np.abs(res.x - np.linalg.solve(Ac, b)).max() < 1e-13
    rel = res.res_hist / res.res_hist[0]
    assert np.argmax(rel < 1e-8) <= 20 and np.argmax(rel < 1e-14) <= 30
    # scale invariance of the iteration count
    r1 = oracle.cg("scalar", 1, nx, ny, nz, h, b, tol=1e-10, maxit=200)
    r2 = oracle.cg("scalar", 1, nx, ny, nz, h, 1e3 * b, tol=1e-10, maxit=200)
    assert r1.converged and r2.converged and r1.iterations == r2.iterations


def test_cg_single_interior_dof_terminates(oracle):
    """2x2x2 Dirichlet: b vanishing on constrained DOFs -> exactly one iteration."""
    b = np.zeros(27); b[13] = 0.7
    res = oracle.cg("scalar", 1, 2, 2, 2, 0.5, b, tol=1e-14, maxit=10)
    assert res.converged and res.iterations == 1
    assert abs(res.x[13] - 0.7 / (4 / 3)) < 1e-15


def test_cg_elastic_matches_dense_solve(oracle):
    nx, ny, nz, h = 3, 3, 2, 0.5
    g = np.random.default_rng(12)
    lam, mu = I.materials(g, nx, ny, nz)
    b = I.interior_rhs(g, nx, ny, nz, 3)
    Ac = oracle.assemble_dense("elastic", 1, nx, ny, nz, h, lam, mu)
    res = oracle.cg("elastic", 1, nx, ny, nz, h, b, tol=1e-14, maxit=500, lam=lam, mu=mu)
    assert res.converged
    xs = np.linalg.solve(Ac, b)
    assert np.abs(res.x - xs).max() < 1e-10 * np.abs(xs).max()


@pytest.mark.parametrize("kind", ["scalar", "elastic"])
def test_cg_iterates_are_krylov_galerkin_solutions(oracle, kind):
    """CG optimality (P:185 Krylov method): with x0 = 0, the k-th iterate is the A-orthogonal
    (Galerkin) projection of x* onto K_k(A, b) = span{b, Ab, ..., A^{k-1} b}. Computed here by a
    dense orthonormal Krylov basis + small solve, independent of the CG recurrences."""
    nx, ny, nz, h = 4, 3, 3, 0.25
    g = np.random.default_rng(21)
    c = I.ncomp(kind)
    lam, mu = I.materials(g, nx, ny, nz)
    A = oracle.assemble_dense(kind, 1, nx, ny, nz, h, lam, mu)
    b = I.interior_rhs(g, nx, ny, nz, c)
    for k in (1, 2, 3, 5, 8):
        V = [b / np.linalg.norm(b)]
        for _ in range(k - 1):
            w = A @ V[-1]
            for v in V:  # two passes of Gram-Schmidt
                w -= (v @ w) * v
            for v in V:
                w -= (v @ w) * v
            V.append(w / np.linalg.norm(w))
        V = np.array(V).T
        xk = V @ np.linalg.solve(V.T @ A @ V, V.T @ b)
        res = oracle.cg(kind, 1, nx, ny, nz, h, b, tol=0.0, maxit=k, lam=lam, mu=mu)
        assert res.iterations == k
        assert np.abs(res.x - xk).max() < 1e-11 * np.abs(xk).max()


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("bc", [0, 1])
def test_apply_nodes_equals_full_apply(oracle, kind, bc):
    """The sampled-node oracle is the same definition restricted to the cells around a node."""
    nx, ny, nz, h = 6, 5, 4, 0.3
    g = np.random.default_rng(30)
    c = I.ncomp(kind)
    lam, mu = I.materials(g, nx, ny, nz)
    x = I.uniform_vector(g, nx, ny, nz, c)
    y = oracle.apply(kind, bc, nx, ny, nz, h, x, lam=lam, mu=mu).reshape(-1, c)
    nodes = np.arange(I.n_nodes(nx, ny, nz))
    ys = oracle.apply_nodes(kind, bc, nx, ny, nz, h, x, nodes, lam=lam, mu=mu)
    assert np.abs(ys - y).max() <= 1e-13 * np.abs(y).max()
