"""Pins of the oracle's general-hexahedron path (orc_apply_hex / orc_cg_hex: Alg. 1 as written,
P:311-360, explicit node map + nodal coordinates, J recomputed per quadrature point).

Independent routes only (none re-types the oracle's quadrature):
  * the box oracle (already pinned by test_oracle_pins.py) on an undeformed lattice;
  * invariants of the continuous problem that 2x2x2 Gauss keeps EXACTLY on trilinear cells:
    - constants / rigid-body modes in the null space (any geometry, any cell-wise lambda, mu);
    - the patch test: for a linear field the interior rows vanish (the quadrature integrand
      cof(J) grad^phi has degree <= 3 per variable);
    - the energy of a linear field: u^T A_e u = vol(e) * |a|^2 (Laplace) or
      vol(e) * (lambda tr(B)^2 + 2 mu |sym B|^2) (elasticity), with vol(e) = int det J computed
      here by a 6-point Gauss rule on an independently written trilinear map (det J has degree
      <= 2 per variable, so both rules are exact);
  * covariance: rotating the mesh rotates the operator (scalar: invariant; elasticity:
    A(QX) = (I (x) Q) A(X) (I (x) Q)^T), scaling by s scales A by s -- a transposed J or a J^-1
    vs J^-T slip breaks these on non-affine cells;
  * relabelling nodes / reordering cells permutes the operator;
  * symmetry, semi-definiteness, and CG recovering a manufactured solution.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2308_09839_b200 import inputs as I


def mesh(n=(3, 2, 2), jitter=0.2, permute=False, seed=0):
    g = I.rng(I.SEED_BASE + 950 + seed)
    return I.hex_box_mesh(*n, h=1.0 / max(n), g=g, jitter=jitter, permute=permute)


def rot(seed=0):
    q, r = np.linalg.qr(np.random.default_rng(seed).normal(size=(3, 3)))
    q = q * np.sign(np.diag(r))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def mats(ncells, seed=0):
    g = np.random.default_rng(70 + seed)
    return 10 ** g.uniform(-1, 1, ncells), 10 ** g.uniform(-1, 1, ncells)


def dense(oracle, kind, coords, cells, dirichlet=None, lam=None, mu=None):
    c = 1 if kind == "scalar" else 3
    n = coords.shape[0] * c
    A = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n); e[j] = 1.0
        A[:, j] = oracle.apply_hex(kind, coords, cells, e, dirichlet, lam, mu)
    return A


def trilinear_volume(X):
    """int det J over [-1,1]^3 for the trilinear map through the 8 VTK-ordered nodes X, by a
    3-point-per-direction Gauss rule written independently of the oracle (exact: det J has
    degree <= 2 per variable)."""
    pts, wts = np.polynomial.legendre.leggauss(3)
    s = np.array(I.VTK_CORNERS, float) * 2 - 1
    vol = 0.0
    for a, wa in zip(pts, wts):
        for b, wb in zip(pts, wts):
            for c, wc in zip(pts, wts):
                xi = np.array([a, b, c])
                f = np.prod(0.5 * (1 + s * xi), axis=1)            # basis values
                J = np.zeros((3, 3))
                for d in range(3):                                   # d/dxi_d by the product rule
                    g = 0.5 * s[:, d] * np.prod(np.delete(0.5 * (1 + s * xi), d, axis=1), axis=1)
                    J[:, d] = X.T @ g
                del f
                vol += wa * wb * wc * np.linalg.det(J)
    return vol


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("bc", [0, 1])
def test_lattice_equals_box_oracle(oracle, kind, bc):
    nx, ny, nz = 4, 3, 2
    h = 1.0 / 4
    coords, cells, dirichlet = I.hex_box_mesh(nx, ny, nz, h=h)
    c = I.ncomp(kind)
    g = I.rng(I.SEED_BASE + 960)
    x = I.uniform_vector(g, nx, ny, nz, c)
    lam, mu = I.materials(g, nx, ny, nz)
    ref = oracle.apply(kind, bc, nx, ny, nz, h, x, lam=lam, mu=mu)
    y = oracle.apply_hex(kind, coords, cells, x, dirichlet if bc else None, lam, mu)
    assert np.abs(y - ref).max() <= 1e-14 * np.abs(ref).max()


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
def test_null_space_deformed(oracle, kind):
    coords, cells, _ = mesh(jitter=0.22)
    lam, mu = mats(cells.shape[0])
    n = coords.shape[0]
    if kind == "elastic":
        modes = [np.tile(np.eye(3)[d], n) for d in range(3)]
        for W in (np.array([[0, -1, 0], [1, 0, 0], [0, 0, 0]]), np.array([[0, 0, -1], [0, 0, 0], [1, 0, 0]]),
                  np.array([[0, 0, 0], [0, 0, -1], [0, 1, 0]])):
            modes.append((coords @ W.T).ravel())
        scale = 1e2
    else:
        modes = [np.ones(n * I.ncomp(kind))]
        scale = 10.0
    for m in modes:
        y = oracle.apply_hex(kind, coords, cells, m, None, lam, mu)
        assert np.abs(y).max() < 1e-13 * scale


@pytest.mark.parametrize("kind", ["scalar", "elastic"])
def test_patch_test_linear_field(oracle, kind):
    """Linear u on non-affine cells: interior rows of A u vanish (constant material)."""
    coords, cells, bnd = mesh(n=(4, 4, 3), jitter=0.22, seed=1)
    g = np.random.default_rng(5)
    if kind == "scalar":
        a = g.normal(size=3)
        u = coords @ a + 0.7
        lam = mu = None
    else:
        B = g.normal(size=(3, 3))
        u = (coords @ B.T + g.normal(size=3)).ravel()
        lam, mu = 1.7, 0.6
    y = oracle.apply_hex(kind, coords, cells, u, None, lam, mu)
    c = I.ncomp(kind)
    interior = np.repeat(bnd == 0, c)
    assert interior.sum() > 0
    assert np.abs(y[interior]).max() < 1e-13 * np.abs(y).max()
    assert np.abs(y[~interior]).max() > 1e-3  # boundary rows carry the flux


@pytest.mark.parametrize("kind", ["scalar", "elastic"])
def test_linear_field_energy_equals_volume(oracle, kind):
    """Per cell, u^T A_e u for a linear field = exact cell volume x the constant energy density."""
    coords, cells, _ = mesh(n=(2, 2, 2), jitter=0.23, seed=2)
    g = np.random.default_rng(9)
    for e in range(cells.shape[0]):
        X = coords[cells[e]]
        sub = cells[e:e + 1]
        vol = trilinear_volume(X)
        if kind == "scalar":
            a = g.normal(size=3)
            u = coords @ a
            dens = a @ a
            lam = mu = None
        else:
            B = g.normal(size=(3, 3))
            u = (coords @ B.T).ravel()
            lam, mu = g.uniform(0.5, 2), g.uniform(0.5, 2)
            S = 0.5 * (B + B.T)
            dens = lam * np.trace(B) ** 2 + 2 * mu * np.sum(S * S)
        y = oracle.apply_hex(kind, coords, sub, u, None, lam, mu)
        assert abs(u @ y - vol * dens) <= 1e-12 * vol * dens


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
def test_rotation_and_scaling_covariance(oracle, kind):
    coords, cells, _ = mesh(jitter=0.2, seed=3)
    lam, mu = mats(cells.shape[0], 3)
    n = coords.shape[0]; c = I.ncomp(kind)
    x = np.random.default_rng(11).uniform(-1, 1, n * c)
    y = oracle.apply_hex(kind, coords, cells, x, None, lam, mu)
    Q = rot(4)
    s = 2.5
    Xr = coords @ Q.T * s
    if kind == "elastic":
        xr = (x.reshape(n, 3) @ Q.T).ravel()
        yr = oracle.apply_hex(kind, Xr, cells, xr, None, lam, mu)
        ref = s * (y.reshape(n, 3) @ Q.T).ravel()
    else:
        yr = oracle.apply_hex(kind, Xr, cells, x, None, lam, mu)
        ref = s * y
    assert np.abs(yr - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("kind", ["scalar", "elastic"])
def test_relabelling_permutes_operator(oracle, kind):
    nx, ny, nz = 3, 2, 2
    g1 = I.rng(7); g2 = I.rng(7)
    c0, e0, d0 = I.hex_box_mesh(nx, ny, nz, g=g1, jitter=0.2)
    c1, e1, d1 = I.hex_box_mesh(nx, ny, nz, g=g2, jitter=0.2, permute=True)
    # recover the node relabelling from the coordinates and the cell map from node sets
    key0 = {tuple(np.round(p, 12)): i for i, p in enumerate(c0)}
    perm = np.array([key0[tuple(np.round(p, 12))] for p in c1])  # new label -> old label
    cellkey = {tuple(sorted(r)): k for k, r in enumerate(e0)}
    cmap = np.array([cellkey[tuple(sorted(perm[r]))] for r in e1])
    lam, mu = mats(e0.shape[0], 5)
    cc = I.ncomp(kind)
    x0 = np.random.default_rng(3).uniform(-1, 1, c0.shape[0] * cc)
    y0 = oracle.apply_hex(kind, c0, e0, x0, d0, lam, mu)
    idx = (perm[:, None] * cc + np.arange(cc)).ravel()
    x1 = x0[idx]
    y1 = oracle.apply_hex(kind, c1, e1, x1, d1, lam[cmap], mu[cmap])
    assert np.abs(y1 - y0[idx]).max() <= 1e-13 * np.abs(y0).max()


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
def test_symmetric_semidefinite_nullity(oracle, kind):
    coords, cells, bnd = mesh(n=(2, 2, 2), jitter=0.22, seed=6)
    lam, mu = mats(cells.shape[0], 6)
    A = dense(oracle, kind, coords, cells, None, lam, mu)
    assert np.abs(A - A.T).max() <= 1e-14 * np.abs(A).max()
    w = np.linalg.eigvalsh(0.5 * (A + A.T))
    tol = 1e-12 * w.max()
    assert w.min() > -tol
    assert int((w < tol).sum()) == {"scalar": 1, "vector": 3, "elastic": 6}[kind]
    Ac = dense(oracle, kind, coords, cells, bnd, lam, mu)
    assert np.linalg.eigvalsh(0.5 * (Ac + Ac.T)).min() > 0  # Dirichlet: SPD


def test_degenerate_cell_rejected(oracle):
    coords, cells, _ = mesh(n=(1, 1, 1), jitter=0.0)
    bad = coords.copy()
    bad[cells[0, 6]] = bad[cells[0, 0]] - 0.1  # fold the far corner through the cell
    with pytest.raises(ValueError):
        oracle.apply_hex("scalar", bad, cells, np.ones(8))


@pytest.mark.parametrize("kind", ["scalar", "elastic"])
def test_cg_manufactured_solution_deformed(oracle, kind):
    coords, cells, bnd = mesh(n=(5, 4, 4), jitter=0.2, permute=True, seed=8)
    lam, mu = mats(cells.shape[0], 8)
    c = I.ncomp(kind)
    g = np.random.default_rng(12)
    xs = g.uniform(-1, 1, coords.shape[0] * c)
    xs[np.repeat(bnd == 1, c)] = 0.0
    b = oracle.apply_hex(kind, coords, cells, xs, bnd, lam, mu)
    r = oracle.cg_hex(kind, coords, cells, b, bnd, tol=1e-14, maxit=2000, lam=lam, mu=mu)
    assert r.converged
    assert np.abs(r.x - xs).max() <= 1e-10
    assert r.true_r_norm <= 1e-12 * r.r0_norm
