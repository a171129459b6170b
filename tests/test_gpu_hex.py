"""GPU parity of the general-hexahedron path (fem_mesh_create_hex; Alg. 1 as written) against the
oracle's orc_apply_hex / orc_cg_hex on the same seeded meshes (jittered, relabelled).

Tolerances as for the box path: apply ||y - y_ref||_inf / ||y_ref||_inf <= 1e-12;
CG solutions past 1e-13 relative residual within 1e-10.  The GPU scatter uses FP64 atomics, so
only the summation order of the <= 8 contributions per node differs from the oracle.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2308_09839_b200 import inputs as I

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

APPLY_TOL = 1e-12


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2308_09839_b200 import fem
    fem.load()
    return fem


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def relerr(y, ref):
    return float(np.abs(y - ref).max() / max(np.abs(ref).max(), 1e-300))


def make(n, jitter, permute, seed):
    g = I.rng(I.SEED_BASE + 1100 + seed)
    coords, cells, bnd = I.hex_box_mesh(*n, h=1.0 / max(n), g=g, jitter=jitter, permute=permute)
    lam, mu = I.materials(g, cells.shape[0], 1, 1)
    return coords, cells, bnd, lam, mu


CASES = [((1, 1, 1), 0.0, False), ((3, 2, 2), 0.2, False), ((5, 4, 3), 0.22, True),
         ((17, 9, 6), 0.2, True), ((33, 32, 5), 0.15, False)]


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("bc", [0, 1])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_hex_apply_parity(F, oracle, kind, bc, case):
    n, jit, perm = CASES[case]
    coords, cells, bnd, lam, mu = make(n, jit, perm, case)
    c = I.ncomp(kind)
    x = np.random.default_rng(case).uniform(-1, 1, coords.shape[0] * c)
    ref = oracle.apply_hex(kind, coords, cells, x, bnd if bc else None, lam, mu)
    mesh = F.HexMesh(dev(coords), dev(cells), dev(bnd))
    op = F.Operator(mesh, kind, bc)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    y = op.apply(dev(x)).cpu().numpy()
    assert relerr(y, ref) <= APPLY_TOL
    if bc:
        m = np.repeat(bnd == 1, c)
        assert np.array_equal(y[m], x[m])


def test_hex_host_pointers(F, oracle):
    coords, cells, bnd, lam, mu = make((4, 3, 3), 0.2, True, 7)
    mesh = F.HexMesh(coords, cells, bnd)  # host arrays
    op = F.Operator(mesh, "elastic", 1)
    op.set_material(lam, mu)
    x = np.random.default_rng(1).uniform(-1, 1, coords.shape[0] * 3)
    y = op.apply(x)
    assert relerr(y, oracle.apply_hex("elastic", coords, cells, x, bnd, lam, mu)) <= APPLY_TOL


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
def test_hex_lattice_equals_box_kernels(F, kind):
    """Two GPU paths, one operator: the explicit mesh of an undeformed box against the structured
    tensor-product / modal kernels."""
    nx, ny, nz = 20, 12, 9
    h = 1.0 / 20
    coords, cells, bnd = I.hex_box_mesh(nx, ny, nz, h=h)
    g = I.rng(I.SEED_BASE + 1200)
    lam, mu = I.materials(g, nx, ny, nz)
    c = I.ncomp(kind)
    x = dev(I.uniform_vector(g, nx, ny, nz, c))
    box = F.Operator(F.Mesh(nx, ny, nz, h), kind, 1)
    hexo = F.Operator(F.HexMesh(dev(coords), dev(cells), dev(bnd)), kind, 1)
    if kind == "elastic":
        box.set_material(dev(lam), dev(mu))
        hexo.set_material(dev(lam), dev(mu))
    y1 = box.apply(x).cpu().numpy()
    y2 = hexo.apply(x).cpu().numpy()
    assert relerr(y2, y1) <= APPLY_TOL


def test_hex_null_space_deformed(F):
    coords, cells, _, lam, mu = make((6, 5, 4), 0.22, True, 3)
    op = F.Operator(F.HexMesh(dev(coords), dev(cells)), "elastic", 0)
    op.set_material(dev(lam), dev(mu))
    n = coords.shape[0]
    modes = [np.tile(np.eye(3)[d], n) for d in range(3)]
    for W in (np.array([[0, -1, 0], [1, 0, 0], [0, 0, 0]]), np.array([[0, 0, -1], [0, 0, 0], [1, 0, 0]])):
        modes.append((coords @ W.T).ravel())
    scale = (lam + 2 * mu).max()
    for m in modes:
        assert np.abs(op.apply(dev(m)).cpu().numpy()).max() < 1e-12 * scale


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
def test_hex_cg_parity(F, oracle, kind):
    coords, cells, bnd, lam, mu = make((9, 8, 7), 0.2, True, 11)
    c = I.ncomp(kind)
    g = np.random.default_rng(21)
    b = g.uniform(-1, 1, coords.shape[0] * c)
    b[np.repeat(bnd == 1, c)] = 0.0
    ref = oracle.cg_hex(kind, coords, cells, b, bnd, tol=1e-14, maxit=3000, lam=lam, mu=mu)
    assert ref.converged
    op = F.Operator(F.HexMesh(dev(coords), dev(cells), dev(bnd)), kind, 1)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    x = torch.zeros(b.size, dtype=torch.float64, device="cuda")
    info = op.cg_solve(dev(b), x, tol=1e-14, maxit=3000)
    assert info["converged"]
    assert abs(info["iterations"] - ref.iterations) <= max(3, ref.iterations // 50)
    assert np.abs(x.cpu().numpy() - ref.x).max() <= 1e-10 * max(1.0, np.abs(ref.x).max())
    assert info["true_r_norm"] <= 1e-12 * info["r0_norm"]


def test_hex_sampled_parity_large(F, oracle):
    """48^3 jittered elasticity (110 k cells, 353 k DOF): full oracle apply, element-wise check."""
    coords, cells, bnd, lam, mu = make((48, 48, 48), 0.2, False, 13)
    x = np.random.default_rng(2).uniform(-1, 1, coords.shape[0] * 3)
    ref = oracle.apply_hex("elastic", coords, cells, x, bnd, lam, mu)
    op = F.Operator(F.HexMesh(dev(coords), dev(cells), dev(bnd)), "elastic", 1)
    op.set_material(dev(lam), dev(mu))
    assert relerr(op.apply(dev(x)).cpu().numpy(), ref) <= APPLY_TOL


def test_hex_errors(F):
    coords, cells, bnd, lam, mu = make((2, 2, 2), 0.0, False, 0)
    bad = cells.copy(); bad[0, 0] = coords.shape[0]
    with pytest.raises(F.FemError) as e:
        F.HexMesh(dev(coords), dev(bad))
    assert e.value.status == F.FEM_EINVAL
    inv = coords.copy(); inv[cells[0, 6]] = inv[cells[0, 0]] - 0.3
    with pytest.raises(F.FemError) as e:
        F.HexMesh(dev(inv), dev(cells))
    assert e.value.status == F.FEM_EINVAL
    mesh = F.HexMesh(dev(coords), dev(cells), dev(bnd))
    op = F.Operator(mesh, "elastic", 1)
    with pytest.raises(F.FemError) as e:
        op.apply(dev(np.zeros(coords.shape[0] * 3)))
    assert e.value.status == F.FEM_ESTATE
    with pytest.raises(F.FemError) as e:
        op.set_material(dev(lam), dev(mu), 0, 2)
    assert e.value.status == F.FEM_EINVAL
    op.set_material(dev(lam), dev(mu))
    with pytest.raises(F.FemError) as e:
        op.csr()
    assert e.value.status == F.FEM_EUNSUPPORTED
    x = dev(np.zeros(coords.shape[0] * 3))
    with pytest.raises(F.FemError) as e:
        op.apply_ghost(x, None, None)
    assert e.value.status == F.FEM_EUNSUPPORTED


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("bc", [0, 1])
def test_hex_partial_assembly_parity(F, oracle, kind, bc):
    """Partial assembly (stored Gauss-point geometry) is the same operator: oracle parity and
    agreement with the matrix-free kernel."""
    coords, cells, bnd, lam, mu = make((7, 6, 5), 0.22, True, 31)
    c = I.ncomp(kind)
    x = np.random.default_rng(4).uniform(-1, 1, coords.shape[0] * c)
    ref = oracle.apply_hex(kind, coords, cells, x, bnd if bc else None, lam, mu)
    op = F.Operator(F.HexMesh(dev(coords), dev(cells), dev(bnd)), kind, bc)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    y_mf = op.apply(dev(x)).cpu().numpy()
    op.set_option("partial_assembly", 1)
    assert op.get_option("partial_assembly") == 1
    y_pa = op.apply(dev(x)).cpu().numpy()
    assert relerr(y_pa, ref) <= APPLY_TOL
    assert relerr(y_pa, y_mf) <= APPLY_TOL


@pytest.mark.parametrize("kind", ["scalar", "elastic"])
def test_hex_partial_assembly_cg(F, oracle, kind):
    coords, cells, bnd, lam, mu = make((9, 8, 7), 0.2, True, 11)
    c = I.ncomp(kind)
    b = np.random.default_rng(21).uniform(-1, 1, coords.shape[0] * c)
    b[np.repeat(bnd == 1, c)] = 0.0
    ref = oracle.cg_hex(kind, coords, cells, b, bnd, tol=1e-14, maxit=3000, lam=lam, mu=mu)
    op = F.Operator(F.HexMesh(dev(coords), dev(cells), dev(bnd)), kind, 1)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    op.set_option("partial_assembly", 1)
    x = torch.zeros(b.size, dtype=torch.float64, device="cuda")
    info = op.cg_solve(dev(b), x, tol=1e-14, maxit=3000)
    assert info["converged"]
    assert np.abs(x.cpu().numpy() - ref.x).max() <= 1e-10 * max(1.0, np.abs(ref.x).max())


def test_partial_assembly_box_unsupported(F):
    """Box partial assembly is the 21-value elasticity operator (Table 3); Laplace kinds and
    multi-rank operators are not supported."""
    op = F.Operator(F.Mesh(4, 4, 4, 0.25), "scalar", 1)
    with pytest.raises(F.FemError) as e:
        op.set_option("partial_assembly", 1)
    assert e.value.status == F.FEM_EUNSUPPORTED


@pytest.mark.parametrize("bc", [0, 1])
@pytest.mark.parametrize("quad", [0, 1])
@pytest.mark.parametrize("dims", [(1, 1, 1), (5, 7, 9), (33, 17, 12), (40, 9, 13)])
def test_box_partial_assembly_21(F, oracle, bc, quad, dims):
    """Elasticity partial assembly on the box (Table 3: 21 values per Gauss point,
    D_q = w_q det J_q C_e): the oracle's operator (Gauss rule; the Lobatto rule against the
    oracle run with that rule) and the matrix-free kernel, within 1e-12."""
    nx, ny, nz = dims
    h = 1.0 / max(dims)
    g = I.rng(I.SEED_BASE + 700 + nx)
    x = I.uniform_vector(g, nx, ny, nz, 3)
    lam, mu = I.materials(g, nx, ny, nz)
    op = F.Operator(F.Mesh(nx, ny, nz, h), "elastic", bc)
    op.set_option("quadrature", quad)
    op.set_option("partial_assembly", 1)  # before the material: D is formed by fem_set_material
    op.set_material(dev(lam), dev(mu))
    assert op.get_option("partial_assembly") == 1 and op.get_option("fused_cg") == 0
    y_pa = op.apply(dev(x)).cpu().numpy()
    with oracle.quadrature("gll" if quad else "gauss"):
        ref = oracle.apply("elastic", bc, nx, ny, nz, h, x, lam=lam, mu=mu)
    assert relerr(y_pa, ref) <= APPLY_TOL
    y_pa_host = op.apply(x)  # host vectors: staged copies, same kernel
    assert np.array_equal(y_pa_host, y_pa)
    op.set_option("partial_assembly", 0)
    y_mf = op.apply(dev(x)).cpu().numpy()
    assert relerr(y_pa, y_mf) <= APPLY_TOL
    # material changed after enabling: D is recomputed
    op.set_option("partial_assembly", 1)
    op.set_material(dev(2.0 * lam), dev(mu))
    with oracle.quadrature("gll" if quad else "gauss"):
        ref2 = oracle.apply("elastic", bc, nx, ny, nz, h, x, lam=2.0 * lam, mu=mu)
    assert relerr(op.apply(dev(x)).cpu().numpy(), ref2) <= APPLY_TOL


def test_box_partial_assembly_cg(F, oracle):
    nx, ny, nz = 9, 8, 7
    h = 1.0 / 9
    g = I.rng(I.SEED_BASE + 710)
    lam, mu = I.materials(g, nx, ny, nz)
    b = I.interior_rhs(g, nx, ny, nz, 3)
    ref = oracle.cg("elastic", 1, nx, ny, nz, h, b, tol=1e-14, maxit=3000, lam=lam, mu=mu)
    op = F.Operator(F.Mesh(nx, ny, nz, h), "elastic", 1)
    op.set_material(dev(lam), dev(mu))
    op.set_option("partial_assembly", 1)
    x = torch.zeros(b.size, dtype=torch.float64, device="cuda")
    info = op.cg_solve(dev(b), x, tol=1e-14, maxit=3000)
    assert info["converged"] and abs(info["iterations"] - ref.iterations) <= 3
    assert np.abs(x.cpu().numpy() - ref.x).max() <= 1e-10 * max(1.0, np.abs(ref.x).max())


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("bc", [0, 1])
@pytest.mark.parametrize("pa", [0, 1])
def test_hex_deterministic_scatter(F, oracle, kind, bc, pa):
    """option "deterministic": element outputs + per-node gather in ascending (cell, corner) order
    instead of FP64 atomics -- oracle parity as before, and bitwise identical applies and CG
    iterates run after run (the atomic scatter's summation order varies)."""
    coords, cells, bnd, lam, mu = make((17, 9, 6), 0.2, True, 3)
    c = I.ncomp(kind)
    x = np.random.default_rng(31).uniform(-1, 1, coords.shape[0] * c)
    ref = oracle.apply_hex(kind, coords, cells, x, bnd if bc else None, lam, mu)
    op = F.Operator(F.HexMesh(dev(coords), dev(cells), dev(bnd)), kind, bc)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    if pa:
        op.set_option("partial_assembly", 1)
    assert op.get_option("deterministic") == 0
    y_atomic = op.apply(dev(x))
    op.set_option("deterministic", 1)
    assert op.get_option("deterministic") == 1
    ys = [op.apply(dev(x)) for _ in range(3)]
    for y in ys[1:]:
        assert torch.equal(y, ys[0])
    assert relerr(ys[0].cpu().numpy(), ref) <= APPLY_TOL
    assert float((ys[0] - y_atomic).abs().max() / y_atomic.abs().max()) <= 1e-14
    if bc:
        b = np.random.default_rng(32).uniform(-1, 1, coords.shape[0] * c)
        b[np.repeat(bnd == 1, c)] = 0.0
        xs = []
        for _ in range(2):
            xg = torch.zeros(b.size, dtype=torch.float64, device="cuda")
            op.cg_solve(dev(b), xg, tol=0.0, maxit=40)
            xs.append(xg)
        assert torch.equal(xs[0], xs[1])
    op.set_option("deterministic", 0)
    assert op.get_option("deterministic") == 0


def test_hex_deterministic_box_only_option(F):
    op = F.Operator(F.Mesh(4, 4, 4, 0.25), "scalar", 1)
    assert op.get_option("deterministic") == 1  # the box kernels are atomic-free
    with pytest.raises(F.FemError):
        op.set_option("deterministic", 1)
