"""GPU parity of the Gauss-Lobatto (GLL, BP5/BP6) variant of every operator path against the
oracle run with the same rule (oracle.quadrature("gll"); pinned in test_oracle_gll_pins.py)."""
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


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("bc", [0, 1])
@pytest.mark.parametrize("dims", [(2, 2, 2), (33, 17, 12), (64, 3, 5)])
def test_gll_box_apply(F, oracle, kind, bc, dims):
    nx, ny, nz = dims
    h = 1.0 / max(dims)
    g = I.rng(I.SEED_BASE + 1300 + nx)
    c = I.ncomp(kind)
    x = I.uniform_vector(g, nx, ny, nz, c)
    lam, mu = I.materials(g, nx, ny, nz)
    with oracle.quadrature("gll"):
        ref = oracle.apply(kind, bc, nx, ny, nz, h, x, lam=lam, mu=mu)
    op = F.Operator(F.Mesh(nx, ny, nz, h), kind, bc)
    op.set_option("quadrature", 1)
    assert op.get_option("quadrature") == 1
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    assert relerr(op.apply(dev(x)).cpu().numpy(), ref) <= APPLY_TOL


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
def test_gll_box_cg(F, oracle, kind):
    """Fused (TMA) CG with the GLL kernels against the oracle's GLL CG."""
    nx, ny, nz = 12, 10, 9
    h = 1.0 / 12
    g = I.rng(I.SEED_BASE + 1310)
    lam, mu = I.materials(g, nx, ny, nz)
    b = I.interior_rhs(g, nx, ny, nz, I.ncomp(kind))
    with oracle.quadrature("gll"):
        ref = oracle.cg(kind, 1, nx, ny, nz, h, b, tol=1e-14, maxit=400, lam=lam, mu=mu)
    assert ref.converged
    op = F.Operator(F.Mesh(nx, ny, nz, h), kind, 1)
    op.set_option("quadrature", 1)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    x = torch.zeros(b.size, dtype=torch.float64, device="cuda")
    info = op.cg_solve(dev(b), x, tol=1e-14, maxit=400)
    assert info["converged"] and abs(info["iterations"] - ref.iterations) <= 3
    assert np.abs(x.cpu().numpy() - ref.x).max() <= 1e-10 * max(1.0, np.abs(ref.x).max())


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("pa", [0, 1])
def test_gll_hex_apply(F, oracle, kind, pa):
    g = I.rng(I.SEED_BASE + 1320)
    coords, cells, bnd = I.hex_box_mesh(6, 5, 4, g=g, jitter=0.2, permute=True)
    lam, mu = I.materials(g, cells.shape[0], 1, 1)
    c = I.ncomp(kind)
    x = np.random.default_rng(8).uniform(-1, 1, coords.shape[0] * c)
    with oracle.quadrature("gll"):
        ref = oracle.apply_hex(kind, coords, cells, x, bnd, lam, mu)
    op = F.Operator(F.HexMesh(dev(coords), dev(cells), dev(bnd)), kind, 1)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    op.set_option("partial_assembly", pa)
    op.set_option("quadrature", 1)
    assert relerr(op.apply(dev(x)).cpu().numpy(), ref) <= APPLY_TOL
    op.set_option("quadrature", 0)  # back to Gauss (PA geometry recomputed)
    assert relerr(op.apply(dev(x)).cpu().numpy(),
                  oracle.apply_hex(kind, coords, cells, x, bnd, lam, mu)) <= APPLY_TOL


@pytest.mark.parametrize("kind", ["scalar", "elastic"])
def test_gll_csr(F, kind):
    nx, ny, nz = 9, 8, 7
    h = 1.0 / 9
    g = I.rng(I.SEED_BASE + 1330)
    lam, mu = I.materials(g, nx, ny, nz)
    op = F.Operator(F.Mesh(nx, ny, nz, h), kind, 1)
    op.set_option("quadrature", 1)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    A = op.csr()
    x = dev(I.uniform_vector(g, nx, ny, nz, I.ncomp(kind)))
    assert relerr(A.apply(x).cpu().numpy(), op.apply(x).cpu().numpy()) <= APPLY_TOL
    A.close()
