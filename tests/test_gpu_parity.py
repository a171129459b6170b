"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Tolerances:
  * apply: ||y - y_ref||_inf / ||y_ref||_inf <= 1e-12 (north_star "max relative error 1e-12");
  * CG: solutions compared once converged past 1e-13 relative residual, |x - x_ref|_inf <= 1e-10;
  * dot: relative 1e-14 (different summation order, both fp64).
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


# (64, 3, 5), (32, 32, 6): nx+1 (ny+1) = 1 mod the Laplace tile, so the last boundary column (row)
# is written by the previous tile's producer warp (kernels_laplace.cu `ext`)
MESHES = [(1, 1, 1), (2, 2, 2), (5, 7, 9), (33, 17, 12), (40, 31, 20), (64, 3, 5), (3, 70, 4), (32, 32, 6)]


# caller vectors with 16-B rows ((nx+1) c even): fem_apply stages them through a tensor map over
# the caller's memory ("direct_tma"); same operator as the bulk-row path, bit for bit
@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("dims", [(32, 17, 12), (64, 40, 21), (30, 45, 4)])
def test_apply_row_pairs_exact_allocation(F, oracle, kind, dims):
    """Odd rows in a buffer that ends exactly where the vector ends (cudaMalloc of the exact size,
    no slack for the row-pair view's last boxes): the view then covers planes 0 .. nz-1 and the
    last plane comes from a one-plane copy -- still the row-pair path, equal to the slack case."""
    import ctypes
    from cuda.bindings import runtime as rt
    nx, ny, nz = dims
    h = 1.0 / max(dims)
    g = I.rng(I.SEED_BASE + 410 + nx + 7 * ny + 31 * nz)
    c = I.ncomp(kind)
    x = I.uniform_vector(g, nx, ny, nz, c)
    lam, mu = I.materials(g, nx, ny, nz)
    op = F.Operator(F.Mesh(nx, ny, nz, h), kind, 1)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    roomy = torch.empty(x.size + 4096, dtype=torch.float64, device="cuda")[:x.size]
    roomy.copy_(torch.from_numpy(x))
    y_ref = op.apply(roomy)
    assert op.get_option("last_apply_path") == 2
    nbytes = x.size * 8
    err, xp = rt.cudaMalloc(nbytes)
    assert err == rt.cudaError_t.cudaSuccess
    err, yp = rt.cudaMalloc(nbytes)
    assert err == rt.cudaError_t.cudaSuccess
    try:
        (err,) = rt.cudaMemcpy(xp, roomy.data_ptr(), nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
        assert err == rt.cudaError_t.cudaSuccess
        torch.cuda.synchronize()
        lib = F.load()
        rc = lib.fem_apply(op.h, ctypes.c_void_p(int(xp)), ctypes.c_void_p(int(yp)), None)
        assert rc == 0, lib.fem_last_error()
        assert op.get_option("last_apply_path") == 2
        y = torch.empty_like(y_ref)
        (err,) = rt.cudaMemcpy(y.data_ptr(), yp, nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
        assert err == rt.cudaError_t.cudaSuccess
        torch.cuda.synchronize()
        assert torch.equal(y, y_ref)
    finally:
        rt.cudaFree(xp)
        rt.cudaFree(yp)
    ref = oracle.apply(kind, 1, nx, ny, nz, h, x, lam=lam, mu=mu)
    assert relerr(y.cpu().numpy(), ref) <= APPLY_TOL


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("bc", [0, 1])
@pytest.mark.parametrize("quad", [0, 1])
@pytest.mark.parametrize("dims", [(5, 7, 9), (33, 17, 12), (63, 40, 21), (1, 1, 1)])
def test_apply_direct_tma(F, oracle, kind, bc, quad, dims):
    nx, ny, nz = dims
    assert (nx + 1) % 2 == 0
    h = 1.0 / max(dims)
    g = I.rng(I.SEED_BASE + 300 + nx + 7 * ny + 31 * nz)
    c = I.ncomp(kind)
    x = I.uniform_vector(g, nx, ny, nz, c)
    lam, mu = I.materials(g, nx, ny, nz)
    op = F.Operator(F.Mesh(nx, ny, nz, h), kind, bc)
    op.set_option("quadrature", quad)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    assert op.get_option("direct_tma") == 1
    y1 = op.apply(dev(x)).cpu().numpy()
    op.set_option("direct_tma", 0)
    y0 = op.apply(dev(x)).cpu().numpy()
    assert np.array_equal(y1, y0)
    if quad == 0:
        ref = oracle.apply(kind, bc, nx, ny, nz, h, x, lam=lam, mu=mu)
        assert relerr(y1, ref) <= APPLY_TOL


# odd rows ((nx+1) c odd) with the Dirichlet box: the Laplace kinds stage caller vectors through
# the row-pair tensor view (two boxes per plane); equal to the bulk-row path (bitwise under Gauss)
@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("quad", [0, 1])
@pytest.mark.parametrize("dims", [(4, 7, 9), (32, 17, 12), (64, 40, 21), (2, 2, 2), (30, 45, 3)])
def test_apply_row_pairs(F, oracle, kind, quad, dims):
    nx, ny, nz = dims
    assert (nx + 1) % 2 == 1
    h = 1.0 / max(dims)
    g = I.rng(I.SEED_BASE + 400 + nx + 7 * ny + 31 * nz)
    c = I.ncomp(kind)
    x = I.uniform_vector(g, nx, ny, nz, c)
    lam, mu = I.materials(g, nx, ny, nz)
    op = F.Operator(F.Mesh(nx, ny, nz, h), kind, 1)
    op.set_option("quadrature", quad)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    xd = torch.empty(x.size + 4096, dtype=torch.float64, device="cuda")[:x.size]  # room past the end
    xd.copy_(torch.from_numpy(x))
    y1 = op.apply(xd).cpu().numpy()
    assert op.get_option("last_apply_path") == 2
    op.set_option("direct_tma", 0)
    y0 = op.apply(xd).cpu().numpy()
    assert op.get_option("last_apply_path") == 0
    if quad == 0:
        if kind != "elastic":  # (elasticity: the bulk path runs the one-row kernel)
            assert np.array_equal(y1, y0)
        else:
            assert relerr(y1, y0) <= 4e-16
        ref = oracle.apply(kind, 1, nx, ny, nz, h, x, lam=lam, mu=mu)
        assert relerr(y1, ref) <= APPLY_TOL
    else:  # the Gauss-Lobatto filters contract into FMAs differently per kernel instance: 1 ulp
        assert relerr(y1, y0) <= 4e-16
        with oracle.quadrature("gll"):
            ref = oracle.apply(kind, 1, nx, ny, nz, h, x, lam=lam, mu=mu)
        assert relerr(y1, ref) <= APPLY_TOL


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("bc", [0, 1])
@pytest.mark.parametrize("dims", MESHES)
def test_apply_parity(F, oracle, kind, bc, dims):
    nx, ny, nz = dims
    h = 1.0 / max(dims)
    g = I.rng(I.SEED_BASE + 100 + nx + 7 * ny + 31 * nz)
    c = I.ncomp(kind)
    x = I.uniform_vector(g, nx, ny, nz, c)
    lam, mu = I.materials(g, nx, ny, nz)
    ref = oracle.apply(kind, bc, nx, ny, nz, h, x, lam=lam, mu=mu)
    mesh = F.Mesh(nx, ny, nz, h)
    op = F.Operator(mesh, kind, bc)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    y = op.apply(dev(x)).cpu().numpy()
    assert relerr(y, ref) <= APPLY_TOL
    if bc:
        bm = np.repeat(I.boundary_mask(nx, ny, nz), c)
        assert np.array_equal(y[bm], x[bm])


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
def test_apply_host_pointers(F, oracle, kind):
    """Host buffers go through the library's staging (the e2e path) with identical results."""
    nx, ny, nz, h = 9, 8, 7, 0.1
    g = I.rng(I.SEED_BASE + 200)
    c = I.ncomp(kind)
    x = I.uniform_vector(g, nx, ny, nz, c)
    lam, mu = I.materials(g, nx, ny, nz)
    op = F.Operator(F.Mesh(nx, ny, nz, h), kind, 1)
    if kind == "elastic":
        op.set_material(lam, mu)  # host material
    yh = op.apply(x)  # numpy in, numpy out
    yd = op.apply(dev(x)).cpu().numpy()
    assert np.array_equal(yh, yd)
    assert relerr(yh, oracle.apply(kind, 1, nx, ny, nz, h, x, lam=lam, mu=mu)) <= APPLY_TOL


def test_apply_deterministic(F):
    nx, ny, nz = 40, 33, 50
    g = I.rng(I.SEED_BASE + 201)
    x = dev(I.uniform_vector(g, nx, ny, nz, 3))
    lam, mu = I.materials(g, nx, ny, nz)
    op = F.Operator(F.Mesh(nx, ny, nz, 0.02), "elastic", 1)
    op.set_material(dev(lam), dev(mu))
    y1 = op.apply(x)
    y2 = op.apply(x)
    assert torch.equal(y1, y2)


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
def test_fused_cg_deterministic(F, kind):
    """the producer-less TMA kernels (ring refilled by a consumer warp, mbarrier hand-offs) give
    bitwise identical CG iterates run after run -- the race check racecheck cannot do (DESIGN 8a)"""
    nx, ny, nz = 70, 45, 61
    g = I.rng(I.SEED_BASE + 203)
    c = I.ncomp(kind)
    lam, mu = I.materials(g, nx, ny, nz)
    b = dev(I.interior_rhs(g, nx, ny, nz, c))
    op = F.Operator(F.Mesh(nx, ny, nz, 1.0 / nx), kind, 1)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    xs = []
    for _ in range(3):
        x = torch.zeros_like(b)
        op.cg_begin(b, x, tol=0.0, maxit=25)
        op.cg_iterate(25)
        op.cg_end()
        xs.append(x)
    assert torch.equal(xs[0], xs[1]) and torch.equal(xs[0], xs[2])


@pytest.mark.parametrize("kind,n", [("scalar", 192), ("vector", 160), ("elastic", 128)])
def test_fused_cg_ring_refill_race(F, kind, n):
    """Regression: at sizes with thousands of CTAs the producer-warp vector kernel sporadically
    read part of a warp row from a ring slot the TMA refill had already overwritten (the refill
    lacked fence.proxy.async after observing the release; kernels_common.cuh PlaneRing::produce).
    One fused CG iteration (x = alpha r) against textbook CG around fem_apply, repeated on the
    captured graph and eagerly: every repeat bitwise identical and within 1e-13."""
    g = I.rng(I.SEED_BASE + 204)
    c = I.ncomp(kind)
    op = F.Operator(F.Mesh(n, n, n, 1.0 / n), kind, 1)
    if kind == "elastic":
        lam, mu = I.materials(g, n, n, n)
        op.set_material(dev(lam), dev(mu))
    b = dev(I.interior_rhs(g, n, n, n, c))
    q = op.apply(b)
    xr = (torch.dot(b, b) / torch.dot(b, q)) * b
    for use_graph in (1, 0):
        op.set_option("use_graph", use_graph)
        xs = []
        for _ in range(6):
            x = torch.zeros_like(b)
            op.cg_begin(b, x, tol=0.0, maxit=1)
            op.cg_iterate(1)
            op.cg_end()
            xs.append(x)
        for x in xs:
            assert torch.equal(x, xs[0])
        assert float((xs[0] - xr).abs().max() / xr.abs().max()) <= 1e-13


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
def test_null_space_and_symmetry_gpu(F, kind):
    """Properties that hold at any size, checked on the GPU alone (no oracle)."""
    nx, ny, nz, h = 37, 29, 23, 0.05
    g = I.rng(I.SEED_BASE + 202)
    c = I.ncomp(kind)
    lam, mu = I.materials(g, nx, ny, nz)
    op = F.Operator(F.Mesh(nx, ny, nz, h), kind, 0)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    n = I.n_nodes(nx, ny, nz)
    if kind == "elastic":
        k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
        X = np.stack([i.ravel() * h, j.ravel() * h, k.ravel() * h], 1)
        modes = [np.tile(np.eye(3)[d], n) for d in range(3)]
        for W in ([[0, -1, 0], [1, 0, 0], [0, 0, 0]], [[0, 0, -1], [0, 0, 0], [1, 0, 0]]):
            modes.append((X @ np.array(W, float).T).ravel())
        scale = (lam + 2 * mu).max() * h * 16
    else:
        modes = [np.ones(n * c)]
        scale = 16 * h
    for m in modes:
        y = op.apply(dev(m)).cpu().numpy()
        assert np.abs(y).max() < 1e-12 * scale
    a = dev(I.uniform_vector(g, nx, ny, nz, c)); b = dev(I.uniform_vector(g, nx, ny, nz, c))
    ab = op.dot(b, op.apply(a)); ba = op.dot(a, op.apply(b))
    assert abs(ab - ba) <= 1e-12 * abs(ab)


def test_dot_parity(F, oracle):
    for n_cells in [(1, 1, 1), (20, 20, 20), (63, 64, 65)]:
        g = I.rng(I.SEED_BASE + 300)
        a = I.uniform_vector(g, *n_cells, 1); b = I.uniform_vector(g, *n_cells, 1)
        op = F.Operator(F.Mesh(*n_cells, 0.1), "scalar", 1)
        d = op.dot(dev(a), dev(b))
        ref = oracle.dot(a, b)
        assert abs(d - ref) <= 1e-14 * np.abs(a * b).sum()
        assert op.dot(a, b) == d  # host pointers, same kernel


@pytest.mark.parametrize("kind", ["scalar", "vector"])
def test_cg_laplace_edge_tiles(F, oracle, kind):
    """Fused (TMA) CG on a mesh whose last boundary column and row are beyond the last tile, with
    a right-hand side that is nonzero on the Dirichlet rows too (identity rows carry p, q, p.q)."""
    nx, ny, nz = 32, 32, 6
    h = 1.0 / 32
    g = I.rng(I.SEED_BASE + 400)
    c = I.ncomp(kind)
    b = I.uniform_vector(g, nx, ny, nz, c)
    ref = oracle.cg(kind, 1, nx, ny, nz, h, b, tol=1e-13, maxit=400)
    assert ref.converged
    op = F.Operator(F.Mesh(nx, ny, nz, h), kind, 1)
    assert op.get_option("fused_cg") == 1
    x = torch.zeros(b.size, dtype=torch.float64, device="cuda")
    info = op.cg_solve(dev(b), x, tol=1e-13, maxit=400)
    assert info["converged"] and abs(info["iterations"] - ref.iterations) <= 2
    assert np.abs(x.cpu().numpy() - ref.x).max() <= 1e-10 * max(1.0, np.abs(ref.x).max())


def test_cg_c1_parity(F, oracle):
    """BASELINE configs[0]: scalar 8^3, Dirichlet, 50 CG iterations, FP64."""
    nx = ny = nz = 8; h = 1 / 8
    g = I.rng(I.SEED_BASE + 0)
    b = I.interior_rhs(g, nx, ny, nz, 1)
    ref = oracle.cg("scalar", 1, nx, ny, nz, h, b, tol=0.0, maxit=50)
    op = F.Operator(F.Mesh(nx, ny, nz, h), "scalar", 1)
    x = torch.zeros(b.size, dtype=torch.float64, device="cuda")
    info = op.cg_solve(dev(b), x, tol=0.0, maxit=50)
    assert info["iterations"] == ref.iterations
    assert np.abs(x.cpu().numpy() - ref.x).max() <= 1e-10
    assert abs(info["r0_norm"] - ref.r0_norm) <= 1e-13 * ref.r0_norm
    assert info["true_r_norm"] <= 1e-12 * ref.r0_norm


@pytest.mark.parametrize("dims,iters", [((8, 8, 8), 150), ((12, 10, 9), 250)])
def test_cg_elastic_parity(F, oracle, dims, iters):
    nx, ny, nz = dims
    h = 1.0 / nx
    g = I.rng(I.SEED_BASE + 3)
    lam, mu = I.materials(g, nx, ny, nz)
    b = I.interior_rhs(g, nx, ny, nz, 3)
    ref = oracle.cg("elastic", 1, nx, ny, nz, h, b, tol=1e-14, maxit=iters, lam=lam, mu=mu)
    assert ref.converged
    op = F.Operator(F.Mesh(nx, ny, nz, h), "elastic", 1)
    op.set_material(dev(lam), dev(mu))
    x = torch.zeros(b.size, dtype=torch.float64, device="cuda")
    info = op.cg_solve(dev(b), x, tol=1e-14, maxit=iters)
    assert info["converged"]
    assert abs(info["iterations"] - ref.iterations) <= 3
    assert np.abs(x.cpu().numpy() - ref.x).max() <= 1e-10 * max(1.0, np.abs(ref.x).max())


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("variant", [0, 1])
def test_cg_r_norm_is_exit_residual(F, kind, variant):
    """fem_cg_info.r_norm is the recurrence residual of the exit iterate: after a
    fixed number of unconverged iterations it equals ||b - A x|| up to rounding (the recurrence
    and the true residual agree long before convergence).  Single-reduction CG reports the
    residual of the iterate its last update started from (include/fem.h), so one iteration more
    gives the comparison point there."""
    nx, ny, nz, h = 11, 10, 9, 0.1
    g = I.rng(I.SEED_BASE + 31)
    lam, mu = I.materials(g, nx, ny, nz)
    b = I.interior_rhs(g, nx, ny, nz, I.ncomp(kind))
    op = F.Operator(F.Mesh(nx, ny, nz, h), kind, 1)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    op.set_option("cg_variant", variant)
    x = torch.zeros(b.size, dtype=torch.float64, device="cuda")
    info = op.cg_solve(dev(b), x, tol=0.0, maxit=6)
    if variant == 0:
        assert abs(info["r_norm"] - info["true_r_norm"]) <= 1e-9 * info["true_r_norm"]
    else:  # r_norm belongs to iterate 5: run 5 iterations and compare its true residual
        x5 = torch.zeros_like(x)
        i5 = op.cg_solve(dev(b), x5, tol=0.0, maxit=5)
        assert abs(info["r_norm"] - i5["true_r_norm"]) <= 1e-9 * i5["true_r_norm"]
    assert info["r_norm"] < info["r0_norm"]


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("dot_mode", [1, 2])
def test_cg_dot_modes(F, oracle, kind, dot_mode):
    """The dot ablation (option dot_mode): separate dot kernels (1) and atomic CTA
    partials (2) give the fused CG of dot_mode 0 up to summation order: 3 iterations within
    1e-12, the converged solution within 1e-10 of the oracle's CG."""
    nx, ny, nz, h = 13, 11, 10, 1.0 / 13
    g = I.rng(I.SEED_BASE + 41)
    lam, mu = I.materials(g, nx, ny, nz)
    b = I.interior_rhs(g, nx, ny, nz, I.ncomp(kind))
    xs = {}
    for dm in (0, dot_mode):
        op = F.Operator(F.Mesh(nx, ny, nz, h), kind, 1)
        if kind == "elastic":
            op.set_material(dev(lam), dev(mu))
        op.set_option("dot_mode", dm)
        assert op.get_option("dot_mode") == dm
        x = torch.zeros(b.size, dtype=torch.float64, device="cuda")
        info = op.cg_solve(dev(b), x, tol=0.0, maxit=3)
        assert info["iterations"] == 3
        xs[dm] = x.cpu().numpy()
        xc = torch.zeros_like(x)
        info = op.cg_solve(dev(b), xc, tol=1e-13, maxit=2000)
        assert info["converged"]
        ref = oracle.cg(kind, 1, nx, ny, nz, h, b, tol=1e-13, maxit=2000, lam=lam, mu=mu)
        assert abs(info["iterations"] - ref.iterations) <= 3
        assert np.abs(xc.cpu().numpy() - ref.x).max() <= 1e-10 * max(1.0, np.abs(ref.x).max())
    assert np.abs(xs[dot_mode] - xs[0]).max() <= 1e-12 * np.abs(xs[0]).max()


def test_cg_vector_host_pointers(F, oracle):
    nx, ny, nz, h = 10, 9, 8, 0.1
    g = I.rng(I.SEED_BASE + 2)
    b = I.interior_rhs(g, nx, ny, nz, 3)
    ref = oracle.cg("vector", 1, nx, ny, nz, h, b, tol=1e-13, maxit=300)
    op = F.Operator(F.Mesh(nx, ny, nz, h), "vector", 1)
    x = np.zeros_like(b)
    info = op.cg_solve(b, x, tol=1e-13, maxit=300)
    assert info["converged"] and abs(info["iterations"] - ref.iterations) <= 2
    assert np.abs(x - ref.x).max() <= 1e-10


def test_cg_breakdown_and_edge_cases(F):
    # b = 0 -> rr = 0: converged at iteration 0, x stays 0
    op = F.Operator(F.Mesh(4, 4, 4, 0.25), "scalar", 1)
    b = torch.zeros(125, dtype=torch.float64, device="cuda")
    x = torch.zeros_like(b)
    info = op.cg_solve(b, x, tol=0.0, maxit=10)
    assert info["iterations"] == 0 and info["converged"] and torch.count_nonzero(x) == 0
    # single interior dof: exactly one iteration
    op2 = F.Operator(F.Mesh(2, 2, 2, 0.5), "scalar", 1)
    b2 = torch.zeros(27, dtype=torch.float64, device="cuda"); b2[13] = 0.7
    x2 = torch.zeros_like(b2)
    info = op2.cg_solve(b2, x2, tol=1e-14, maxit=10)
    assert info["iterations"] == 1 and abs(x2[13].item() - 0.7 * 0.75) < 1e-15
    # bc = none on a Laplace operator is singular: b = constant is in the null space's range
    # complement -> p.Ap = 0 after r = 0? use b with a constant component to force breakdown
    op3 = F.Operator(F.Mesh(3, 3, 3, 1 / 3), "scalar", 0)
    b3 = torch.ones(64, dtype=torch.float64, device="cuda")
    x3 = torch.zeros_like(b3)
    info = op3.cg_solve(b3, x3, tol=0.0, maxit=5)
    assert info["status"] == F.FEM_EBREAKDOWN and info["breakdown_iter"] == 0


def test_material_validation(F):
    op = F.Operator(F.Mesh(3, 3, 3, 0.1), "elastic", 1)
    lam = np.ones(27); mu = np.ones(27); mu[5] = 0.0
    with pytest.raises(F.FemError) as e:
        op.set_material(lam, mu)
    assert e.value.status == F.FEM_EMATERIAL
    mu[5] = 1.0; lam[3] = -1.0  # lambda + 2mu/3 < 0
    with pytest.raises(F.FemError):
        op.set_material(lam, mu)
    x = torch.zeros(64 * 3, dtype=torch.float64, device="cuda")
    with pytest.raises(F.FemError) as e:
        op.apply(x)
    assert e.value.status == F.FEM_ESTATE
    with pytest.raises(F.FemError):
        F.Operator(F.Mesh(3, 3, 3, 0.1), "scalar", 1).set_material(lam, mu)


def test_aliasing_and_alignment(F):
    op = F.Operator(F.Mesh(3, 3, 3, 0.1), "scalar", 1)
    x = torch.zeros(65, dtype=torch.float64, device="cuda")
    with pytest.raises(F.FemError):
        op.apply(x[:64], x[:64])


@pytest.mark.parametrize("kind,dims", [("scalar", (40, 30, 20)), ("vector", (21, 22, 23)),
                                       ("elastic", (20, 21, 22))])
@pytest.mark.parametrize("bc", [0, 1])
def test_csr_parity(F, oracle, kind, dims, bc):
    nx, ny, nz = dims
    h = 0.07
    g = I.rng(I.SEED_BASE + 400)
    c = I.ncomp(kind)
    x = I.uniform_vector(g, nx, ny, nz, c)
    lam, mu = I.materials(g, nx, ny, nz)
    op = F.Operator(F.Mesh(nx, ny, nz, h), kind, bc)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    A = op.csr()
    y = A.apply(dev(x)).cpu().numpy()
    ref = oracle.apply(kind, bc, nx, ny, nz, h, x, lam=lam, mu=mu)
    assert relerr(y, ref) <= APPLY_TOL
    # interior rows carry 27 (scalar) / 81 (vector, elasticity) entries (Table 1)
    n_int = (nx - 1) * (ny - 1) * (nz - 1) if bc else None
    if bc:
        # interior nodes whose neighbours are all interior: (nx-3)(ny-3)(nz-3) rows of full stencil
        full = (nx - 3) * (ny - 3) * (nz - 3)
        assert A.nnz >= full * 27 * c * c
        assert A.nnz <= n_int * 27 * c * c + (I.n_nodes(nx, ny, nz) - n_int) * c


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
def test_cg_chronopoulos_gear_parity(F, oracle, kind):
    """Single-reduction CG (option cg_variant = 1): same Krylov iterates in exact arithmetic, so
    the converged solution matches the oracle's Hestenes-Stiefel CG."""
    nx, ny, nz = 12, 10, 9
    h = 1.0 / 12
    g = I.rng(I.SEED_BASE + 1400)
    lam, mu = I.materials(g, nx, ny, nz)
    b = I.interior_rhs(g, nx, ny, nz, I.ncomp(kind))
    ref = oracle.cg(kind, 1, nx, ny, nz, h, b, tol=1e-14, maxit=500, lam=lam, mu=mu)
    assert ref.converged
    op = F.Operator(F.Mesh(nx, ny, nz, h), kind, 1)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    op.set_option("cg_variant", 1)
    assert op.get_option("cg_variant") == 1
    x = torch.zeros(b.size, dtype=torch.float64, device="cuda")
    info = op.cg_solve(dev(b), x, tol=1e-14, maxit=500)
    assert info["converged"]
    assert abs(info["iterations"] - ref.iterations) <= 3
    assert np.abs(x.cpu().numpy() - ref.x).max() <= 1e-10 * max(1.0, np.abs(ref.x).max())
    assert info["true_r_norm"] <= 1e-12 * info["r0_norm"]


def test_cg_chronopoulos_gear_fixed_iterations(F, oracle):
    """tol = 0: exactly maxit updates, iterate close to the Hestenes-Stiefel one (C1)."""
    nx = ny = nz = 8
    g = I.rng(I.SEED_BASE + 0)
    b = I.interior_rhs(g, nx, ny, nz, 1)
    ref = oracle.cg("scalar", 1, nx, ny, nz, 1 / 8, b, tol=0.0, maxit=50)
    op = F.Operator(F.Mesh(nx, ny, nz, 1 / 8), "scalar", 1)
    op.set_option("cg_variant", 1)
    x = torch.zeros(b.size, dtype=torch.float64, device="cuda")
    info = op.cg_solve(dev(b), x, tol=0.0, maxit=50)
    assert info["iterations"] == ref.iterations
    assert np.abs(x.cpu().numpy() - ref.x).max() <= 1e-10


# Tile-seam sweep: node counts around the tile widths of every kernel (Laplace 32/29 columns x
# 24/21 (scalar) or 7 (vector) rows; elasticity 31/30 x 15 (CG kernel) or 14 (caller-vector
# kernel)), odd and even rows (caller vectors with 16-B rows take the tensor-map path), both the
# apply (against the oracle) and the fused CG kernels (against textbook CG around fem_apply).
SEAM_MESHES = [(29, 14, 3), (30, 15, 4), (31, 16, 3), (32, 13, 2), (33, 23, 3), (61, 29, 2), (62, 30, 3)]


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("dims", SEAM_MESHES)
def test_tile_seams(F, oracle, kind, dims):
    nx, ny, nz = dims
    h = 1.0 / nx
    g = I.rng(I.SEED_BASE + 700 + nx + 7 * ny + 31 * nz)
    c = I.ncomp(kind)
    x = I.uniform_vector(g, nx, ny, nz, c)
    lam, mu = I.materials(g, nx, ny, nz)
    op = F.Operator(F.Mesh(nx, ny, nz, h), kind, 1)
    if kind == "elastic":
        op.set_material(dev(lam), dev(mu))
    ref = oracle.apply(kind, 1, nx, ny, nz, h, x, lam=lam, mu=mu)
    y = op.apply(dev(x)).cpu().numpy()
    assert relerr(y, ref) <= APPLY_TOL
    b = dev(I.interior_rhs(g, nx, ny, nz, c))
    iters = 4
    xg = torch.zeros_like(b)
    op.cg_begin(b, xg, tol=0.0, maxit=iters)
    op.cg_iterate(iters)
    assert op.cg_end()["iterations"] == iters
    xr = torch.zeros_like(b); r = b.clone(); p = r.clone(); rr = torch.dot(r, r)
    for _ in range(iters):
        q = op.apply(p)
        alpha = rr / torch.dot(p, q)
        xr += alpha * p
        r -= alpha * q
        rr_new = torch.dot(r, r)
        p = r + (rr_new / rr) * p
        rr = rr_new
    assert float((xg - xr).abs().max() / xr.abs().max()) <= 1e-11
