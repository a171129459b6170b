"""Deferred x update of the fused CG (option x_defer = m): x is advanced once per
group of m iterations, x = ((x + alpha_0 p_0) + ...) + alpha_{m-1} p_{m-1}, from the m p buffers
the fused apply writes in turn -- the same FMAs per entry in the same order as the per-iteration
update.  So the iterates must be BITWISE equal to x_defer = 1 (which the oracle-parity tests
cover) for every iteration count (every position inside a group), for every way the iterations
are issued (one graph, several graphs, eagerly), when the solve stops early on the tolerance,
and with each dot implementation that is deterministic."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2308_09839_b200 import inputs as I

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2308_09839_b200 import fem
    fem.load()
    return fem


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def make(F, kind, dims, seed):
    nx, ny, nz = dims
    g = I.rng(I.SEED_BASE + seed)
    c = I.ncomp(kind)
    op = F.Operator(F.Mesh(nx, ny, nz, 1.0 / nx), kind, 1)
    if kind == "elastic":
        lam, mu = I.materials(g, nx, ny, nz)
        op.set_material(dev(lam), dev(mu))
    b = dev(I.interior_rhs(g, nx, ny, nz, c))
    return op, b


def run(op, b, chunks, tol=0.0, maxit=None):
    x = torch.zeros_like(b)
    op.cg_begin(b, x, tol=tol, maxit=maxit if maxit is not None else sum(chunks))
    for k in chunks:
        op.cg_iterate(k)
    info = op.cg_end()
    return x, info


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
def test_x_defer_bitwise(F, kind):
    op, b = make(F, kind, (40, 31, 20), 610)
    assert op.get_option("x_defer") == 8  # the default on the fused path
    for use_graph in (1, 0):
        op.set_option("use_graph", use_graph)
        for chunks in ([1], [2], [3], [4], [5], [7], [8], [9], [15], [17], [3, 4], [1, 1, 1], [5, 6], [2, 3, 2], [7, 9, 3]):
            xs = []
            for m in (1, 2, 4, 8):
                op.set_option("x_defer", m)
                assert op.get_option("x_defer") == m
                x, info = run(op, b, chunks)
                assert info["iterations"] == sum(chunks)
                xs.append((x, info))
            for x, info in xs[1:]:
                assert torch.equal(xs[0][0], x), (use_graph, chunks, float((xs[0][0] - x).abs().max()))
                assert info["true_r_norm"] == xs[0][1]["true_r_norm"]


@pytest.mark.parametrize("kind", ["scalar", "elastic"])
def test_x_defer_early_stop(F, kind):
    """tol > 0: the solve stops wherever convergence happens inside a group (cg_end adds the
    pending updates); extra requested iterations are no-ops on the device."""
    op, b = make(F, kind, (24, 20, 18), 611)
    for tol in (1e-3, 1e-6, 1e-9):
        res = []
        for m in (1, 2, 4, 8):
            op.set_option("x_defer", m)
            res.append(run(op, b, [200], tol=tol))
        for x, info in res:
            assert info["converged"] and info["iterations"] == res[0][1]["iterations"] < 200
            assert torch.equal(x, res[0][0])
    op.set_option("x_defer", 8)
    iters = {run(op, b, [200], tol=t)[1]["iterations"] % 8 for t in (1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 1e-7, 1e-8, 1e-9, 1e-10)}
    assert len(iters) >= 3  # the solve ended at several positions inside a group


@pytest.mark.parametrize("dot_mode", [0, 1])
def test_x_defer_dot_modes(F, dot_mode):
    op, b = make(F, "vector", (33, 17, 12), 612)
    op.set_option("dot_mode", dot_mode)
    xs = []
    for m in (1, 2, 4, 8):
        op.set_option("x_defer", m)
        xs.append(run(op, b, [11])[0])
    for x in xs[1:]:
        assert torch.equal(xs[0], x)


def test_x_defer_applicability(F):
    """x_defer takes 1, 2, 4 or 8 only and can not change during a solve."""
    op, b = make(F, "elastic", (20, 20, 20), 613)
    assert op.get_option("x_defer") == 8
    for bad in (0, 3, 5, 16):
        with pytest.raises(F.FemError):
            op.set_option("x_defer", bad)
    x = torch.zeros_like(b)
    op.cg_begin(b, x, tol=0.0, maxit=4)
    with pytest.raises(F.FemError):
        op.set_option("x_defer", 2)
    op.cg_iterate(4)
    op.cg_end()


@pytest.mark.parametrize("kind", ["scalar", "elastic"])
def test_x_defer_single_reduction(F, kind):
    """Chronopoulos-Gear CG (cg_variant 1): its update writes p into the ring and
    defers x the same way -- bitwise equal to m = 1 (x += alpha p every iteration, p in place)."""
    op, b = make(F, kind, (33, 21, 17), 614)
    op.set_option("cg_variant", 1)
    for use_graph in (1, 0):
        op.set_option("use_graph", use_graph)
        for chunks in ([1], [7], [8], [9], [3, 6], [17]):
            xs = []
            for m in (1, 2, 4, 8):
                op.set_option("x_defer", m)
                assert op.get_option("x_defer") == m
                xs.append(run(op, b, chunks)[0])
            for x in xs[1:]:
                assert torch.equal(xs[0], x), (use_graph, chunks)
    for tol in (1e-4, 1e-9):
        res = []
        for m in (1, 8):
            op.set_option("x_defer", m)
            res.append(run(op, b, [300], tol=tol))
        assert res[0][1]["iterations"] == res[1][1]["iterations"] < 300
        assert torch.equal(res[0][0], res[1][0])


def _unfused_ops(F):
    """Operators on the unfused CG iteration (apply, update, p-update): general hexes (matrix-free
    and partial assembly, with the deterministic scatter -- the FP64-atomic one is not bitwise
    reproducible run to run), partial assembly on the box, and a degenerate box (one cell thick:
    no interior nodes in z, so no TMA path)."""
    g = I.rng(I.SEED_BASE + 616)
    out = []
    for kind in ("scalar", "elastic"):
        c = I.ncomp(kind)
        coords, cells, bnd = I.hex_box_mesh(9, 7, 6, h=1.0 / 9, g=g, jitter=0.15, permute=True)
        b = torch.zeros(coords.shape[0] * c, dtype=torch.float64, device="cuda").uniform_(-1, 1)
        hl, hm = I.materials(g, cells.shape[0], 1, 1)
        for pa in (0, 1):
            op = F.Operator(F.HexMesh(dev(coords), dev(cells), dev(bnd)), kind, 1)
            if kind == "elastic":
                op.set_material(dev(hl), dev(hm))
            op.set_option("deterministic", 1)
            op.set_option("partial_assembly", pa)
            out.append((f"hex-{kind}-pa{pa}", op, b))
    op, b = make(F, "elastic", (14, 11, 9), 617)
    op.set_option("partial_assembly", 1)
    out.append(("box-pa", op, b))
    op, b = make(F, "vector", (12, 10, 1), 618)
    out.append(("box-degenerate", op, b))
    return out


def test_x_defer_unfused_iteration(F):
    """The unfused iteration defers x the same way (p_{k+1} = r + beta p_k written into the next
    ring buffer by the p-update kernel): bitwise equal to m = 1 (p updated in place)."""
    for name, op, b in _unfused_ops(F):
        for chunks in ([1], [5], [8], [11], [4, 5]):
            xs = []
            for m in (1, 2, 4, 8):
                op.set_option("x_defer", m)
                assert op.get_option("x_defer") == m, name
                x, info = run(op, b, chunks)
                assert info["iterations"] == sum(chunks) or info["converged"], name
                xs.append(x)
            for x in xs[1:]:
                assert torch.equal(xs[0], x), (name, chunks, float((xs[0] - x).abs().max()))
