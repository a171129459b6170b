"""Paired x update of the fused CG (option x_pairs): x is advanced every other
iteration as x = (x + alpha_{k-1} p_{k-1}) + alpha_k p_k from the two p ping-pong buffers, i.e.
the same two FMAs per entry in the same order as the per-iteration update.  So the iterates must
be BITWISE equal to x_pairs = 0 (which the oracle-parity tests cover) for every iteration count,
odd or even, for every way the iterations are issued (one graph, several graphs, eagerly), when
the solve stops early on the tolerance, and with each dot implementation that is deterministic."""
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
def test_x_pairs_bitwise(F, kind):
    op, b = make(F, kind, (40, 31, 20), 610)
    assert op.get_option("x_pairs") == 1  # the default on the fused path
    for use_graph in (1, 0):
        op.set_option("use_graph", use_graph)
        for chunks in ([1], [2], [7], [8], [3, 4], [1, 1, 1], [5, 6]):
            op.set_option("x_pairs", 0)
            x0, i0 = run(op, b, chunks)
            op.set_option("x_pairs", 1)
            x1, i1 = run(op, b, chunks)
            assert torch.equal(x0, x1), (use_graph, chunks, float((x0 - x1).abs().max()))
            assert i0["iterations"] == i1["iterations"] == sum(chunks)
            assert i0["true_r_norm"] == i1["true_r_norm"]


@pytest.mark.parametrize("kind", ["scalar", "elastic"])
def test_x_pairs_early_stop(F, kind):
    """tol > 0: the solve stops at whatever parity convergence happens (a pending first half is
    added by cg_end); extra requested iterations are no-ops on the device."""
    op, b = make(F, kind, (24, 20, 18), 611)
    for tol in (1e-3, 1e-6, 1e-9):
        op.set_option("x_pairs", 0)
        x0, i0 = run(op, b, [200], tol=tol)
        op.set_option("x_pairs", 1)
        x1, i1 = run(op, b, [200], tol=tol)
        assert i0["converged"] and i1["converged"]
        assert i0["iterations"] == i1["iterations"] < 200
        assert torch.equal(x0, x1)
    iters = {run(op, b, [200], tol=t)[1]["iterations"] % 2 for t in (1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 1e-7)}
    assert iters == {0, 1}  # both parities of the stopping iteration were exercised


@pytest.mark.parametrize("dot_mode", [0, 1])
def test_x_pairs_dot_modes(F, dot_mode):
    op, b = make(F, "vector", (33, 17, 12), 612)
    op.set_option("dot_mode", dot_mode)
    op.set_option("x_pairs", 0)
    x0, _ = run(op, b, [9])
    op.set_option("x_pairs", 1)
    x1, _ = run(op, b, [9])
    assert torch.equal(x0, x1)


def test_x_pairs_applicability(F):
    """x_pairs acts on the fused Hestenes-Stiefel iteration only: it reads back 0 under the
    single-reduction variant (whose update carries its own p / s recurrences) and can not change
    during a solve."""
    op, b = make(F, "elastic", (20, 20, 20), 613)
    op.set_option("cg_variant", 1)
    assert op.get_option("x_pairs") == 0
    op.set_option("cg_variant", 0)
    assert op.get_option("x_pairs") == 1
    x = torch.zeros_like(b)
    op.cg_begin(b, x, tol=0.0, maxit=4)
    with pytest.raises(F.FemError):
        op.set_option("x_pairs", 0)
    op.cg_iterate(4)
    op.cg_end()
