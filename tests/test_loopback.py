"""Multi-rank slab decomposition run end to end on one GPU.

fem_comm_create_loopback gives P in-process ranks on one device.  Each rank is driven by its own
host thread and stream and calls the ordinary ABI (fem_apply, fem_dot, fem_cg_solve, option
"peer_halo"); the library's collective call sites (node-plane halo, CG-scalar allreduce, peer
handle exchange) take their loopback branch -- device copies and a rank-ordered sum kernel,
ordered across streams by events.  So the multi-rank CG drivers (fused Hestenes-Stiefel,
Chronopoulos-Gear, NCCL-style halo or peer halo) run exactly as at P > 1 on several GPUs, minus
the NCCL transport, and are checked here against the single-rank CUDA path (itself checked
against the oracle in test_gpu_parity.py) and against the oracle directly:

  * apply: bitwise equal to P = 1 (per-node summation order is slab independent);
  * dots (fem_dot, ||r0||, true residual): equal to P = 1 within 1e-14 relative;
  * CG: 3 iterations elementwise within 1e-12 (no time for dot-order drift); after convergence
    (relative residual 1e-13) within 1e-12 of P = 1 and of the oracle's CG (reading R14).
"""
from __future__ import annotations

import threading

import numpy as np
import pytest
import torch

from paper_2308_09839_b200 import inputs as I

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2308_09839_b200 import fem
    fem.load(build_if_missing=False)
    return fem


def _run_ranks(P, fn):
    """fn(rank, stream) in P threads (one stream each); returns the per-rank results."""
    out, err = [None] * P, [None] * P

    def body(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                out[r] = fn(r, st)
            st.synchronize()
        except BaseException as ex:  # reported below
            err[r] = ex

    ts = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    for e in err:
        if e is not None:
            raise e
    return out


def _slab_op(F, comm, kind, nx, ny, nz, h, lam, mu):
    mesh = F.Mesh(nx, ny, nz, h, comm)
    op = F.Operator(mesh, kind, 1)
    if kind == "elastic":
        k0, k1 = mesh.plane_begin, mesh.plane_end
        lb, le = max(k0 - 1, 0), min(k1, nz)
        op.set_material(np.ascontiguousarray(lam[lb * nx * ny:le * nx * ny]),
                        np.ascontiguousarray(mu[lb * nx * ny:le * nx * ny]), lb, le - lb)
    return mesh, op


def _ref_op(F, kind, nx, ny, nz, h, lam, mu):
    op = F.Operator(F.Mesh(nx, ny, nz, h), kind, 1)
    if kind == "elastic":
        op.set_material(lam, mu)
    return op


MESH = (13, 11, 14)  # ragged against every tile width; 15 node planes: 2-3 per rank at P = 5


@pytest.mark.parametrize("mesh", [MESH, (12, 11, 14), (40, 30, 24)])
@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("P", [2, 3, 5])
def test_loopback_apply_and_dot(F, kind, P, mesh):
    """fem_apply on caller vectors at P > 1 goes through the TMA views of the owned planes (even
    rows: direct tensor map; odd rows: row-pair view) with the ghost planes substituted from the
    halo buffers -- bitwise equal to P = 1 either way."""
    nx, ny, nz = mesh
    h = 1.0 / nx
    c = I.ncomp(kind)
    g = I.rng(I.SEED_BASE + 600)
    x = I.uniform_vector(g, nx, ny, nz, c)
    z = I.uniform_vector(g, nx, ny, nz, c)
    lam, mu = I.materials(g, nx, ny, nz)
    ref = _ref_op(F, kind, nx, ny, nz, h, lam, mu)
    y_ref = ref.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    d_ref = ref.dot(torch.from_numpy(x).cuda(), torch.from_numpy(z).cuda())
    comms = F.Comm.loopback(P)
    plane = (nx + 1) * (ny + 1) * c

    def rank(r, st):
        mesh, op = _slab_op(F, comms[r], kind, nx, ny, nz, h, lam, mu)
        k0, k1 = mesh.plane_begin, mesh.plane_end
        xl = torch.from_numpy(x[k0 * plane:k1 * plane].copy()).cuda()
        zl = torch.from_numpy(z[k0 * plane:k1 * plane].copy()).cuda()
        y = op.apply(xl, stream=st)  # caller vectors: halo through the loopback, TMA views
        path = op.get_option("last_apply_path")
        d = op.dot(xl, zl, stream=st)
        yh = op.apply(x[k0 * plane:k1 * plane].copy())  # host vectors (staged)
        st.synchronize()
        res = (y.cpu().numpy(), d, yh, path)
        op.close(); mesh.close()
        return res

    res = _run_ranks(P, rank)
    for cm in comms:
        cm.close()
    for r in res:  # 1: direct tensor map (even rows); 2: row-pair view (odd rows, when the
        # allocation has the slack the view reads), else 0: bulk rows
        assert r[3] == 1 if ((nx + 1) * c) % 2 == 0 else r[3] in (0, 2)
    y = np.concatenate([r[0] for r in res])
    assert np.array_equal(y, y_ref)
    assert np.array_equal(np.concatenate([r[2] for r in res]), y_ref)
    for r in res:
        assert r[1] == res[0][1]  # every rank holds the same global value
        assert abs(r[1] - d_ref) <= 1e-14 * abs(d_ref) + 1e-300


def _cg_case(F, kind, P, variant, peer, iters, tol, overlap=1):
    nx, ny, nz = MESH
    h = 1.0 / nx
    c = I.ncomp(kind)
    g = I.rng(I.SEED_BASE + 610)
    lam, mu = I.materials(g, nx, ny, nz)
    b = I.interior_rhs(g, nx, ny, nz, c)
    ref = _ref_op(F, kind, nx, ny, nz, h, lam, mu)
    if variant:
        ref.set_option("cg_variant", 1)
    xr = torch.zeros(b.size, dtype=torch.float64, device="cuda")
    info_ref = ref.cg_solve(torch.from_numpy(b).cuda(), xr, tol=tol, maxit=iters)
    comms = F.Comm.loopback(P)
    plane = (nx + 1) * (ny + 1) * c

    def rank(r, st):
        mesh, op = _slab_op(F, comms[r], kind, nx, ny, nz, h, lam, mu)
        if variant:
            op.set_option("cg_variant", 1)
        op.set_option("halo_overlap", overlap)
        if peer:
            op.set_option("peer_halo", 1)
            assert op.get_option("peer_halo") == 1
        k0, k1 = mesh.plane_begin, mesh.plane_end
        bl = torch.from_numpy(b[k0 * plane:k1 * plane].copy()).cuda()
        xl = torch.zeros_like(bl)
        info = op.cg_solve(bl, xl, tol=tol, maxit=iters, stream=st)
        st.synchronize()
        out = (xl.cpu().numpy(), info)
        op.close(); mesh.close()
        return out

    res = _run_ranks(P, rank)
    for cm in comms:
        cm.close()
    x = np.concatenate([r[0] for r in res])
    return x, xr.cpu().numpy(), [r[1] for r in res], info_ref, b, lam, mu


@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("P", [2, 3, 5])
@pytest.mark.parametrize("variant,peer,overlap", [(0, False, 1), (1, False, 1), (0, True, 1), (1, True, 1),
                                                  (0, False, 0), (1, False, 0)])
def test_loopback_cg_three_iterations(F, kind, P, variant, peer, overlap):
    """overlap = 1: the halo runs on the comm stream beside the interior planes (apply_split)."""
    x, xr, infos, ir, *_ = _cg_case(F, kind, P, variant, peer, 3, 0.0, overlap)
    assert np.abs(x - xr).max() <= 1e-12 * np.abs(xr).max()
    for info in infos:
        assert info["iterations"] == 3 and info["rc"] == 0
        assert info["r0_norm"] == infos[0]["r0_norm"] and info["true_r_norm"] == infos[0]["true_r_norm"]
    assert abs(infos[0]["r0_norm"] - ir["r0_norm"]) <= 1e-14 * ir["r0_norm"]
    assert abs(infos[0]["r_norm"] - ir["r_norm"]) <= 1e-12 * ir["r_norm"]
    assert abs(infos[0]["true_r_norm"] - ir["true_r_norm"]) <= 1e-11 * ir["true_r_norm"]


@pytest.mark.parametrize("kind", ["scalar", "elastic"])
@pytest.mark.parametrize("P", [2, 5])
@pytest.mark.parametrize("variant,peer", [(0, False), (0, True), (1, False)])
def test_loopback_cg_converged_vs_oracle(F, oracle, kind, P, variant, peer):
    nx, ny, nz = MESH
    x, xr, infos, ir, b, lam, mu = _cg_case(F, kind, P, variant, peer, 2000, 1e-13)
    assert all(i["converged"] for i in infos) and ir["converged"]
    scale = np.abs(xr).max()
    assert np.abs(x - xr).max() <= 1e-12 * scale
    o = oracle.cg(kind, 1, nx, ny, nz, 1.0 / nx, b, tol=1e-13, maxit=2000, lam=lam, mu=mu)
    assert np.abs(x - o.x).max() <= 1e-12 * scale
    for info in infos:
        assert info["true_r_norm"] <= 1e-12 * info["r0_norm"]


def test_loopback_missing_rank_fails(F):
    """A rank that never enters the collective: the other gets FEM_ESTATE (no hang)."""
    import os
    if os.environ.get("FEM_SLOW_TESTS") != "1":
        pytest.skip("takes the 120 s rendezvous timeout; FEM_SLOW_TESTS=1 to run")
    comms = F.Comm.loopback(2)
    mesh = F.Mesh(6, 6, 6, 1 / 6, comms[0])
    op = F.Operator(mesh, "scalar", 1)
    x = torch.zeros(op.n_local, dtype=torch.float64, device="cuda")
    with pytest.raises(F.FemError) as e:
        op.apply(x)
    assert e.value.status == F.FEM_ESTATE


@pytest.mark.parametrize("overlap", [1, 0])
def test_loopback_trace_timeline(F, overlap):
    """option "trace": device timeline of an exchange apply -- halo on the comm stream, interior
    planes on the caller's stream, then the boundary planes (SURVEY §5 tracing)."""
    nx, ny, nz = 40, 36, 30
    kind = "vector"
    c = I.ncomp(kind)
    g = I.rng(I.SEED_BASE + 620)
    x = I.uniform_vector(g, nx, ny, nz, c)
    comms = F.Comm.loopback(2)
    plane = (nx + 1) * (ny + 1) * c

    def rank(r, st):
        mesh, op = _slab_op(F, comms[r], kind, nx, ny, nz, 1.0 / nx, None, None)
        op.set_option("halo_overlap", overlap)
        with pytest.raises(F.FemError):
            op.get_option("trace_total_ns")  # nothing traced yet
        op.set_option("trace", 1)
        k0, k1 = mesh.plane_begin, mesh.plane_end
        xl = torch.from_numpy(x[k0 * plane:k1 * plane].copy()).cuda()
        op.apply(xl, stream=st)
        t = {k: op.get_option("trace_%s_ns" % k) for k in ("halo", "interior", "boundary", "total")}
        op.close(); mesh.close()
        return t

    res = _run_ranks(2, rank)
    for cm in comms:
        cm.close()
    for t in res:
        assert all(v >= 0 for v in t.values())
        assert t["total"] > 0
        assert t["interior"] <= t["total"] and t["halo"] <= t["total"]
        assert t["boundary"] <= t["total"]


@pytest.mark.parametrize("kind", ["scalar", "elastic"])
@pytest.mark.parametrize("variant,peer", [(0, False), (0, True), (1, False), (1, True)])
def test_loopback_x_defer_bitwise(F, kind, variant, peer):
    """Deferred x update at P = 3: for the same slab split the iterates of
    x_defer = 8 (Hestenes-Stiefel with the peer halo: capped at 2) are bitwise those of
    x_defer = 1 after 11 iterations -- a complete group plus pending updates added by cg_end,
    with the halo / allreduce call sites of the multi-rank drivers in between."""
    P = 3
    nx, ny, nz = MESH
    h = 1.0 / nx
    c = I.ncomp(kind)
    g = I.rng(I.SEED_BASE + 615)
    lam, mu = I.materials(g, nx, ny, nz)
    b = I.interior_rhs(g, nx, ny, nz, c)
    plane = (nx + 1) * (ny + 1) * c
    res = {}
    for m in (1, 8):
        comms = F.Comm.loopback(P)

        def rank(r, st):
            mesh, op = _slab_op(F, comms[r], kind, nx, ny, nz, h, lam, mu)
            op.set_option("cg_variant", variant)
            if peer:
                op.set_option("peer_halo", 1)
            op.set_option("x_defer", m)
            want = m if (variant == 1 or not peer) else min(m, 2)
            assert op.get_option("x_defer") == want
            k0, k1 = mesh.plane_begin, mesh.plane_end
            bl = torch.from_numpy(b[k0 * plane:k1 * plane].copy()).cuda()
            xl = torch.zeros_like(bl)
            info = op.cg_solve(bl, xl, tol=0.0, maxit=11, stream=st)
            st.synchronize()
            out = (xl.cpu().numpy(), info["true_r_norm"])
            op.close(); mesh.close()
            return out

        res[m] = _run_ranks(P, rank)
        for cm in comms:
            cm.close()
    for a, bb in zip(res[1], res[8]):
        assert np.array_equal(a[0], bb[0])
        assert a[1] == bb[1]
