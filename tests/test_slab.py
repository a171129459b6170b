"""Slab decomposition.

CPU (gloo, world_size 2/3): every rank computes its plane range with the library's own
fem_partition, the ranges tile [0, nz] exactly, and the one-plane halo protocol of the library
(send the first owned plane down, the last one up) delivers each neighbour's boundary planes.

GPU (single-process loopback, NCCL cannot put two ranks on one GPU): P virtual slabs applied
one after the other with explicit ghost planes (fem_apply_ghost) reproduce the P = 1 apply
BITWISE, for every kind and P in {2, 3, 5}.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_09839_b200 import inputs as I


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nx, ny, nz, c, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2308_09839_b200 import fem
        fem.load()
        k0, k1 = fem.partition(nz, world, rank)
        # 1) ranges tile the node planes
        rng = torch.tensor([k0, k1], dtype=torch.int64)
        allr = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allr, rng)
        allr = [tuple(int(v) for v in t) for t in allr]
        assert allr[0][0] == 0 and allr[-1][1] == nz + 1
        for a, b in zip(allr, allr[1:]):
            assert a[1] == b[0]
        sizes = [e - b for b, e in allr]
        assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1
        # 2) halo protocol on a global field (plane index encoded in the values)
        plane = (nx + 1) * (ny + 1) * c
        glob = torch.arange((nz + 1) * plane, dtype=torch.float64)
        mine = glob[k0 * plane:k1 * plane].clone()
        lo = torch.full((plane,), float("nan"), dtype=torch.float64)
        hi = torch.full((plane,), float("nan"), dtype=torch.float64)
        ops = []
        if rank > 0:
            ops += [dist.P2POp(dist.isend, mine[:plane].clone(), rank - 1),
                    dist.P2POp(dist.irecv, lo, rank - 1)]
        if rank < world - 1:
            ops += [dist.P2POp(dist.isend, mine[-plane:].clone(), rank + 1),
                    dist.P2POp(dist.irecv, hi, rank + 1)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        if rank > 0:
            assert torch.equal(lo, glob[(k0 - 1) * plane:k0 * plane])
        if rank < world - 1:
            assert torch.equal(hi, glob[k1 * plane:(k1 + 1) * plane])
        # 3) material layers a rank needs: cells adjacent to its owned planes
        need0, need1 = max(k0 - 1, 0), min(k1 - 1, nz - 1)
        assert need0 <= need1
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported through the queue
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partition_and_halo_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 6, 5, 10, 3, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res


def test_partition_edge_cases():
    from paper_2308_09839_b200 import fem
    assert fem.partition(7, 1, 0) == (0, 8)
    assert fem.partition(7, 8, 7) == (7, 8)
    with pytest.raises(fem.FemError):
        fem.partition(6, 8, 0)  # 7 planes, 8 ranks
    with pytest.raises(fem.FemError):
        fem.partition(10, 2, 2)
    # C4 at P = 8: 385 planes -> 48 or 49 per rank
    sizes = [e - b for b, e in (fem.partition(384, 8, r) for r in range(8))]
    assert sorted(set(sizes)) == [48, 49] and sum(sizes) == 385


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("P", [2, 3, 5])
def test_loopback_slabs_bitwise(kind, P):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2308_09839_b200 import fem
    nx, ny, nz, h = 37, 30, 23, 0.04
    c = I.ncomp(kind)
    g = I.rng(I.SEED_BASE + 500)
    x = torch.from_numpy(I.uniform_vector(g, nx, ny, nz, c)).cuda()
    lam, mu = I.materials(g, nx, ny, nz)
    ref_op = fem.Operator(fem.Mesh(nx, ny, nz, h), kind, 1)
    if kind == "elastic":
        ref_op.set_material(lam, mu)
    ref = ref_op.apply(x)
    plane = (nx + 1) * (ny + 1) * c
    outs, outs_tma = [], []
    for r in range(P):
        comm = fem.Comm(P, r)  # virtual: partition only
        mesh = fem.Mesh(nx, ny, nz, h, comm)
        k0, k1 = mesh.plane_begin, mesh.plane_end
        op = fem.Operator(mesh, kind, 1)
        if kind == "elastic":
            lb, le = max(k0 - 1, 0), min(k1, nz)
            op.set_material(np.ascontiguousarray(lam[lb * nx * ny:le * nx * ny]),
                            np.ascontiguousarray(mu[lb * nx * ny:le * nx * ny]), lb, le - lb)
        xl = x[k0 * plane:k1 * plane].contiguous()
        lo = x[(k0 - 1) * plane:k0 * plane].contiguous() if k0 > 0 else None
        hi = x[k1 * plane:(k1 + 1) * plane].contiguous() if k1 <= nz else None
        outs.append(op.apply_ghost(xl, lo, hi))
        outs_tma.append(op.apply_ghost_padded(xl, lo, hi))  # the CG kernels' TMA path
        with pytest.raises(fem.FemError) as e:
            op.apply(xl)  # a virtual communicator cannot exchange
        assert e.value.status == fem.FEM_EUNSUPPORTED
    y = torch.cat(outs)
    assert torch.equal(y, ref)
    # TMA (padded-layout) path: bitwise equal to its own P = 1 result across slabs
    ref_tma = ref_op.apply_ghost_padded(x, None, None)
    assert torch.equal(torch.cat(outs_tma), ref_tma)
    assert float((ref_tma - ref).abs().max()) <= 1e-12 * float(ref.abs().max())


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["scalar", "vector", "elastic"])
@pytest.mark.parametrize("P", [2, 3])
def test_loopback_peer_halo_bitwise(kind, P):
    """Peer halo: every slab operator reads its ghost planes from the neighbour operators' padded
    buffers inside the TMA pipeline (fem_op_link_peers), reproducing P = 1 bitwise."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2308_09839_b200 import fem
    nx, ny, nz, h = 37, 30, 23, 0.04
    c = I.ncomp(kind)
    g = I.rng(I.SEED_BASE + 510)
    x = torch.from_numpy(I.uniform_vector(g, nx, ny, nz, c)).cuda()
    lam, mu = I.materials(g, nx, ny, nz)
    ref_op = fem.Operator(fem.Mesh(nx, ny, nz, h), kind, 1)
    if kind == "elastic":
        ref_op.set_material(lam, mu)
    ref = ref_op.apply_ghost_padded(x, None, None)
    plane = (nx + 1) * (ny + 1) * c
    ops, xs, keep = [], [], []
    for r in range(P):
        comm = fem.Comm(P, r)
        mesh = fem.Mesh(nx, ny, nz, h, comm)
        k0, k1 = mesh.plane_begin, mesh.plane_end
        op = fem.Operator(mesh, kind, 1)
        if kind == "elastic":
            lb, le = max(k0 - 1, 0), min(k1, nz)
            op.set_material(np.ascontiguousarray(lam[lb * nx * ny:le * nx * ny]),
                            np.ascontiguousarray(mu[lb * nx * ny:le * nx * ny]), lb, le - lb)
        ops.append(op); xs.append(x[k0 * plane:k1 * plane].contiguous()); keep.append((comm, mesh))
    for r, op in enumerate(ops):
        op.link_peers(ops[r - 1] if r > 0 else None, ops[r + 1] if r < P - 1 else None)
        assert op.get_option("peer_halo") == 1
    for r, op in enumerate(ops):  # first pass stages every slab's x in its padded buffer
        op.apply_ghost_padded(xs[r], None, None)
    y = torch.cat([op.apply_ghost_padded(xs[r], None, None) for r, op in enumerate(ops)])
    assert torch.equal(y, ref)


def _ipc_worker(rank, world, port, kind, q):
    import torch.distributed as dist
    from paper_2308_09839_b200 import fem
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        nx, ny, nz, h = 37, 30, 23, 0.04
        c = I.ncomp(kind)
        g = I.rng(I.SEED_BASE + 520)
        xfull = I.uniform_vector(g, nx, ny, nz, c)
        lam, mu = I.materials(g, nx, ny, nz)
        comm = fem.Comm(world, rank)  # virtual: the partition; the exchange goes through IPC
        mesh = fem.Mesh(nx, ny, nz, h, comm)
        k0, k1 = mesh.plane_begin, mesh.plane_end
        op = fem.Operator(mesh, kind, 1)
        if kind == "elastic":
            lb, le = max(k0 - 1, 0), min(k1, nz)
            op.set_material(np.ascontiguousarray(lam[lb * nx * ny:le * nx * ny]),
                            np.ascontiguousarray(mu[lb * nx * ny:le * nx * ny]), lb, le - lb)
        infos = [None] * world
        dist.all_gather_object(infos, op.peer_info())
        op.open_peers(infos[rank - 1] if rank > 0 else None, infos[rank + 1] if rank < world - 1 else None)
        plane = (nx + 1) * (ny + 1) * c
        xl = torch.from_numpy(xfull[k0 * plane:k1 * plane].copy()).cuda()
        op.apply_ghost_padded(xl, None, None)  # stage x in the padded buffer the neighbours read
        torch.cuda.synchronize(); dist.barrier()
        y = op.apply_ghost_padded(xl, None, None)
        torch.cuda.synchronize(); dist.barrier()
        outs = [None] * world
        dist.all_gather_object(outs, y.cpu().numpy())
        if rank == 0:
            ref_op = fem.Operator(fem.Mesh(nx, ny, nz, h), kind, 1)
            if kind == "elastic":
                ref_op.set_material(lam, mu)
            ref = ref_op.apply_ghost_padded(torch.from_numpy(xfull).cuda(), None, None).cpu().numpy()
            q.put(bool(np.array_equal(np.concatenate(outs), ref)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as ex:  # reported to the parent
        q.put(repr(ex))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["scalar", "elastic"])
def test_ipc_peer_halo_two_processes(kind):
    """Two processes on one GPU exchange CUDA IPC handles (fem_op_peer_info / fem_op_open_peers,
    bytes sent over gloo); each slab's apply loads its ghost planes from the other process's
    memory inside the TMA pipeline; the slabs reproduce P = 1 bitwise."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert res is True, res
