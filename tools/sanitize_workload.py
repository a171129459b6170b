#!/usr/bin/env python
"""Small workload touching every kernel of libfem.so, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): SURVEY §4 "Sanitizers" on C1 and a 16^3 mesh.

    compute-sanitizer --tool memcheck python tools/sanitize_workload.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2308_09839_b200 import inputs as I  # noqa: E402


def main():
    import torch
    from paper_2308_09839_b200 import fem
    fem.load(build_if_missing=False)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    for n in (8, 16):
        g = I.rng(I.SEED_BASE + 77 + n)
        lam, mu = I.materials(g, n, n, n)
        for kind in ("scalar", "vector", "elastic"):
            c = I.ncomp(kind)
            for quad in (0, 1):
                op = fem.Operator(fem.Mesh(n, n, n, 1.0 / n), kind, 1)
                op.set_option("quadrature", quad)
                if kind == "elastic":
                    op.set_material(dev(lam), dev(mu))
                x = dev(I.uniform_vector(g, n, n, n, c))
                y = op.apply(x)                                   # dense (bulk-row) apply
                op.apply_ghost_padded(x, None, None)              # TMA apply
                op.dot(x, y)
                b = dev(I.interior_rhs(g, n, n, n, c))
                for variant in (0, 1):                            # fused CG, single-reduction CG
                    op.set_option("cg_variant", variant)
                    xs = torch.zeros_like(b)
                    op.cg_solve(b, xs, tol=1e-10, maxit=12)
                if quad == 0 and n == 8:
                    A = op.csr()
                    A.apply(x)
                    A.close()
                op.close()
        # general hex mesh, matrix-free and partial assembly
        coords, cells, bnd = I.hex_box_mesh(n, n, n, g=g, jitter=0.15, permute=True)
        hl, hm = I.materials(g, cells.shape[0], 1, 1)
        for kind in ("scalar", "elastic"):
            op = fem.Operator(fem.HexMesh(dev(coords), dev(cells), dev(bnd)), kind, 1)
            if kind == "elastic":
                op.set_material(dev(hl), dev(hm))
            x = dev(np.random.default_rng(0).uniform(-1, 1, coords.shape[0] * I.ncomp(kind)))
            for pa in (0, 1):
                op.set_option("partial_assembly", pa)
                for det in (0, 1):  # atomic scatter / element outputs + ordered node gather
                    op.set_option("deterministic", det)
                    op.apply(x)
                    b = torch.zeros_like(x); b.uniform_(-1, 1)
                    xs = torch.zeros_like(b)
                    op.cg_solve(b, xs, tol=1e-10, maxit=8)
                op.set_option("deterministic", 0)
            op.close()
    # round 2: meshes with interior CTAs (Laplace interior march, elasticity interior / edge
    # grids side by side), the dot-implementation modes, box partial assembly (21 values), and
    # P = 2 slab ranks through the loopback communicator (halo overlap, peer halo)
    n = 72
    g = I.rng(I.SEED_BASE + 177)
    lam, mu = I.materials(g, n, n, n)
    for kind in ("scalar", "vector", "elastic"):
        c = I.ncomp(kind)
        op = fem.Operator(fem.Mesh(n, n, n, 1.0 / n), kind, 1)
        if kind == "elastic":
            op.set_material(dev(lam), dev(mu))
        x = dev(I.uniform_vector(g, n, n, n, c))
        op.apply(x)
        b = dev(I.interior_rhs(g, n, n, n, c))
        for dm in (0, 1, 2):
            op.set_option("dot_mode", dm)
            xs = torch.zeros_like(b)
            op.cg_solve(b, xs, tol=0.0, maxit=4)
        op.set_option("dot_mode", 0)
        for m in (1, 2, 4, 8):  # deferred x update: complete groups + pending updates at cg_end
            op.set_option("x_defer", m)
            xs = torch.zeros_like(b)
            op.cg_solve(b, xs, tol=0.0, maxit=11)
        op.set_option("x_defer", 8)
        if kind == "elastic":
            op.set_option("partial_assembly", 1)
            op.apply(x)
            xs = torch.zeros_like(b)
            op.cg_solve(b, xs, tol=0.0, maxit=3)
        op.close()
    import threading
    nx, ny, nz = 40, 36, 30
    x = I.uniform_vector(g, nx, ny, nz, 3)
    lam, mu = I.materials(g, nx, ny, nz)
    for peer in (False, True):
        comms = fem.Comm.loopback(2)
        errs = []

        def rank(r):
            try:
                torch.cuda.set_device(0)
                st = torch.cuda.Stream()
                with torch.cuda.stream(st):
                    mesh = fem.Mesh(nx, ny, nz, 1.0 / nx, comms[r])
                    op = fem.Operator(mesh, "elastic", 1)
                    k0, k1 = mesh.plane_begin, mesh.plane_end
                    lb, le = max(k0 - 1, 0), min(k1, nz)
                    op.set_material(np.ascontiguousarray(lam[lb * nx * ny:le * nx * ny]),
                                    np.ascontiguousarray(mu[lb * nx * ny:le * nx * ny]), lb, le - lb)
                    if peer:
                        op.set_option("peer_halo", 1)
                    plane = (nx + 1) * (ny + 1) * 3
                    xl = dev(x[k0 * plane:k1 * plane])
                    op.apply(xl, stream=st)
                    xs = torch.zeros_like(xl)
                    op.cg_solve(xl, xs, tol=0.0, maxit=11, stream=st)
                    st.synchronize()
                    op.close(); mesh.close()
            except BaseException as ex:
                errs.append(ex)

        ts = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for cm in comms:
            cm.close()
        if errs:
            raise errs[0]
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
