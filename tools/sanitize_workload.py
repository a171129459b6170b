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
                op.apply(x)
                b = torch.zeros_like(x); b.uniform_(-1, 1)
                xs = torch.zeros_like(b)
                op.cg_solve(b, xs, tol=1e-10, maxit=8)
            op.close()
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
