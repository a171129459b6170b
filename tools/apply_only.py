#!/usr/bin/env python
"""fem_apply on caller vectors (dense ABI layout) of a bench config, a few times: a short
program for ncu captures of the standalone apply kernels.  python tools/apply_only.py CONFIG [REPS]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2308_09839_b200 import inputs as I  # noqa: E402


def main():
    import torch
    from paper_2308_09839_b200 import fem
    fem.load(build_if_missing=False)
    idx = int(sys.argv[1])
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    cfg = I.CONFIGS[idx]
    kind = cfg["kind"]
    nx, ny, nz = I.config_cells(cfg)
    op = fem.Operator(fem.Mesh(nx, ny, nz, 1.0 / nx), kind, 1)
    if kind == "elastic":
        g = I.rng(I.SEED_BASE + idx)
        lam, mu = I.materials(g, nx, ny, nz)
        op.set_material(torch.from_numpy(lam).cuda(), torch.from_numpy(mu).cuda())
    x = torch.empty(op.n_local, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    y = torch.empty_like(x)
    for _ in range(reps):
        op.apply(x, y)
    torch.cuda.synchronize()
    print("apply path", op.get_option("last_apply_path"))


if __name__ == "__main__":
    main()
