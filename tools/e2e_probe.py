#!/usr/bin/env python
"""Where the time of one end-to-end fem_cg_solve on host buffers goes (C4 by default): the solve
as a whole, and its parts issued separately (H2D copies, cg_begin, the iterations, cg_end, D2H).
    python tools/e2e_probe.py [CONFIG] [ITERS]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2308_09839_b200 import inputs as I  # noqa: E402


def main():
    import torch
    from paper_2308_09839_b200 import fem
    fem.load(build_if_missing=False)
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    M = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    cfg = I.CONFIGS[idx]
    kind = cfg["kind"]
    nx, ny, nz = I.config_cells(cfg)
    op = fem.Operator(fem.Mesh(nx, ny, nz, 1.0 / nx), kind, 1)
    if kind == "elastic":
        g = I.rng(I.SEED_BASE + idx)
        lam, mu = I.materials(g, nx, ny, nz)
        op.set_material(torch.from_numpy(lam).cuda(), torch.from_numpy(mu).cuda())
        del lam, mu
    gb = I.rng(I.SEED_BASE + idx + 1000)
    bh = torch.from_numpy(I.interior_rhs(gb, nx, ny, nz, I.ncomp(kind))).pin_memory()
    xh = torch.zeros_like(bh).pin_memory()
    op.cg_solve(bh.numpy(), xh.numpy(), tol=0.0, maxit=M)  # warm
    T = []
    for _ in range(3):
        xh.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op.cg_solve(bh.numpy(), xh.numpy(), tol=0.0, maxit=M)
        T.append(time.perf_counter() - t0)
    print("solve on host buffers: %.1f ms (min of 3), %.2f GDOF/s" % (1e3 * min(T), op.n_local * M / min(T) / 1e9))
    bd = torch.empty(op.n_local, dtype=torch.float64, device="cuda")
    xd = torch.empty_like(bd)
    s = torch.cuda.current_stream()

    def timed(name, fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print("  %-22s %8.2f ms" % (name, 1e3 * dt))
        return dt

    tot = 0.0
    tot += timed("H2D b", lambda: bd.copy_(bh, non_blocking=True))
    xh.zero_()
    tot += timed("H2D x0", lambda: xd.copy_(xh, non_blocking=True))
    tot += timed("cg_begin", lambda: op.cg_begin(bd, xd, tol=0.0, maxit=M))
    tot += timed("cg_iterate(%d)" % M, lambda: op.cg_iterate(M))
    tot += timed("cg_end", lambda: op.cg_end())
    tot += timed("D2H x", lambda: xh.copy_(xd, non_blocking=True))
    print("  %-22s %8.2f ms" % ("sum of parts", 1e3 * tot))


if __name__ == "__main__":
    main()
