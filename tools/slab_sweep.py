#!/usr/bin/env python
"""Strong-scaling compute proxy: one rank's share of C4 (elasticity
384^3) and C2 / C3 (Laplace 256^3) at P = 1, 2, 4, 8 z-slabs, run as a single-GPU mesh of the
rank's cell layers (nz / P) -- the per-rank apply + update work of the slab-decomposed CG without
the halo and allreduce (which this one-GPU pool cannot measure).  CUDA graphs of K iterations,
events on the stream; one JSON line per point with the compute efficiency t(1) / (P t(P)).

    python tools/slab_sweep.py [--out FILE] [--steps K]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2308_09839_b200 import inputs as I  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--steps", type=int, default=24)
    args = ap.parse_args()
    import torch
    from paper_2308_09839_b200 import fem
    fem.load()
    s = torch.cuda.current_stream()
    out = open(args.out, "w") if args.out else None
    for kind, n in (("elastic", 384), ("scalar", 256), ("vector", 256)):
        t1 = None
        for P in (1, 2, 4, 8):
            nz = n // P
            g = I.rng(I.SEED_BASE + 900 + P)
            c = I.ncomp(kind)
            op = fem.Operator(fem.Mesh(n, n, nz, 1.0 / n), kind, 1)
            if kind == "elastic":
                lam, mu = I.materials(g, n, n, nz)
                op.set_material(torch.from_numpy(lam).cuda(), torch.from_numpy(mu).cuda())
                del lam, mu
            b = torch.from_numpy(I.interior_rhs(g, n, n, nz, c)).cuda()
            x = torch.zeros_like(b)
            op.cg_begin(b, x, tol=0.0, maxit=1 << 30)
            op.cg_iterate(8 + args.steps)  # warm-up + graph capture (K is a multiple of 8)
            op.cg_iterate(args.steps)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            op.cg_iterate(args.steps)
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            op.cg_end()
            t1 = ms if P == 1 else t1
            rec = {"kind": kind, "cells": [n, n, nz], "P": P, "ndof_rank": op.n_local,
                   "ms_per_iteration": ms, "gdofs_per_gpu": op.n_local / (ms / 1e3) / 1e9,
                   "compute_efficiency": t1 / (P * ms)}
            print(json.dumps(rec), flush=True)
            if out:
                out.write(json.dumps(rec) + "\n")
            del op, b, x
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
