#!/usr/bin/env python
"""Size sweep (SURVEY §8(d) "locates where peak is reached").

For each kind and cube size: operator-only GDOF/s (fem_apply on caller vectors, dense layout;
issued from the host per call, and replayed from one captured CUDA graph -- the GPU-side time
without the per-call host cost) and CG-iteration GDOF/s (fused CG, CUDA graphs), CUDA events on
the launching stream, one JSON line per point.  Working sets below 2x L2 are flagged "l2_resident" (not an HBM number).

    python tools/size_sweep.py [--kinds scalar,vector,elastic] [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2308_09839_b200 import inputs as I  # noqa: E402

SIZES = {"scalar": [16, 32, 64, 96, 128, 192, 256, 320, 384, 512],
         "vector": [16, 32, 64, 96, 128, 192, 256, 320],
         "elastic": [16, 32, 64, 96, 128, 192, 256, 320, 384]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kinds", default="scalar,vector,elastic")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import torch
    from paper_2308_09839_b200 import fem
    fem.load()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    s = torch.cuda.current_stream()
    out = open(args.out, "w") if args.out else None

    def events(fn, reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(s)
        for _ in range(reps):
            fn()
        b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    for kind in args.kinds.split(","):
        for n in SIZES[kind]:
            op = fem.Operator(fem.Mesh(n, n, n, 1.0 / n), kind, "dirichlet")
            g = I.rng(I.SEED_BASE + 500 + n)
            if kind == "elastic":
                lam, mu = I.materials(g, n, n, n)
                op.set_material(torch.from_numpy(lam).cuda(), torch.from_numpy(mu).cuda())
            ndof = op.n_global
            x = torch.empty(ndof, dtype=torch.float64, device="cuda").uniform_(-1, 1)
            y = torch.empty_like(x)
            for _ in range(3):
                op.apply(x, y)
            reps = max(5, min(200, int(2e9 / max(ndof, 1) / 8)))
            t_apply = events(lambda: op.apply(x, y), reps)
            # the same applies replayed from one captured CUDA graph: GPU time per apply without
            # the host's per-call cost (ctypes, argument checks, pointer query, launch)
            gs = torch.cuda.Stream()
            gs.wait_stream(s)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=gs):
                for _ in range(20):
                    op.apply(x, y, stream=gs)
            torch.cuda.synchronize()
            graph.replay()
            t_graph = events(lambda: graph.replay(), max(2, reps // 20)) / 20
            del graph
            b = torch.from_numpy(I.interior_rhs(g, n, n, n, I.ncomp(kind))).cuda()
            xs = torch.zeros_like(b)
            op.cg_begin(b, xs, tol=0.0, maxit=1 << 30)
            op.cg_iterate(8)
            its = max(8, min(400, reps))
            t_cg = events(lambda: op.cg_iterate(its), 1) / its
            op.cg_end()
            ws_bytes = 5 * ndof * 8 + (16 * n ** 3 if kind == "elastic" else 0)
            line = {"kind": kind, "cells": n, "ndof": ndof, "apply_ms": t_apply, "apply_graph_ms": t_graph,
                    "apply_gdofs": ndof / t_apply / 1e6, "cg_iter_ms": t_cg,
                    "cg_gdofs": ndof / t_cg / 1e6, "fused_cg": op.get_option("fused_cg"),
                    "l2_resident": ws_bytes < 2 * l2}
            print(json.dumps(line), flush=True)
            if out:
                out.write(json.dumps(line) + "\n"); out.flush()
            op.close()
            del x, y, b, xs
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
