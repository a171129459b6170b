#!/usr/bin/env python
"""Benchmark of the hot path: FP64 matrix-free Q1 operator inside CG on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl native|reference]

Default workload: BASELINE.json configs[3] -- isotropic elasticity on 384^3 hexes with cell-wise
discontinuous lambda/mu, homogeneous Dirichlet box, CG (the configuration the headline metric
"CG operator apply GDOF/s (FP64) and % of HBM roofline at 1/2/4/8 B200 vs CSR SpMV" is quoted
on).  A step is one CG iteration = apply (+ fused p.Ap) + x/r update (+ fused r.r) + p update
(+ the NCCL halo and the two allreduces when N > 1).  value = global DOF x steps / time.
N > 1: the same global mesh is slab-decomposed in z (strong scaling), one rank per GPU.

--impl reference: the CPU oracle (oracle/, plain quadrature apply + CG) timed on the host
cores on a bounded sub-box of the same workload (this tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2308_09839_b200 import inputs as I  # noqa: E402

METRIC = "CG operator apply GDOF/s (FP64) and % of HBM roofline at 1/2/4/8 B200 vs CSR SpMV"
UNIT = "GDOF/s"


# ------------------------------------------------------------------------------------------
# helpers
# ------------------------------------------------------------------------------------------
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def algorithmic_apply_bytes(kind, nx, ny, nz):
    """SURVEY §8(d) / DESIGN.md §6: x read once + y written once (8 B each per DOF), plus
    lambda, mu once per cell for elasticity (16 B/cell).  Connectivity, coordinates and the
    Dirichlet mask are implicit (0 B)."""
    ndof = I.n_nodes(nx, ny, nz) * I.ncomp(kind)
    b = 16 * ndof
    if kind == "elastic":
        b += 16 * nx * ny * nz
    return b


def cg_apply_bytes(kind, nx, ny, nz, fused):
    """Algorithmic bytes of the apply launched inside one CG iteration.  Fused:
    read r and p_old, write p and q (32 B/DOF) + lambda, mu (16 B/cell); unfused: 16 B/DOF."""
    ndof = I.n_nodes(nx, ny, nz) * I.ncomp(kind)
    b = (32 if fused else 16) * ndof
    if kind == "elastic":
        b += 16 * nx * ny * nz
    return b


# General-hex kernel (kernels_hex.cu): FP64 operations per cell of the per-cell body, counted
# from the SASS (DADD + DMUL + 2 DFMA; tools/sass_mix.sh), CG mode (with the energy for p.Ap).
HEX_FLOPS_PER_CELL = {"elastic": 635 + 337 + 2 * 609, "vector": 594 + 345 + 2 * 609,
                      "scalar": 302 + 175 + 2 * 323}
FP64_PEAK_TFLOPS = 2 * 17.08  # own DFMA microbenchmark, profiles/r01_microbench_fp64_hbm.txt


def cg_vector_bytes(ndof, fused, x_defer=1, steps=None, cgcg=False):
    # update: read x,p,r,q write x,r (48 B/DOF); unfused p-update: read r,p write p (24 B/DOF);
    # deferred x update over m iterations: r, q -> r every iteration, x and the
    # group's m p vectors -> x once per group: 24 + (16 + 8 m) / m = 32 + 16 / m B/DOF in the
    # steady state; a timed pass of K steps ending on a group boundary holds ceil(K / m) x updates
    if cgcg:  # single reduction: r, w, p_old, s -> p, s, r (56 B/DOF) + x += alpha p (16 B/DOF every
        # iteration, or x and the group's m - 1 older p vectors once per group of m)
        if x_defer <= 1:
            return 72 * ndof
        per_group = 16 + 8 * (x_defer - 1)
        if steps:
            return (56 + -(-steps // x_defer) * per_group / steps) * ndof
        return (56 + per_group / x_defer) * ndof
    if x_defer > 1:  # fused: r, q -> r; unfused: the same + the p-update r, p -> p (24 B/DOF)
        base = 24 if fused else 48
        if steps:
            return (base + -(-steps // x_defer) * (16 + 8 * x_defer) / steps) * ndof
        return (base + 8 + 16 / x_defer) * ndof
    return (48 if fused else 72) * ndof


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------------------------------
# CPU oracle legs (cpu_baseline and --impl reference)
# ------------------------------------------------------------------------------------------
def oracle_sample_dims(kind):
    # bounded sub-box of the same workload: ~3-5 s per oracle CG iteration on 16 cores
    return {"elastic": (96, 96, 96), "vector": (48, 48, 48), "scalar": (160, 160, 160)}[kind]


def oracle_cg_rate(kind, iters=2, hexmesh=False):
    from oracle import oracle as O
    nx, ny, nz = oracle_sample_dims(kind)
    h = 1.0 / nx
    g = I.rng(I.SEED_BASE + 77)
    lam, mu = I.materials(g, nx, ny, nz)
    b = I.interior_rhs(g, nx, ny, nz, I.ncomp(kind))
    if hexmesh:
        coords, cells, bnd = I.hex_box_mesh(nx, ny, nz, h=h, g=g, jitter=0.2)

        def run(m):
            O.cg_hex(kind, coords, cells, b, bnd, tol=0.0, maxit=m, lam=lam, mu=mu)
    else:
        def run(m):
            O.cg(kind, 1, nx, ny, nz, h, b, tol=0.0, maxit=m, lam=lam, mu=mu)
    t0 = time.perf_counter()
    run(0)
    t1 = time.perf_counter()
    run(iters)
    t2 = time.perf_counter()
    it_time = max((t2 - t1) - (t1 - t0), 1e-9) / iters
    cores = O.max_threads()
    return b.size / it_time / 1e9, cores, f"oracle CG on {kind} {nx}x{ny}x{nz}" \
        f"{' general hex (jittered)' if hexmesh else ''} (same recipe), " \
        f"{iters} iterations timed (init/true-residual applies subtracted), {b.size} DOF"


def run_reference(args, cfg):
    """Reference arm: the oracle as it stands, on host cores; rank 0 only."""
    ws, rank, _ = dist_setup()
    if rank != 0:
        return
    from oracle import oracle as O
    O.build()
    kind = cfg["kind"]
    nx, ny, nz = oracle_sample_dims(kind)
    h = 1.0 / nx
    g = I.rng(I.SEED_BASE + 77)
    lam, mu = I.materials(g, nx, ny, nz)
    b = I.interior_rhs(g, nx, ny, nz, I.ncomp(kind))
    hexmesh = cfg.get("mesh") == "hex"
    if hexmesh:  # general-hex workload: the oracle's Alg. 1 path on a jittered sub-box
        coords, cells, bnd = I.hex_box_mesh(nx, ny, nz, h=h, g=g, jitter=cfg["jitter"])

        def run(m):
            O.cg_hex(kind, coords, cells, b, bnd, tol=0.0, maxit=m, lam=lam, mu=mu)
    else:
        def run(m):
            O.cg(kind, 1, nx, ny, nz, h, b, tol=0.0, maxit=m, lam=lam, mu=mu)
    # each step = one oracle CG iteration on the bounded sub-box
    run(0)  # warm the library
    ta = time.perf_counter()
    run(0)
    t_fixed = time.perf_counter() - ta
    for _ in range(args.warmup):
        pass  # the oracle has no warm-up state; warm-up steps are not re-run to bound the time
    t0 = time.perf_counter()
    run(args.steps)
    t = max(time.perf_counter() - t0 - t_fixed, 1e-9)
    value = b.size * args.steps / t / 1e9
    cores = O.max_threads()
    sample = (f"oracle CG on {kind} {nx}x{ny}x{nz} cells (sub-box of {cfg['name']}, same input "
              f"recipe), {args.steps} iterations, init/true-residual applies subtracted")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True,
        "scaling": "weak" if ("planes_per_rank" in cfg or cfg.get("mesh") == "hex") else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "kind": kind, "cells": list(I.config_cells(cfg, ws)),
                   "sample_cells": [nx, ny, nz], "bc": "dirichlet_box"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# native arm
# ------------------------------------------------------------------------------------------
def run_native(args, cfg):
    import torch

    ws, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2308_09839_b200 import fem
    fem.load(build_if_missing=(rank == 0 and ws == 1))

    kind = cfg["kind"]
    nx, ny, nz = I.config_cells(cfg, ws)
    h = 1.0 / nx
    c = I.ncomp(kind)
    hexmesh = cfg.get("mesh") == "hex"
    scaling = "weak" if ("planes_per_rank" in cfg or hexmesh) else "strong"
    comm = None
    if ws > 1 and not hexmesh:
        uid = [fem.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = fem.Comm(ws, rank, uid[0])
    if hexmesh:  # single-GPU operator: N ranks run N independent replicas ("replicas only")
        gm = I.rng(I.SEED_BASE + args.config + 2000)
        coords, cells, bnd = I.hex_box_mesh(nx, ny, nz, h=h, g=gm, jitter=cfg["jitter"])
        mesh = fem.HexMesh(torch.from_numpy(coords).cuda(), torch.from_numpy(cells).cuda(),
                           torch.from_numpy(bnd).cuda())
        del coords, cells, bnd
    else:
        mesh = fem.Mesh(nx, ny, nz, h, comm)
    op = fem.Operator(mesh, kind, "dirichlet")
    if args.pa:  # partial assembly (Table 3): hex -- stored geometry; box elasticity --
        op.set_option("partial_assembly", 1)  # 21 values per Gauss point, D_q = w det J C_e
    if args.x_defer > 0:  # option x_defer (fused CG: x advanced every m-th iteration)
        op.set_option("x_defer", args.x_defer)
    if args.det and hexmesh:  # general hexes: no FP64 atomics, bitwise reproducible
        op.set_option("deterministic", 1)
    if args.gll:  # Gauss-Lobatto quadrature: the BP5 / BP6 operators (reading R1)
        op.set_option("quadrature", 1)
    if args.cgcg:  # Chronopoulos-Gear single-reduction CG (NEXT #1)
        op.set_option("cg_variant", 1)
    if args.dot != "fused":  # the dot ablation: separate dot kernels / atomic partials
        op.set_option("dot_mode", {"separate": 1, "atomic": 2}[args.dot])
    if args.peer_halo and ws > 1 and not hexmesh:  # ghost planes over NVLink inside the apply (NEXT #3)
        op.set_option("peer_halo", 1)
    ndof_global = op.n_global * (ws if hexmesh else 1)
    k0, k1 = (0, nz + 1) if hexmesh else (mesh.plane_begin, mesh.plane_end)
    plane = (nx + 1) * (ny + 1)

    # ---- inputs (seeded, synthetic, SURVEY §8(d) recipe) ----
    g = I.rng(I.SEED_BASE + args.config)
    if kind == "elastic":
        lam, mu = I.materials(g, nx, ny, nz)
        lb = max(k0 - 1, 0)
        le = min(k1, nz)
        sl = slice(lb * nx * ny, le * nx * ny)
        if hexmesh:
            op.set_material(torch.from_numpy(lam).cuda(), torch.from_numpy(mu).cuda())
        else:
            op.set_material(torch.from_numpy(lam[sl]).cuda(), torch.from_numpy(mu[sl]).cuda(),
                            layer_begin=lb, n_layers=le - lb)
        del lam, mu
    gb = I.rng(I.SEED_BASE + args.config + 1000)
    b_full = I.interior_rhs(gb, nx, ny, nz, c)
    b_loc = np.ascontiguousarray(b_full[k0 * plane * c:k1 * plane * c])
    del b_full
    b = torch.from_numpy(b_loc).cuda()
    x = torch.zeros_like(b)
    stream = torch.cuda.current_stream()

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up (W CG steps) ----
    # The timed region replays the library's plain CUDA graph of K iterations (fem_cg_iterate
    # captures graphs of exactly k <= 64 iterations per p-ring phase), as fem_cg_solve runs
    # them; the warm-up runs W iterations and then K more, so the graph is captured beforehand.
    op.set_option("time_apply", 0)
    op.cg_begin(b, x, tol=0.0, maxit=1 << 30)
    its = [0]  # iterations run so far: every K-step pass starts at the same ring phase, so

    def iterate(k):  # the graphs the timed passes replay are the ones captured before them
        op.cg_iterate(k)
        its[0] += k

    def even():
        # every K-step pass starts at the same phase of the p-buffer ring (m <= 8 buffers, option
        # x_defer), chosen so that the pass ENDS on a group boundary: its last iteration performs
        # the x update of its group, so a pass of K iterations contains ceil(K / m) x updates --
        # never fewer than the steady-state K / m (the bytes below count exactly these)
        want = (-args.steps) % 8
        if its[0] % 8 != want:
            iterate((want - its[0]) % 8)

    iterate(args.warmup)
    even()
    iterate(args.steps)  # captures the plain K-iteration graph
    even()
    torch.cuda.synchronize()

    # ---- the apply's duration: option time_apply runs K iterations as ONE captured graph whose
    # event-record nodes bracket every apply launch (fem_apply_time).  One such pass right before
    # and one right after the timed region; their mean brackets the timed region in time (the
    # clocks drift under the power cap from pass to pass) ----
    def apply_pass():
        op.set_option("time_apply", 1)
        op.apply_time()  # discard earlier events
        f0 = torch.cuda.Event(enable_timing=True); f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        iterate(args.steps)
        f1.record(stream)
        torch.cuda.synchronize()
        tot, n = op.apply_time()
        op.set_option("time_apply", 0)
        even()
        return f0.elapsed_time(f1), tot / max(n, 1), n

    op.set_option("time_apply", 1)
    iterate(args.steps)  # captures (and runs once) the K-iteration timed graph
    op.set_option("time_apply", 0)
    even()
    torch.cuda.synchronize()
    ev_ms_a, apply_a, n_apply = apply_pass()

    # ---- timed region: exactly K CG steps (the library's plain CUDA graphs) ----
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    l0 = fem.launch_count()
    wall0 = time.perf_counter()
    e0.record(stream)
    iterate(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    wall = time.perf_counter() - wall0
    launches = fem.launch_count() - l0
    clocks = sampler.stop()
    ms = max_over_ranks(e0.elapsed_time(e1))
    even()
    ev_ms_b, apply_b, _ = apply_pass()
    ms_event_graph = max_over_ranks(0.5 * (ev_ms_a + ev_ms_b))
    apply_ms = max_over_ranks(0.5 * (apply_a + apply_b))
    info = op.cg_end()
    value = ndof_global * args.steps / (ms / 1e3) / 1e9

    # ---- roofline of the dominant kernel (the apply) ----
    hbm_peak, peak_src = measured_peaks()
    nloc_planes = k1 - k0
    fused = bool(op.get_option("fused_cg"))
    cgcg = bool(op.get_option("cg_variant"))
    if cgcg:  # apply reads r, writes w (16 B/DOF); update: cg_vector_bytes
        fused = False
    # algorithmic bytes of one rank's apply launch: owned planes (+ its cell layers)
    x_defer = op.get_option("x_defer")
    alg_bytes = cg_apply_bytes(kind, nx, ny, nz, fused) * nloc_planes / (nz + 1)
    if args.pa and not hexmesh:  # box PA: 21 x 8 stored doubles per cell (Table 3) + u read + y write
        alg_bytes = 21 * 8 * 8 * nx * ny * nz + 16 * op.n_global
    achieved = alg_bytes / (apply_ms / 1e3) / 1e9
    if hexmesh:  # FP64-bound: flops of the per-cell body / apply time
        hex_flops = HEX_FLOPS_PER_CELL[kind] * nx * ny * nz
        achieved_tf = hex_flops / (apply_ms / 1e3) / 1e12
        if args.pa:  # partial assembly is HBM-bound: stored geometry + node map + vectors
            ncell = nx * ny * nz
            K = 9 if kind == "elastic" else 6
            alg_bytes = (8 * K * 8 + 32 + (16 if kind == "elastic" else 0)) * ncell + \
                (8 + 8 + 8) * op.n_global  # geometry, node map, material; u read, y zero + write
            achieved = alg_bytes / (apply_ms / 1e3) / 1e9
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", f"traffic_{cfg['name']}.json")
    if os.path.exists(tr_path) and ws == 1:
        with open(tr_path) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    share = apply_ms * args.steps / ms

    extra = {}
    # ---- operator-only throughput (Fig. 3/9 analogue) on the same stream ----
    xx = torch.empty_like(b).uniform_(-1, 1)
    yy = torch.empty_like(b)
    for _ in range(3):
        op.apply(xx, yy)
    torch.cuda.synchronize()
    R = 10
    a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
    barrier()
    a0.record(stream)
    for _ in range(R):
        op.apply(xx, yy)
    a1.record(stream)
    torch.cuda.synchronize()
    ams = max_over_ranks(a0.elapsed_time(a1) / R)
    extra["apply_only_gdofs"] = ndof_global / (ams / 1e3) / 1e9
    extra["apply_only_ms"] = ams
    if not hexmesh:  # fem_apply on the caller's vectors: algorithmic bytes / time vs the HBM peak
        ab = algorithmic_apply_bytes(kind, nx, ny, nz) * nloc_planes / (nz + 1)
        if args.pa:  # the stored 21 x 8 values per cell instead of lambda, mu
            ab = 21 * 8 * 8 * nx * ny * nz + 16 * op.n_global
        extra["apply_only_gbs"] = ab / (ams / 1e3) / 1e9
        extra["apply_only_frac"] = extra["apply_only_gbs"] / hbm_peak
        extra["apply_only_path"] = ["bulk rows", "tensor map", "row-pair tensor map"][op.get_option("last_apply_path")]
    extra["apply_in_cg_ms"] = apply_ms
    extra["apply_launches_timed"] = n_apply
    extra["cg_iteration_ms_event_graph"] = ms_event_graph / args.steps  # the time_apply pass
    extra["apply_share_of_step"] = share
    extra["cg_iteration_ms"] = ms / args.steps
    cg_bytes = cg_apply_bytes(kind, nx, ny, nz, fused) + cg_vector_bytes(ndof_global, fused, x_defer, args.steps, cgcg)
    extra["cg_bytes_per_dof_alg"] = cg_bytes / ndof_global
    extra["cg_iteration_gbs"] = cg_bytes / (ms / args.steps / 1e3) / 1e9
    extra["cg_iteration_frac"] = extra["cg_iteration_gbs"] / hbm_peak  # whole step (apply + updates)
    extra["fused_cg"] = fused
    extra["cg_variant"] = "chronopoulos-gear" if cgcg else "hestenes-stiefel"
    extra["dot_mode"] = "single reduction (CG-CG)" if cgcg else args.dot
    extra["x_defer"] = x_defer
    del xx, yy

    # ---- e2e: the public call a user makes, with pinned HOST buffers ----
    e2e = None
    if not args.no_e2e:
        bh = torch.from_numpy(b_loc).pin_memory()
        xh = torch.zeros(b_loc.size, dtype=torch.float64).pin_memory()
        M = args.e2e_iters
        op.set_option("time_apply", 0)
        op.cg_solve(bh.numpy(), xh.numpy(), tol=0.0, maxit=M)  # warm (graph capture)
        reps, tsum = 2, 0.0
        for _ in range(reps):
            xh.zero_()  # the caller's x0 (outside the timed call: input preparation, not the solve)
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            op.cg_solve(bh.numpy(), xh.numpy(), tol=0.0, maxit=M)  # H2D b, x0 ... D2H x, synchronising
            torch.cuda.synchronize()
            tsum += time.perf_counter() - t0
        barrier()
        et = max_over_ranks(tsum / reps)
        e2e = {"value": ndof_global * M / et / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(2 * b_loc.nbytes), "d2h_bytes_per_step": int(b_loc.nbytes),
               "step": f"one fem_cg_solve call ({M} iterations) with pinned host b, x; per-rank bytes"}

    # ---- CSR SpMV baseline, same box (N = 1) ----
    if ws == 1 and not args.no_csr and not hexmesh:
        extra.update(csr_compare(fem, torch, kind, args))

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N = 1) ----
    cpu = None
    if ws == 1 and rank == 0 and not args.no_cpu:
        try:
            v, cores, sample = oracle_cg_rate(kind, hexmesh=hexmesh)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}
        except Exception as ex:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "oracle",
                   "sample": f"failed: {ex}"}

    l2_bytes = torch.cuda.get_device_properties(local).L2_cache_size
    vec_bytes = 8 * op.n_local
    if 2 * vec_bytes > l2_bytes:
        l2_label = ("inputs larger than L2 (vectors %.3f GB each per rank, L2 %.0f MB)"
                    % (vec_bytes / 1e9, l2_bytes / 1e6))
    else:
        l2_label = ("L2-resident (vectors %.2f MB each per rank, L2 %.0f MB): latency-bound, "
                    "not a roofline number" % (vec_bytes / 1e6, l2_bytes / 1e6))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": cfg["name"], "kind": kind, "cells": [nx, ny, nz],
                       "mesh": ("general hex: explicit node map + coordinates, interior nodes jittered "
                                f"U(-{cfg['jitter']}, {cfg['jitter']}) h" if hexmesh else "box"),
                       "ndof": ndof_global, "bc": "dirichlet_box",
                       "material": "E=10^U(0,2), nu=U(0.20,0.35) per cell" if kind == "elastic" else None,
                       "parallelism": (f"z-slab x{ws}" + (" peer-halo" if args.peer_halo else " nccl-halo"))
                                      if ws > 1 else "single GPU",
                       "l2": l2_label},
            "roofline": ({"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                          "frac": achieved / hbm_peak, "traffic": traffic,
                          "kernel": (f"{kind} fused CG apply (p = r + beta p_old, q = A p, p.q)" if fused
                                     else (f"{kind} apply (single-reduction CG: w = A r, w.r, r.r)" if cgcg
                                           else ("pa21_kernel (partial assembly, 21 values per Gauss point, "
                                                 "CG mode)" if args.pa else f"{kind} apply (CG mode, fused p.Ap)"))),
                          "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src,
                          "frac_of_8TBps_nominal": achieved / 8000.0} if not hexmesh else
                         {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                          "frac": achieved / hbm_peak, "traffic": None,
                          "kernel": f"hex_pa_apply_kernel<{kind}, CG mode> (partial assembly)",
                          "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src} if args.pa else
                         {"bound": "alu", "achieved": achieved_tf, "peak": FP64_PEAK_TFLOPS,
                          "unit": "TFLOP/s", "frac": achieved_tf / FP64_PEAK_TFLOPS, "traffic": None,
                          "kernel": f"hex_apply_kernel<{kind}, CG mode> (Alg. 1, J per Gauss point)",
                          "flops_per_cell": HEX_FLOPS_PER_CELL[kind],
                          "peak_source": "FP64 DFMA microbenchmark x 2 (profiles/r01_microbench_fp64_hbm.txt)"}),
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "cpu_baseline": cpu,
            "cg_info": {k: info[k] for k in ("iterations", "r0_norm", "r_norm", "true_r_norm")},
            "wall_s_timed": wall,
            "extra": extra,
        }
        print(json.dumps(line), flush=True)
    # release the library objects in dependency order (operator -> mesh -> communicator) before
    # the process group goes away, instead of leaving it to interpreter-exit garbage collection
    torch.cuda.synchronize()
    op.close()
    mesh.close()
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()


def cusparse_compare(torch, A, x, y_own, timeit):
    """cuSPARSE SpMV (torch sparse CSR, int32 indices) on the matrix exported from our CSR."""
    try:
        nr, nnz = A.nrows, A.nnz
        rowptr = torch.empty(nr + 1, dtype=torch.int64, device="cuda")
        col = torch.empty(nnz, dtype=torch.int32, device="cuda")
        val = torch.empty(nnz, dtype=torch.float64, device="cuda")
        A.export(rowptr, col, val)
        crow = rowptr.to(torch.int32)
        del rowptr
        M = torch.sparse_csr_tensor(crow, col, val, size=(nr, nr))
        t_cus = timeit(lambda: torch.mv(M, x))
        y3 = torch.mv(M, x)
        out = {"cusparse_spmv_ms": t_cus, "cusparse_gdofs": nr / (t_cus / 1e3) / 1e9,
               "cusparse_gbs": (nnz * 12 + (nr + 1) * 4 + 16 * nr) / (t_cus / 1e3) / 1e9,
               "cusparse_vs_own_max_rel_diff": float((y3 - y_own).abs().max() / y_own.abs().max())}
        del M, crow, col, val, y3
        torch.cuda.empty_cache()
        return out
    except Exception as ex:  # the library leg is a reported baseline, never required
        return {"cusparse_error": str(ex)[:200]}


def csr_compare(fem, torch, kind, args):
    """Matrix-free apply vs assembled CSR SpMV on the same box and operator (Table 1 analogue).
    Elasticity at 384^3 needs 167 GB of CSR, so the comparison uses 256^3."""
    n = args.csr_n if args.csr_n else (256 if kind == "elastic" else 256)
    out = {}
    try:
        mesh = fem.Mesh(n, n, n, 1.0 / n)
        op = fem.Operator(mesh, kind, "dirichlet")
        if args.gll:
            op.set_option("quadrature", 1)
        if kind == "elastic":
            g = I.rng(I.SEED_BASE + 55)
            lam, mu = I.materials(g, n, n, n)
            op.set_material(torch.from_numpy(lam).cuda(), torch.from_numpy(mu).cuda())
            del lam, mu
        t0 = time.perf_counter()
        A = op.csr()
        torch.cuda.synchronize()
        build_s = time.perf_counter() - t0
        x = torch.empty(op.n_global, dtype=torch.float64, device="cuda").uniform_(-1, 1)
        y1 = torch.empty_like(x); y2 = torch.empty_like(x)
        s = torch.cuda.current_stream()

        def timeit(fn, R=10):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(R):
                fn()
            b.record(s)
            torch.cuda.synchronize()
            return a.elapsed_time(b) / R

        t_csr = timeit(lambda: A.apply(x, y1))
        t_mf = timeit(lambda: op.apply(x, y2))
        rel = float((y1 - y2).abs().max() / y2.abs().max())
        # library baseline on the identical matrix: cuSPARSE SpMV through torch's sparse CSR
        # (int32 indices; cuSPARSE rejects the 4e9-nnz 3-DOF 256^3 matrix, so those kinds are
        # compared -- own kernel vs cuSPARSE -- on the largest box with nnz < 2^31, 176^3)
        if A.nnz < 2 ** 31 - 1:
            cus = cusparse_compare(torch, A, x, y1, timeit)
        else:
            cus = {}
            try:
                m = 176
                mesh2 = fem.Mesh(m, m, m, 1.0 / m)
                op2 = fem.Operator(mesh2, kind, "dirichlet")
                if args.gll:
                    op2.set_option("quadrature", 1)
                if kind == "elastic":
                    g2 = I.rng(I.SEED_BASE + 56)
                    l2, m2 = I.materials(g2, m, m, m)
                    op2.set_material(torch.from_numpy(l2).cuda(), torch.from_numpy(m2).cuda())
                A.close()
                A2 = op2.csr()
                x2 = torch.empty(op2.n_global, dtype=torch.float64, device="cuda").uniform_(-1, 1)
                y2b = torch.empty_like(x2)
                t_own2 = timeit(lambda: A2.apply(x2, y2b))
                cus = cusparse_compare(torch, A2, x2, y2b, timeit)
                cus.update({"cusparse_box_cells": [m, m, m], "own_csr_same_box_ms": t_own2,
                            "own_csr_same_box_gdofs": op2.n_global / (t_own2 / 1e3) / 1e9})
                A2.close()
                op2.close()
            except Exception as ex:
                cus = {"cusparse_error": str(ex)[:200]}
        out = {"csr_cells": [n, n, n], "csr_nnz": A.nnz, "csr_bytes": A.bytes,
               "csr_build_s": build_s, "csr_spmv_ms": t_csr,
               "csr_gdofs": op.n_global / (t_csr / 1e3) / 1e9,
               "csr_gbs": (A.bytes + 16 * op.n_global) / (t_csr / 1e3) / 1e9,
               "mf_same_box_ms": t_mf, "mf_same_box_gdofs": op.n_global / (t_mf / 1e3) / 1e9,
               "mf_over_csr": t_csr / t_mf, "mf_vs_csr_max_rel_diff": rel, **cus}
        try:
            A.close()
        except Exception:
            pass
        del A
        torch.cuda.empty_cache()
    except Exception as ex:
        out = {"csr_error": str(ex)}
    return out


def relaunch_multi_gpu(args):
    """--gpus N > 1 outside torchrun: start N ranks (one per GPU) under torch.distributed.run on
    this node, or fail loudly if fewer than N GPUs are visible.  Rank 0's JSON line is the output."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} needs {args.gpus} GPUs; "
                          f"{have} visible", "n_gpus": args.gpus}), flush=True)
        sys.exit(2)
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=24)  # a multiple of the x_defer group (8): steady-state x-update share
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3,
                    help="0-3: BASELINE.json configs[0..3]; 4/5: configs[4] weak scaling (scalar / elasticity)")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-csr", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--csr-n", type=int, default=0)
    ap.add_argument("--e2e-iters", type=int, default=100)
    ap.add_argument("--n", type=int, default=0, help="override cells per direction (debug)")
    ap.add_argument("--peer-halo", action="store_true",
                    help="N > 1: ghost planes read by the apply kernels from the neighbours' memory (CUDA IPC)")
    ap.add_argument("--cgcg", action="store_true",
                    help="Chronopoulos-Gear single-reduction CG (one allreduce of 2 values per iteration)")
    ap.add_argument("--dot", default="fused", choices=["fused", "separate", "atomic"],
                    help="how the fused CG forms p.Ap and r.r (option dot_mode; P:714-728 ablation)")
    ap.add_argument("--gll", action="store_true",
                    help="2x2x2 Gauss-Lobatto quadrature (the CEED BP5/BP6 operators) instead of Gauss")
    ap.add_argument("--x-defer", type=int, default=0, choices=[0, 1, 2, 4, 8],
                    help="fused CG: x updated every m-th iteration from the group's p buffers (0: library default)")
    ap.add_argument("--det", action="store_true",
                    help="general-hex configs (6/7): deterministic scatter (element outputs + node gather)")
    ap.add_argument("--pa", action="store_true",
                    help="general-hex configs (6/7): partial assembly instead of matrix-free")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = dict(I.CONFIGS[args.config])
    if args.n:
        cfg["n"] = (args.n, args.n, args.n)
        cfg["name"] += f"_n{args.n}"
    if args.pa:
        cfg["name"] += "_pa"
    if args.det:
        cfg["name"] += "_det"
    if args.gll:
        cfg["name"] += "_gll"
    if args.cgcg:
        cfg["name"] += "_cgcg"
    if args.dot != "fused":
        cfg["name"] += "_dot-" + args.dot
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, cfg)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_multi_gpu(args)
    else:
        if ws != args.gpus and "WORLD_SIZE" in os.environ:
            print(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}; using WORLD_SIZE", file=sys.stderr)
        run_native(args, cfg)


if __name__ == "__main__":
    main()
