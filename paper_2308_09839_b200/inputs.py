"""Seeded synthetic input generators shared by the tests, bench.py and the oracle legs.

This module holds NO arithmetic of the method (no element matrices, no operator, no CG):
only random numbers and index bookkeeping, so the CUDA path and the CPU oracle can be fed
identical inputs ("Input recipe").

Recipe:
  * seed = 2308_09839 + config index (C1 -> +0, C2 -> +1, ...), numpy PCG64;
  * apply inputs x ~ U(-1, 1) on every DOF;
  * CG right-hand side b ~ U(-1, 1) on interior DOFs, 0 on the 6 box faces (all components);
  * materials (paper P:9 "highly discontinuous (cell-wise) material property fields"):
    E_e = 10**U(0, 2), nu_e ~ U(0.20, 0.35), lambda = E nu / ((1+nu)(1-2nu)), mu = E / (2(1+nu)),
    drawn independently per cell (contrast 100, discontinuous).
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 2308_09839

# BASELINE.json configs (index -> description); sizes are cells per direction.
CONFIGS = {
    0: dict(name="C1_scalar_8", kind="scalar", n=(8, 8, 8), bc=1, cg_iters=50),
    1: dict(name="C2_scalar_256", kind="scalar", n=(256, 256, 256), bc=1, cg_iters=100),
    2: dict(name="C3_vector_256", kind="vector", n=(256, 256, 256), bc=1, cg_iters=100),
    3: dict(name="C4_elastic_384", kind="elastic", n=(384, 384, 384), bc=1, cg_iters=100),
    # BASELINE configs[4], weak scaling: fixed node planes per GPU,
    # nz = planes_per_rank * P - 1 cells -> ~1.25e8 DOF per GPU, ~1e9 DOF at P = 8
    4: dict(name="C5a_scalar_weak", kind="scalar", n=(999, 999, None), planes_per_rank=125, bc=1,
            cg_iters=100),
    5: dict(name="C5b_elastic_weak", kind="elastic", n=(665, 665, None), planes_per_rank=94, bc=1,
            cg_iters=100),
    # NEXT #2 of SURVEY §8(f): general (deformed) hexahedra, Alg. 1 as written -- explicit node
    # map + coordinates, interior nodes jittered by U(-0.2, 0.2) h (non-affine cells)
    6: dict(name="H1_elastic_hex_256", kind="elastic", n=(256, 256, 256), mesh="hex", jitter=0.2, bc=1,
            cg_iters=100),
    7: dict(name="H2_scalar_hex_256", kind="scalar", n=(256, 256, 256), mesh="hex", jitter=0.2, bc=1,
            cg_iters=100),
}


def config_cells(cfg: dict, nranks: int = 1):
    """Cells per direction of a config at P ranks (weak configs grow in z with P)."""
    nx, ny, nz = cfg["n"]
    if nz is None:
        nz = cfg["planes_per_rank"] * nranks - 1
    return nx, ny, nz


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


def ncomp(kind: str) -> int:
    return 1 if kind == "scalar" else 3


def n_nodes(nx: int, ny: int, nz: int) -> int:
    return (nx + 1) * (ny + 1) * (nz + 1)


def boundary_mask(nx: int, ny: int, nz: int) -> np.ndarray:
    """Boolean per node (lexicographic, x fastest): any lattice index at 0 or its maximum."""
    i = np.arange(nx + 1)
    j = np.arange(ny + 1)
    k = np.arange(nz + 1)
    bi = (i == 0) | (i == nx)
    bj = (j == 0) | (j == ny)
    bk = (k == 0) | (k == nz)
    return (bk[:, None, None] | bj[None, :, None] | bi[None, None, :]).reshape(-1)


def uniform_vector(g: np.random.Generator, nx, ny, nz, c, lo=-1.0, hi=1.0) -> np.ndarray:
    return g.uniform(lo, hi, size=n_nodes(nx, ny, nz) * c)


def interior_rhs(g: np.random.Generator, nx, ny, nz, c) -> np.ndarray:
    b = g.uniform(-1.0, 1.0, size=(n_nodes(nx, ny, nz), c))
    b[boundary_mask(nx, ny, nz)] = 0.0
    return b.reshape(-1)


def materials(g: np.random.Generator, nx, ny, nz):
    """Cell-wise discontinuous (lambda, mu), cell-lexicographic e = i + nx (j + ny k)."""
    ne = nx * ny * nz
    E = 10.0 ** g.uniform(0.0, 2.0, size=ne)
    nu = g.uniform(0.20, 0.35, size=ne)
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = E / (2.0 * (1.0 + nu))
    return lam, mu


def lognormal_materials(g: np.random.Generator, nx, ny, nz, lo=-1.0, hi=1.0):
    """Independent lambda, mu = 10**U(lo, hi) (parity-test variant)."""
    ne = nx * ny * nz
    return 10.0 ** g.uniform(lo, hi, size=ne), 10.0 ** g.uniform(lo, hi, size=ne)


# ------------------------------------------------------------------------------------------
# General hexahedral meshes (Alg. 1 as written: explicit node map + nodal coordinates)
# ------------------------------------------------------------------------------------------
VTK_CORNERS = ((0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1))


def hex_box_mesh(nx, ny, nz, h=None, g=None, jitter=0.0, permute=False):
    """Box of nx*ny*nz hexahedra as an explicit (unstructured) mesh.

    Returns coords (n, 3) float64, cells (ne, 8) int32 in VTK corner order and
    dirichlet (n,) uint8 marking the nodes on the 6 box faces.
      jitter  : interior nodes moved by U(-jitter, jitter) * h per coordinate (non-affine
                cells; |jitter| < 0.25 keeps every det J > 0), boundary nodes stay on the box;
      permute : random node labels and random cell order (a genuinely unstructured numbering).
    Index bookkeeping and random numbers only (no arithmetic of the method).
    """
    h = 1.0 / nx if h is None else h
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    coords = np.stack([i.ravel() * h, j.ravel() * h, k.ravel() * h], 1).astype(np.float64)
    bnd = boundary_mask(nx, ny, nz)
    if jitter:
        g = rng(SEED_BASE + 900) if g is None else g
        d = g.uniform(-jitter, jitter, size=coords.shape) * h
        d[bnd] = 0.0
        coords = coords + d
    ck, cj, ci = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ci, cj, ck = ci.ravel(), cj.ravel(), ck.ravel()
    cells = np.stack([(ci + a) + (nx + 1) * ((cj + b) + (ny + 1) * (ck + c)) for a, b, c in VTK_CORNERS],
                     1).astype(np.int64)
    dirichlet = bnd.astype(np.uint8)
    if permute:
        g = rng(SEED_BASE + 901) if g is None else g
        perm = g.permutation(coords.shape[0])  # new label of old node n: perm[n]
        inv = np.empty_like(perm); inv[perm] = np.arange(perm.size)
        coords = coords[inv]
        dirichlet = dirichlet[inv]
        cells = perm[cells]
        cells = cells[g.permutation(cells.shape[0])]
    return coords, cells.astype(np.int32), dirichlet
