"""Python loader for the CPU oracle (oracle/fem_oracle.c).

TEST INFRASTRUCTURE ONLY. Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module. The product path
(``paper_2308_09839_b200``) never imports it and shares no code with it.

Every wrapper below forwards to the C function of the same name; the C file cites the
paper passage each one follows (Eq. 4-6, Table 4).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "fem_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

SCALAR, VECTOR, ELASTIC = 0, 1, 2
BC_NONE, BC_DIRICHLET = 0, 1
_KIND = {"scalar": SCALAR, "vector": VECTOR, "elastic": ELASTIC, "elasticity": ELASTIC}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, OpenMP over colour classes)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c11",
               "-Wall", "-Wno-unused-function", "-o", LIB, SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        d = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        L.orc_apply.argtypes = [ctypes.c_int, ctypes.c_int, i64, i64, i64, ctypes.c_double, d, d, d,
                                d, ctypes.c_int]
        L.orc_apply.restype = ctypes.c_int
        L.orc_assemble_dense.argtypes = [ctypes.c_int, ctypes.c_int, i64, i64, i64, ctypes.c_double,
                                         d, d, d]
        L.orc_assemble_dense.restype = ctypes.c_int
        L.orc_element_matrix.argtypes = [ctypes.c_int, d, ctypes.c_double, ctypes.c_double, d]
        L.orc_element_matrix.restype = ctypes.c_int
        L.orc_reference_element.argtypes = [d, d, d, d]
        L.orc_reference_element.restype = None
        L.orc_basis_gradients.argtypes = [d, d]
        L.orc_basis_gradients.restype = None
        L.orc_basis_values.argtypes = [d, d]
        L.orc_basis_values.restype = None
        L.orc_dot.argtypes = [i64, d, d]
        L.orc_dot.restype = ctypes.c_double
        L.orc_cg.argtypes = [ctypes.c_int, ctypes.c_int, i64, i64, i64, ctypes.c_double, d, d, d, d,
                             ctypes.c_double, ctypes.c_int, ctypes.POINTER(CgInfoC), d, ctypes.c_int]
        L.orc_cg.restype = ctypes.c_int
        L.orc_apply_nodes.argtypes = [ctypes.c_int, ctypes.c_int, i64, i64, i64, ctypes.c_double,
                                      d, d, d, ctypes.POINTER(ctypes.c_int64), i64, d, ctypes.c_int]
        L.orc_apply_nodes.restype = ctypes.c_int
        u8p = ctypes.POINTER(ctypes.c_uint8); i32p = ctypes.POINTER(ctypes.c_int32)
        L.orc_apply_hex.argtypes = [ctypes.c_int, i64, i64, d, i32p, u8p, d, d, d, d, ctypes.c_int]
        L.orc_apply_hex.restype = ctypes.c_int
        L.orc_cg_hex.argtypes = [ctypes.c_int, i64, i64, d, i32p, u8p, d, d, d, d, ctypes.c_double,
                                 ctypes.c_int, ctypes.POINTER(CgInfoC), d, ctypes.c_int]
        L.orc_cg_hex.restype = ctypes.c_int
        L.orc_set_quadrature.argtypes = [ctypes.c_int]
        L.orc_set_quadrature.restype = ctypes.c_int
        L.orc_max_threads.argtypes = []
        L.orc_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


class CgInfoC(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("converged", ctypes.c_int),
                ("breakdown_iter", ctypes.c_int), ("status", ctypes.c_int),
                ("r0_norm", ctypes.c_double), ("r_norm", ctypes.c_double),
                ("true_r_norm", ctypes.c_double)]


@dataclass
class CgResult:
    x: np.ndarray
    iterations: int
    converged: bool
    breakdown_iter: int
    status: int
    r0_norm: float
    r_norm: float
    true_r_norm: float
    res_hist: np.ndarray


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _kind(kind):
    return _KIND[kind] if isinstance(kind, str) else int(kind)


def ncomp(kind) -> int:
    return 1 if _kind(kind) == SCALAR else 3


def reference_element():
    xq = np.zeros((8, 3)); wq = np.zeros(8); dphi = np.zeros((8, 8, 3)); phi = np.zeros((8, 8))
    lib().orc_reference_element(_p(xq), _p(wq), _p(dphi), _p(phi))
    return xq, wq, dphi, phi


def basis_gradients(xi):
    xi = np.ascontiguousarray(xi, dtype=np.float64); out = np.zeros((8, 3))
    lib().orc_basis_gradients(_p(xi), _p(out))
    return out


def basis_values(xi):
    xi = np.ascontiguousarray(xi, dtype=np.float64); out = np.zeros(8)
    lib().orc_basis_values(_p(xi), _p(out))
    return out


def element_matrix(kind, X, lam=0.0, mu=0.0):
    k = _kind(kind); c = 1 if k == SCALAR else 3
    X = np.ascontiguousarray(X, dtype=np.float64).reshape(8, 3)
    Ae = np.zeros((8 * c, 8 * c))
    rc = lib().orc_element_matrix(k, _p(X), float(lam), float(mu), _p(Ae))
    if rc:
        raise ValueError(f"orc_element_matrix failed: {rc}")
    return Ae


def _mat(kind, nx, ny, nz, lam, mu):
    if _kind(kind) != ELASTIC:
        return None, None
    ne = nx * ny * nz
    lam = np.ascontiguousarray(np.broadcast_to(np.asarray(lam, dtype=np.float64), (ne,)))
    mu = np.ascontiguousarray(np.broadcast_to(np.asarray(mu, dtype=np.float64), (ne,)))
    return lam, mu


def apply(kind, bc, nx, ny, nz, h, x, lam=None, mu=None, nthreads=0):
    """y = A_c x (oracle). x: float64 array of length c*(nx+1)(ny+1)(nz+1)."""
    k = _kind(kind)
    lam, mu = _mat(k, nx, ny, nz, lam, mu)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    rc = lib().orc_apply(k, int(bc), nx, ny, nz, float(h), _p(lam), _p(mu), _p(x), _p(y),
                         int(nthreads))
    if rc:
        raise ValueError(f"orc_apply failed: {rc}")
    return y


def apply_nodes(kind, bc, nx, ny, nz, h, x, nodes, lam=None, mu=None, nthreads=0):
    """(A_c x) at the given node ids only: array (len(nodes), c)."""
    k = _kind(kind); c = 1 if k == SCALAR else 3
    lam, mu = _mat(k, nx, ny, nz, lam, mu)
    x = np.ascontiguousarray(x, dtype=np.float64)
    nodes = np.ascontiguousarray(nodes, dtype=np.int64)
    out = np.empty((nodes.size, c))
    rc = lib().orc_apply_nodes(k, int(bc), nx, ny, nz, float(h), _p(lam), _p(mu), _p(x),
                               nodes.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), nodes.size,
                               _p(out), int(nthreads))
    if rc:
        raise ValueError(f"orc_apply_nodes failed: {rc}")
    return out


def assemble_dense(kind, bc, nx, ny, nz, h, lam=None, mu=None):
    k = _kind(kind); c = 1 if k == SCALAR else 3
    lam, mu = _mat(k, nx, ny, nz, lam, mu)
    n = (nx + 1) * (ny + 1) * (nz + 1) * c
    A = np.zeros((n, n))
    rc = lib().orc_assemble_dense(k, int(bc), nx, ny, nz, float(h), _p(lam), _p(mu), _p(A))
    if rc:
        raise ValueError(f"orc_assemble_dense failed: {rc}")
    return A


def dot(a, b) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64); b = np.ascontiguousarray(b, dtype=np.float64)
    return lib().orc_dot(a.size, _p(a), _p(b))


def cg(kind, bc, nx, ny, nz, h, b, x0=None, tol=0.0, maxit=50, lam=None, mu=None, nthreads=0):
    k = _kind(kind)
    lam, mu = _mat(k, nx, ny, nz, lam, mu)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    info = CgInfoC()
    hist = np.full(maxit + 1, np.nan)
    rc = lib().orc_cg(k, int(bc), nx, ny, nz, float(h), _p(lam), _p(mu), _p(b), _p(x),
                      float(tol), int(maxit), ctypes.byref(info), _p(hist), int(nthreads))
    if rc not in (0, 3):
        raise ValueError(f"orc_cg failed: {rc}")
    return CgResult(x=x, iterations=info.iterations, converged=bool(info.converged),
                    breakdown_iter=info.breakdown_iter, status=info.status, r0_norm=info.r0_norm,
                    r_norm=info.r_norm, true_r_norm=info.true_r_norm,
                    res_hist=hist[: info.iterations + 1])


def _hex_args(kind, coords, cells, dirichlet, lam, mu):
    k = _kind(kind)
    coords = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, 3)
    cells = np.ascontiguousarray(cells, dtype=np.int32).reshape(-1, 8)
    dp = None
    if dirichlet is not None:
        dirichlet = np.ascontiguousarray(dirichlet, dtype=np.uint8).reshape(-1)
        dp = dirichlet.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    if k == ELASTIC:
        ne = cells.shape[0]
        lam = np.ascontiguousarray(np.broadcast_to(np.asarray(lam, dtype=np.float64), (ne,)))
        mu = np.ascontiguousarray(np.broadcast_to(np.asarray(mu, dtype=np.float64), (ne,)))
    else:
        lam = mu = None
    keep = (coords, cells, dirichlet, lam, mu)
    return k, keep, dp


def apply_hex(kind, coords, cells, x, dirichlet=None, lam=None, mu=None, nthreads=0):
    """y = A_c x on a general hexahedral mesh (Alg. 1 as written): coords (n, 3), cells (ne, 8)
    int32 in VTK corner order, dirichlet (n,) flags or None."""
    k, (co, ce, di, la, m), dp = _hex_args(kind, coords, cells, dirichlet, lam, mu)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    rc = lib().orc_apply_hex(k, co.shape[0], ce.shape[0], _p(co),
                             ce.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), dp, _p(la), _p(m),
                             _p(x), _p(y), int(nthreads))
    if rc:
        raise ValueError(f"orc_apply_hex failed: {rc}")
    return y


def cg_hex(kind, coords, cells, b, dirichlet=None, x0=None, tol=0.0, maxit=50, lam=None, mu=None,
           nthreads=0):
    k, (co, ce, di, la, m), dp = _hex_args(kind, coords, cells, dirichlet, lam, mu)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    info = CgInfoC()
    hist = np.full(maxit + 1, np.nan)
    rc = lib().orc_cg_hex(k, co.shape[0], ce.shape[0], _p(co),
                          ce.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), dp, _p(la), _p(m),
                          _p(b), _p(x), float(tol), int(maxit), ctypes.byref(info), _p(hist),
                          int(nthreads))
    if rc not in (0, 3):
        raise ValueError(f"orc_cg_hex failed: {rc}")
    return CgResult(x=x, iterations=info.iterations, converged=bool(info.converged),
                    breakdown_iter=info.breakdown_iter, status=info.status, r0_norm=info.r0_norm,
                    r_norm=info.r_norm, true_r_norm=info.true_r_norm,
                    res_hist=hist[: info.iterations + 1])


QUAD = {"gauss": 0, "gll": 1}


class quadrature:
    """Context manager selecting the oracle's quadrature rule ("gauss" default, "gll")."""

    def __init__(self, rule: str):
        self.rule = QUAD[rule]

    def __enter__(self):
        self.old = lib().orc_set_quadrature(self.rule)
        return self

    def __exit__(self, *exc):
        lib().orc_set_quadrature(self.old)
        return False


def max_threads() -> int:
    return lib().orc_max_threads()
