"""Thin Python binding of libfem.so (include/fem.h).  Argument marshalling only: every step of
the hot path runs in the library's CUDA kernels.  There is no CPU fallback: if the shared
library is missing or fails to load, importing this module raises.

Vectors may be torch CUDA tensors (device pointers, zero copy) or numpy / pinned host buffers
(host pointers: the library stages them, which is the end-to-end path measured by bench.py).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

KINDS = {"scalar": 0, "vector": 1, "elastic": 2, "elasticity": 2}
BCS = {"none": 0, "dirichlet": 1}

FEM_OK, FEM_EINVAL, FEM_ENOMEM, FEM_ECUDA, FEM_ENCCL, FEM_EOVERFLOW, FEM_EMATERIAL, \
    FEM_EBREAKDOWN, FEM_ESTATE, FEM_EUNSUPPORTED = range(10)
_NAMES = ["FEM_OK", "FEM_EINVAL", "FEM_ENOMEM", "FEM_ECUDA", "FEM_ENCCL", "FEM_EOVERFLOW",
          "FEM_EMATERIAL", "FEM_EBREAKDOWN", "FEM_ESTATE", "FEM_EUNSUPPORTED"]


class FemError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"{_NAMES[status] if 0 <= status < len(_NAMES) else status}: {msg}")


class CgInfo(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("breakdown_iter", ctypes.c_int32), ("status", ctypes.c_int32),
                ("r0_norm", ctypes.c_double), ("r_norm", ctypes.c_double),
                ("true_r_norm", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# every symbol include/fem.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "fem_last_error", "fem_version", "fem_launch_count", "fem_get_unique_id", "fem_comm_create",
    "fem_comm_create_loopback",
    "fem_comm_destroy", "fem_partition", "fem_apply_ghost", "fem_apply_ghost_padded", "fem_op_link_peers",
    "fem_op_peer_info", "fem_op_open_peers", "fem_mesh_create", "fem_mesh_local", "fem_mesh_destroy",
    "fem_mesh_create_hex", "fem_mesh_info_hex", "fem_op_create",
    "fem_op_ndof", "fem_set_material", "fem_apply", "fem_dot", "fem_cg_solve", "fem_cg_begin",
    "fem_cg_iterate", "fem_cg_end", "fem_set_option", "fem_get_option", "fem_apply_time", "fem_op_destroy",
    "fem_csr_create", "fem_csr_info", "fem_csr_apply", "fem_csr_export", "fem_csr_destroy",
]

_lib = None


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libfem.so (building it in-tree with nvcc if absent).  Raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing:
        _build.build()
    if not os.path.exists(_build.LIB):
        raise ImportError(f"libfem.so not found at {_build.LIB}; run paper_2308_09839_b200.build")
    L = ctypes.CDLL(_build.LIB)
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    P = ctypes.POINTER
    sig = {
        "fem_last_error": ([], ctypes.c_char_p), "fem_version": ([], ctypes.c_char_p),
        "fem_launch_count": ([], i64),
        "fem_get_unique_id": ([vp, i64], ctypes.c_int),
        "fem_comm_create": ([i32, i32, vp, P(vp)], ctypes.c_int),
        "fem_comm_create_loopback": ([i32, P(vp)], ctypes.c_int),
        "fem_comm_destroy": ([vp], None),
        "fem_partition": ([i64, i32, i32, P(i64), P(i64)], ctypes.c_int),
        "fem_apply_ghost": ([vp, vp, vp, vp, vp, vp], ctypes.c_int),
        "fem_apply_ghost_padded": ([vp, vp, vp, vp, vp, vp], ctypes.c_int),
        "fem_op_link_peers": ([vp, vp, vp], ctypes.c_int),
        "fem_op_peer_info": ([vp, vp, i64], ctypes.c_int),
        "fem_op_open_peers": ([vp, vp, vp], ctypes.c_int),
        "fem_mesh_create": ([i64, i64, i64, dbl, vp, P(vp)], ctypes.c_int),
        "fem_mesh_local": ([vp, P(i64), P(i64), P(i64)], ctypes.c_int),
        "fem_mesh_destroy": ([vp], None),
        "fem_mesh_create_hex": ([i64, i64, vp, vp, vp, P(vp)], ctypes.c_int),
        "fem_mesh_info_hex": ([vp, P(i64), P(i64), P(i64)], ctypes.c_int),
        "fem_op_create": ([vp, i32, i32, P(vp)], ctypes.c_int),
        "fem_op_ndof": ([vp, P(i64), P(i64)], ctypes.c_int),
        "fem_set_material": ([vp, vp, vp, i64, i64], ctypes.c_int),
        "fem_apply": ([vp, vp, vp, vp], ctypes.c_int),
        "fem_dot": ([vp, vp, vp, P(dbl), vp], ctypes.c_int),
        "fem_cg_solve": ([vp, vp, vp, dbl, i32, P(CgInfo), vp], ctypes.c_int),
        "fem_cg_begin": ([vp, vp, vp, dbl, i32, vp], ctypes.c_int),
        "fem_cg_iterate": ([vp, i32, vp], ctypes.c_int),
        "fem_cg_end": ([vp, P(CgInfo), vp], ctypes.c_int),
        "fem_set_option": ([vp, ctypes.c_char_p, i64], ctypes.c_int),
        "fem_get_option": ([vp, ctypes.c_char_p, P(i64)], ctypes.c_int),
        "fem_apply_time": ([vp, P(dbl), P(i64)], ctypes.c_int),
        "fem_op_destroy": ([vp], None),
        "fem_csr_create": ([vp, P(vp)], ctypes.c_int),
        "fem_csr_info": ([vp, P(i64), P(i64), P(i64)], ctypes.c_int),
        "fem_csr_apply": ([vp, vp, vp, vp], ctypes.c_int),
        "fem_csr_export": ([vp, vp, vp, vp, vp], ctypes.c_int),
        "fem_csr_destroy": ([vp], None),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(rc: int):
    if rc != FEM_OK:
        raise FemError(rc, load().fem_last_error().decode())


def _numel(a) -> int:
    return int(a.size) if isinstance(a, np.ndarray) else int(a.numel())


def _ptr(a, dtype: str = "float64", n: int | None = None, name: str = "buffer"):
    """Raw pointer of a torch tensor (device or host) or numpy array; checks dtype, contiguity
    and, when `n` is given, the element count (the C ABI receives only the pointer, so a short
    buffer would be over-read / over-written by the library)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if a.dtype != np.dtype(dtype) or not a.flags.c_contiguous:
            raise TypeError(f"numpy arrays must be contiguous {dtype}")
        ptr = a.ctypes.data
    else:
        import torch
        if not isinstance(a, torch.Tensor):
            raise TypeError(f"unsupported buffer type {type(a)}")
        if a.dtype != getattr(torch, dtype) or not a.is_contiguous():
            raise TypeError(f"tensors must be contiguous {dtype}")
        ptr = a.data_ptr()
    if n is not None and _numel(a) != n:
        raise ValueError(f"{name} has {_numel(a)} elements, the operator needs {n}")
    return ptr


def _stream(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def partition(nz: int, nranks: int, rank: int):
    """Slab partition of the nz+1 node planes (pure host call, no GPU needed)."""
    b, e = ctypes.c_int64(), ctypes.c_int64()
    _check(load().fem_partition(nz, nranks, rank, ctypes.byref(b), ctypes.byref(e)))
    return b.value, e.value


def launch_count() -> int:
    return int(load().fem_launch_count())


def unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().fem_get_unique_id(buf, 128))
    return buf.raw


class Comm:
    def __init__(self, nranks: int, rank: int, uid: bytes | None = None):
        self.nranks, self.rank = nranks, rank
        h = ctypes.c_void_p()
        idbuf = ctypes.create_string_buffer(uid, 128) if uid is not None else None
        _check(load().fem_comm_create(nranks, rank, idbuf, ctypes.byref(h)))
        self.h = h

    @classmethod
    def loopback(cls, nranks: int) -> "list[Comm]":
        """`nranks` in-process slab ranks on the current device (fem_comm_create_loopback): drive
        each from its own thread and stream; the library's collectives run as device copies."""
        arr = (ctypes.c_void_p * nranks)()
        _check(load().fem_comm_create_loopback(nranks, arr))
        out = []
        for r in range(nranks):
            c = cls.__new__(cls)
            c.nranks, c.rank, c.h = nranks, r, ctypes.c_void_p(arr[r])
            out.append(c)
        return out

    def close(self):
        if self.h:
            load().fem_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Mesh:
    def __init__(self, nx: int, ny: int, nz: int, h: float, comm: Comm | None = None):
        self.nx, self.ny, self.nz, self.h, self.comm = nx, ny, nz, h, comm
        m = ctypes.c_void_p()
        _check(load().fem_mesh_create(nx, ny, nz, h, comm.h if comm else None, ctypes.byref(m)))
        self.h_ = m
        pb, pe, nl = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(load().fem_mesh_local(m, ctypes.byref(pb), ctypes.byref(pe), ctypes.byref(nl)))
        self.plane_begin, self.plane_end, self.n_local_nodes = pb.value, pe.value, nl.value

    def close(self):
        if self.h_:
            load().fem_mesh_destroy(self.h_)
            self.h_ = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HexMesh:
    """General (deformed) hexahedral mesh: Alg. 1 input -- coordinates (n, 3) float64, node map
    (ne, 8) int32 in VTK corner order, optional Dirichlet flags (n,) uint8 (include/fem.h)."""

    def __init__(self, coords, cells, dirichlet=None):
        if tuple(coords.shape[1:]) != (3,) or coords.ndim != 2:
            raise ValueError(f"coords must have shape (n, 3), got {tuple(coords.shape)}")
        if tuple(cells.shape[1:]) != (8,) or cells.ndim != 2:
            raise ValueError(f"cells must have shape (n_cells, 8), got {tuple(cells.shape)}")
        n, ne = int(coords.shape[0]), int(cells.shape[0])
        m = ctypes.c_void_p()
        _check(load().fem_mesh_create_hex(n, ne, _ptr(coords), _ptr(cells, "int32"),
                                          _ptr(dirichlet, "uint8", n, "dirichlet"), ctypes.byref(m)))
        self.h_ = m
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(load().fem_mesh_info_hex(m, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        self.n_nodes, self.n_cells, self.n_constrained = a.value, b.value, c.value
        self.comm = None
        self.plane_begin, self.plane_end, self.n_local_nodes = 0, 1, self.n_nodes

    def close(self):
        if self.h_:
            load().fem_mesh_destroy(self.h_)
            self.h_ = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Operator:
    def __init__(self, mesh: Mesh, kind: str | int, bc: str | int = "dirichlet"):
        self.mesh = mesh
        self.kind = KINDS[kind] if isinstance(kind, str) else int(kind)
        self.bc = BCS[bc] if isinstance(bc, str) else int(bc)
        self.comps = 1 if self.kind == 0 else 3
        o = ctypes.c_void_p()
        _check(load().fem_op_create(mesh.h_, self.kind, self.bc, ctypes.byref(o)))
        self.h = o
        nl, ng = ctypes.c_int64(), ctypes.c_int64()
        _check(load().fem_op_ndof(o, ctypes.byref(nl), ctypes.byref(ng)))
        self.n_local, self.n_global = nl.value, ng.value

    def _plane_dofs(self) -> int | None:
        if isinstance(self.mesh, HexMesh):  # no node planes (the library rejects ghost applies)
            return None
        return (self.mesh.nx + 1) * (self.mesh.ny + 1) * self.comps

    # -- material ---------------------------------------------------------------------------
    def set_material(self, lam, mu, layer_begin: int = 0, n_layers: int | None = None):
        if isinstance(self.mesh, HexMesh):
            if n_layers is None:
                n_layers = 1
            cnt = self.mesh.n_cells
        else:
            if n_layers is None:
                n_layers = self.mesh.nz - layer_begin
            cnt = self.mesh.nx * self.mesh.ny * n_layers
        _check(load().fem_set_material(self.h, _ptr(lam, n=cnt, name="lambda"), _ptr(mu, n=cnt, name="mu"),
                                       layer_begin, n_layers))

    # -- operator ---------------------------------------------------------------------------
    def apply(self, x, y=None, stream=None):
        if y is None:
            if isinstance(x, np.ndarray):
                y = np.empty_like(x)
            else:
                import torch
                y = torch.empty_like(x)
        n = self.n_local
        _check(load().fem_apply(self.h, _ptr(x, n=n, name="x"), _ptr(y, n=n, name="y"), _stream(stream)))
        return y

    def apply_ghost(self, x, ghost_lo, ghost_hi, y=None, stream=None):
        """y = A_c x with caller-provided ghost planes (single-process slab tests)."""
        if y is None:
            import torch
            y = torch.empty_like(x)
        n, pd = self.n_local, self._plane_dofs()
        _check(load().fem_apply_ghost(self.h, _ptr(x, n=n, name="x"), _ptr(ghost_lo, n=pd, name="ghost_lo"),
                                      _ptr(ghost_hi, n=pd, name="ghost_hi"), _ptr(y, n=n, name="y"),
                                      _stream(stream)))
        return y

    def link_peers(self, lo: "Operator | None", hi: "Operator | None"):
        """Single-process loopback of the peer halo (ghost planes from the neighbours' buffers).
        The neighbours' device buffers are read by this operator's kernels: keep them alive."""
        _check(load().fem_op_link_peers(self.h, lo.h if lo else None, hi.h if hi else None))
        self._peers = (lo, hi)

    def peer_info(self) -> bytes:
        buf = ctypes.create_string_buffer(320)
        _check(load().fem_op_peer_info(self.h, buf, 320))
        return buf.raw

    def open_peers(self, lo_info: bytes | None, hi_info: bytes | None):
        lo = ctypes.create_string_buffer(lo_info, 320) if lo_info else None
        hi = ctypes.create_string_buffer(hi_info, 320) if hi_info else None
        _check(load().fem_op_open_peers(self.h, lo, hi))

    def apply_ghost_padded(self, x, ghost_lo, ghost_hi, y=None, stream=None):
        """As apply_ghost, through the CG-internal padded layout and its TMA tensor maps."""
        if y is None:
            import torch
            y = torch.empty_like(x)
        n, pd = self.n_local, self._plane_dofs()
        _check(load().fem_apply_ghost_padded(self.h, _ptr(x, n=n, name="x"), _ptr(ghost_lo, n=pd, name="ghost_lo"),
                                             _ptr(ghost_hi, n=pd, name="ghost_hi"), _ptr(y, n=n, name="y"),
                                             _stream(stream)))
        return y

    def dot(self, a, b, stream=None) -> float:
        out = ctypes.c_double()
        n = self.n_local
        _check(load().fem_dot(self.h, _ptr(a, n=n, name="a"), _ptr(b, n=n, name="b"), ctypes.byref(out),
                              _stream(stream)))
        return out.value

    def cg_solve(self, b, x, tol: float = 0.0, maxit: int = 100, stream=None, check=True):
        info = CgInfo()
        n = self.n_local
        rc = load().fem_cg_solve(self.h, _ptr(b, n=n, name="b"), _ptr(x, n=n, name="x"), float(tol), int(maxit),
                                 ctypes.byref(info), _stream(stream))
        if check and rc not in (FEM_OK, FEM_EBREAKDOWN):
            _check(rc)
        d = info.as_dict()
        d["rc"] = rc
        return d

    def cg_begin(self, b, x, tol: float = 0.0, maxit: int = 1 << 30, stream=None):
        n = self.n_local
        _check(load().fem_cg_begin(self.h, _ptr(b, n=n, name="b"), _ptr(x, n=n, name="x"), float(tol), int(maxit),
                                   _stream(stream)))

    def cg_iterate(self, iters: int, stream=None):
        _check(load().fem_cg_iterate(self.h, int(iters), _stream(stream)))

    def cg_end(self, stream=None):
        info = CgInfo()
        rc = load().fem_cg_end(self.h, ctypes.byref(info), _stream(stream))
        if rc not in (FEM_OK, FEM_EBREAKDOWN):
            _check(rc)
        d = info.as_dict()
        d["rc"] = rc
        return d

    def set_option(self, key: str, value: int):
        _check(load().fem_set_option(self.h, key.encode(), int(value)))

    def get_option(self, key: str) -> int:
        v = ctypes.c_int64()
        _check(load().fem_get_option(self.h, key.encode(), ctypes.byref(v)))
        return v.value

    def apply_time(self):
        ms, n = ctypes.c_double(), ctypes.c_int64()
        _check(load().fem_apply_time(self.h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def csr(self) -> "Csr":
        return Csr(self)

    def close(self):
        if self.h:
            load().fem_op_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Csr:
    def __init__(self, op: Operator):
        c = ctypes.c_void_p()
        _check(load().fem_csr_create(op.h, ctypes.byref(c)))
        self.h = c
        nr, nnz, nb = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(load().fem_csr_info(c, ctypes.byref(nr), ctypes.byref(nnz), ctypes.byref(nb)))
        self.nrows, self.nnz, self.bytes = nr.value, nnz.value, nb.value

    def apply(self, x, y=None, stream=None):
        if y is None:
            import torch
            y = torch.empty_like(x)
        n = self.nrows
        _check(load().fem_csr_apply(self.h, _ptr(x, n=n, name="x"), _ptr(y, n=n, name="y"), _stream(stream)))
        return y

    def export(self, rowptr, col, val, stream=None):
        """Copy rowptr (int64), col (int32), val (float64) into the given buffers."""
        _check(load().fem_csr_export(self.h, _ptr(rowptr, "int64", self.nrows + 1, "rowptr"),
                                     _ptr(col, "int32", self.nnz, "col"), _ptr(val, n=self.nnz, name="val"),
                                     _stream(stream)))

    def close(self):
        if self.h:
            load().fem_csr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
