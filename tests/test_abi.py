"""The C-ABI library loads, exports every symbol include/fem.h declares, and validates its
arguments (calls below never reach a kernel, so they run without a GPU)."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

from paper_2308_09839_b200 import build as B
from paper_2308_09839_b200 import fem as F

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "fem.h")


@pytest.fixture(scope="module")
def lib():
    B.build()
    return F.load()


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fem_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(F.EXPORTS) == names


def test_version_and_counters(lib):
    assert b"sm_100a" in lib.fem_version()
    assert lib.fem_launch_count() >= 0
    assert lib.fem_last_error() is not None


def _status(rc):
    return F._NAMES[rc]


def test_mesh_validation(lib):
    m = ctypes.c_void_p()
    assert _status(lib.fem_mesh_create(0, 4, 4, 0.1, None, ctypes.byref(m))) == "FEM_EINVAL"
    assert b"dims" in lib.fem_last_error()
    assert _status(lib.fem_mesh_create(4, 4, 4, -1.0, None, ctypes.byref(m))) == "FEM_EINVAL"
    assert _status(lib.fem_mesh_create(4, 4, 4, float("nan"), None, ctypes.byref(m))) == "FEM_EINVAL"
    assert _status(lib.fem_mesh_create(4, 4, 4, float("inf"), None, ctypes.byref(m))) == "FEM_EINVAL"
    # 2^32 node limit: 2048^3 cells -> 2049^3 > 2^32 nodes
    assert _status(lib.fem_mesh_create(2048, 2048, 2048, 1.0, None, ctypes.byref(m))) == "FEM_EOVERFLOW"
    assert _status(lib.fem_mesh_create(4, 4, 4, 1.0, None, None)) == "FEM_EINVAL"


def test_handle_validation(lib):
    o = ctypes.c_void_p()
    assert _status(lib.fem_op_create(None, 0, 0, ctypes.byref(o))) == "FEM_EINVAL"
    assert _status(lib.fem_apply(None, None, None, None)) == "FEM_EINVAL"
    d = ctypes.c_double()
    assert _status(lib.fem_dot(None, None, None, ctypes.byref(d), None)) == "FEM_EINVAL"
    assert _status(lib.fem_cg_solve(None, None, None, 0.0, 1, None, None)) == "FEM_EINVAL"
    assert _status(lib.fem_set_option(None, b"use_graph", 1)) == "FEM_EINVAL"
    assert _status(lib.fem_comm_create(0, 0, None, ctypes.byref(ctypes.c_void_p()))) == "FEM_EINVAL"
    assert _status(lib.fem_comm_create(2, 2, None, ctypes.byref(ctypes.c_void_p()))) == "FEM_EINVAL"
    assert _status(lib.fem_get_unique_id(None, 128)) == "FEM_EINVAL"
    assert _status(lib.fem_csr_create(None, ctypes.byref(ctypes.c_void_p()))) == "FEM_EINVAL"
    # destroy functions accept NULL
    lib.fem_op_destroy(None); lib.fem_mesh_destroy(None); lib.fem_comm_destroy(None)
    lib.fem_csr_destroy(None)


def test_binding_has_no_cpu_fallback():
    """The product binding must not import the oracle or any CPU implementation."""
    pkg = os.path.dirname(F.__file__)
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in src.replace("oracle/", "").lower() or fn == "inputs.py", fn


def test_binding_checks_buffer_lengths():
    """The ABI receives bare pointers: the binding rejects buffers of the wrong length (a short
    y would be written past its end, a short x over-read)."""
    import numpy as np
    import pytest
    a = np.zeros(4)
    assert F._ptr(a, n=4) == a.ctypes.data
    with pytest.raises(ValueError):
        F._ptr(np.zeros(3), n=4, name="x")
    with pytest.raises(ValueError):
        F._ptr(np.zeros(5), n=4, name="x")
    with pytest.raises(TypeError):
        F._ptr(np.zeros(4, dtype=np.float32), n=4)
    assert _status(F.load().fem_comm_create_loopback(0, None)) == "FEM_EINVAL"
