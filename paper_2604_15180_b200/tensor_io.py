"""ATN1 tensor files and the `atn attn` input stream.

Thin wrappers over the C-ABI in ``include/adattn_b200.h`` (implemented in
``csrc/io.cu``, restating /root/reference/proj/src/tensor_io.cpp:39-112 and
include/adattn/rng.hpp:10-72):

* ``save_tensor(path, array, dtype)`` / ``load_tensor(path)`` -- magic "ATN1",
  dtype byte (0 = f32, 1 = f64), rank 1..3, little-endian row-major payload,
  atomic temp-file rename; parse errors raise ``RuntimeError`` naming the byte
  offset (the reference's std::runtime_error), bad arguments ``ValueError``.
* ``attn_inputs(seed, n, d, qscale)`` -- Q, K, V, dO exactly as ``atn attn``
  draws them (atn_main.cpp:227-232).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

F32, F64 = 0, 1


def _io_check(rc: int) -> None:
    if rc == _lib.ADATTN_OK:
        return
    msg = _lib.load().adattn_b200_io_last_error().decode()
    if rc == _lib.ADATTN_ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError(msg)


def save_tensor(path: str, values, dtype: int = F64) -> None:
    a = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    dims = (C.c_uint32 * max(a.ndim, 1))(*[int(x) for x in a.shape])
    _io_check(_lib.load().adattn_b200_tensor_save(
        str(path).encode(), int(dtype), int(a.ndim), dims,
        a.ctypes.data_as(C.POINTER(C.c_double))))


def load_tensor(path: str):
    """Returns (values as float64 ndarray of the stored shape, dtype code)."""
    lib = _lib.load()
    dt, rank, cnt = C.c_int(), C.c_int(), C.c_size_t()
    dims = (C.c_uint32 * 3)()
    _io_check(lib.adattn_b200_tensor_load(str(path).encode(), C.byref(dt), C.byref(rank), dims,
                                          None, 0, C.byref(cnt)))
    out = np.empty(cnt.value, dtype=np.float64)
    _io_check(lib.adattn_b200_tensor_load(str(path).encode(), C.byref(dt), C.byref(rank), dims,
                                          out.ctypes.data_as(C.POINTER(C.c_double)), out.size,
                                          C.byref(cnt)))
    return out.reshape([int(dims[i]) for i in range(rank.value)]), int(dt.value)


def attn_inputs(seed: int, n: int, d: int, qscale: float = 1.0):
    """(q, k, v, dout) as float64 [n, d] arrays, atn_main.cpp:227-232's stream."""
    arrs = [np.empty((n, d), dtype=np.float64) for _ in range(4)]
    P = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    _lib.load().adattn_b200_attn_inputs(int(seed) & 0xFFFFFFFFFFFFFFFF, int(n), int(d),
                                        float(qscale), *[P(a) for a in arrs])
    return tuple(arrs)


def xoshiro(seed: int, n_next: int, n_gauss: int):
    nx = np.empty(n_next, dtype=np.uint64)
    gs = np.empty(n_gauss, dtype=np.float64)
    _lib.load().adattn_b200_xoshiro(int(seed), nx.ctypes.data_as(C.POINTER(C.c_uint64)), n_next,
                                    gs.ctypes.data_as(C.POINTER(C.c_double)), n_gauss)
    return nx, gs
