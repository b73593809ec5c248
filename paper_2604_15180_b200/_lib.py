"""ctypes binding of libadattn_b200.so (include/adattn_b200.h).

The library is built in-tree by ``paper_2604_15180_b200/Makefile`` (see
``__graft_entry__.build``).  There is no fallback: if the shared object is
missing or fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libadattn_b200.so")

ADATTN_OK = 0
ADATTN_ERR_INVALID = 1
ADATTN_ERR_UNSUPPORTED = 4
ADATTN_ERR_CUDA = 5
ADATTN_ERR_WORKSPACE = 6
ADATTN_ERR_IO = 7

F32, BF16, F64 = 0, 1, 2
PATH_AUTO, PATH_EXACT, PATH_TC = 0, 1, 2

# every symbol include/adattn_b200.h declares
EXPORTS = (
    "adattn_b200_abi_version", "adattn_b200_last_error", "adattn_b200_validate",
    "adattn_b200_resolved_path", "adattn_b200_forward_workspace",
    "adattn_b200_backward_workspace", "adattn_b200_forward", "adattn_b200_compute_delta",
    "adattn_b200_backward", "adattn_b200_stats", "adattn_b200_mask_sparsity",
    "adattn_b200_run_host",
    "adattn_b200_launch_count", "adattn_b200_profile_enable", "adattn_b200_profile_read",
    "adattn_b200_tensor_save", "adattn_b200_tensor_load", "adattn_b200_io_last_error",
    "adattn_b200_attn_inputs", "adattn_b200_xoshiro", "adattn_b200_entmax_rows",
    "adattn_b200_block_lists", "adattn_b200_forward_timed", "adattn_b200_forward_ex",
    "adattn_b200_backward_ex", "adattn_b200_delta_aux_bytes",
)


class Problem(C.Structure):
    _fields_ = [
        ("batch", C.c_int32), ("heads", C.c_int32),
        ("n", C.c_int32), ("m", C.c_int32), ("d", C.c_int32), ("dv", C.c_int32),
        ("alpha", C.c_double), ("scale", C.c_double),
        ("causal", C.c_int32), ("block_r", C.c_int32), ("block_c", C.c_int32),
        ("bins", C.c_int32), ("refine_iters", C.c_int32), ("refine_tol", C.c_double),
        ("in_dtype", C.c_int32), ("out_dtype", C.c_int32), ("path", C.c_int32),
        ("reserved", C.c_int32),
    ]


class ForwardExtras(C.Structure):
    _fields_ = [("phase_ms", C.POINTER(C.c_double)), ("tau_h", C.c_void_p),
                ("block_cnt", C.c_void_p), ("block_cols", C.c_void_p),
                ("delta_aux", C.c_void_p)]


class BackwardExtras(C.Structure):
    _fields_ = [("block_cnt", C.c_void_p), ("block_cols", C.c_void_p),
                ("delta_aux", C.c_void_p)]


class Stats(C.Structure):
    _fields_ = [("block_sparsity", C.c_double), ("blocks_visited_fwd", C.c_uint64),
                ("blocks_visited_bwd", C.c_uint64), ("flushes", C.c_uint64),
                ("addressable_blocks", C.c_uint64), ("active_blocks", C.c_uint64)]


class RowsProblem(C.Structure):
    _fields_ = [("rows", C.c_int64), ("n", C.c_int32), ("in_dtype", C.c_int32),
                ("alpha", C.c_double), ("bins", C.c_int32), ("max_iters", C.c_int32),
                ("tol", C.c_double), ("method", C.c_int32), ("trace_len", C.c_int32)]


ROWS_HISTOGRAM_HYBRID, ROWS_HYBRID, ROWS_BISECTION = 0, 1, 2


class AdattnError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


_lock = threading.Lock()
_lib = None


def load() -> C.CDLL:
    """Load the in-tree shared object; raise loudly when it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(no CPU fallback exists)")
        lib = C.CDLL(LIB_PATH)
        vp, P, S = C.c_void_p, C.POINTER(Problem), C.POINTER(Stats)
        lib.adattn_b200_abi_version.restype = C.c_int
        lib.adattn_b200_last_error.restype = C.c_char_p
        lib.adattn_b200_validate.argtypes = [P]
        lib.adattn_b200_resolved_path.argtypes = [P]
        lib.adattn_b200_forward_workspace.argtypes = [P]
        lib.adattn_b200_forward_workspace.restype = C.c_size_t
        lib.adattn_b200_backward_workspace.argtypes = [P]
        lib.adattn_b200_backward_workspace.restype = C.c_size_t
        lib.adattn_b200_delta_aux_bytes.argtypes = [P]
        lib.adattn_b200_delta_aux_bytes.restype = C.c_size_t
        lib.adattn_b200_forward.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp]
        lib.adattn_b200_forward_timed.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                                  C.c_size_t, vp, C.POINTER(C.c_double)]
        lib.adattn_b200_forward_ex.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                               C.c_size_t, vp, C.POINTER(ForwardExtras)]
        lib.adattn_b200_compute_delta.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                                  C.c_size_t, vp]
        lib.adattn_b200_backward.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                             C.c_size_t, vp]
        lib.adattn_b200_backward_ex.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                                vp, C.c_size_t, vp, C.POINTER(BackwardExtras)]
        lib.adattn_b200_stats.argtypes = [P, vp, S, vp]
        lib.adattn_b200_mask_sparsity.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                                  S, vp]
        lib.adattn_b200_block_lists.argtypes = [P, vp, vp, vp, vp, vp, vp]
        lib.adattn_b200_run_host.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, S]
        lib.adattn_b200_launch_count.restype = C.c_uint64
        lib.adattn_b200_profile_enable.argtypes = [C.c_int]
        lib.adattn_b200_profile_enable.restype = None
        lib.adattn_b200_profile_read.argtypes = [C.c_char_p, C.c_size_t,
                                                 C.POINTER(C.c_double), C.c_int]
        dp, u32p = C.POINTER(C.c_double), C.POINTER(C.c_uint32)
        lib.adattn_b200_tensor_save.argtypes = [C.c_char_p, C.c_int, C.c_int, u32p, dp]
        lib.adattn_b200_tensor_load.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                                u32p, dp, C.c_size_t, C.POINTER(C.c_size_t)]
        lib.adattn_b200_io_last_error.restype = C.c_char_p
        lib.adattn_b200_attn_inputs.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_double,
                                                dp, dp, dp, dp]
        lib.adattn_b200_attn_inputs.restype = None
        lib.adattn_b200_xoshiro.argtypes = [C.c_uint64, C.POINTER(C.c_uint64), C.c_size_t, dp,
                                            C.c_size_t]
        lib.adattn_b200_xoshiro.restype = None
        lib.adattn_b200_entmax_rows.argtypes = [C.POINTER(RowsProblem), vp, vp, vp, vp, vp, vp,
                                                vp, vp, vp]
        if lib.adattn_b200_abi_version() != 2:
            raise RuntimeError("libadattn_b200.so ABI mismatch")
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == ADATTN_OK:
        return
    msg = load().adattn_b200_last_error().decode()
    if rc == ADATTN_ERR_INVALID:
        raise ValueError(msg)  # the reference's std::invalid_argument
    if rc == ADATTN_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise AdattnError(rc, msg)


def profile_enable(on: bool = True) -> None:
    load().adattn_b200_profile_enable(1 if on else 0)


def profile_read(max_n: int = 4096):
    """[(kernel name, ms)] of the launches recorded since the last read."""
    lib = load()
    names = C.create_string_buffer(64 * max_n)
    ms = (C.c_double * max_n)()
    n = lib.adattn_b200_profile_read(names, len(names), ms, max_n)
    keys = names.value.decode().split("\n")[:n]
    return list(zip(keys, [ms[i] for i in range(n)]))
