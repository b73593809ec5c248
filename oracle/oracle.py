"""oracle.py -- TEST INFRASTRUCTURE ONLY (the CPU checker, never the product).

ctypes binding over two CPU libraries with identical entry points:

* ``liboracle.so``          -- plain-C restatement (adattn_oracle.c), kind "port"
* ``_ref/libadattn_ref.so`` -- the reference itself, compiled from its own
  sources under /root/reference by oracle/Makefile, kind "reference"

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module.  The product package (``paper_2604_15180_b200``) never
does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libadattn_ref.so")


class OrcParams(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("m", C.c_int32), ("d", C.c_int32), ("dv", C.c_int32),
        ("alpha", C.c_double), ("scale", C.c_double),
        ("causal", C.c_int32), ("block_r", C.c_int32), ("block_c", C.c_int32),
        ("bins", C.c_int32), ("refine_iters", C.c_int32), ("refine_tol", C.c_double),
    ]


class OrcStats(C.Structure):
    _fields_ = [("block_sparsity", C.c_double), ("blocks_visited_fwd", C.c_uint64),
                ("blocks_visited_bwd", C.c_uint64), ("flushes", C.c_uint64)]


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


_DP = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_U32P = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_I32P = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_U64P = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


def _build_if_missing(path: str) -> None:
    if os.path.exists(path):
        return
    import subprocess
    subprocess.run(["make", "-C", HERE, "-s"], check=True)
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} was not built (is /root/reference present?)")


@dataclass
class Problem:
    """Mirror of AttentionProblem (attention.hpp:24-36)."""
    q: np.ndarray
    k: np.ndarray
    v: np.ndarray
    alpha: float = 1.5
    scale: float = 0.0
    causal: bool = False
    block_r: int = 64
    block_c: int = 64
    bins: int = 8
    refine_iters: int = 2
    refine_tol: float = 1e-6

    def params(self) -> OrcParams:
        return OrcParams(self.q.shape[0], self.k.shape[0], self.q.shape[1], self.v.shape[1],
                         float(self.alpha), float(self.scale), int(bool(self.causal)),
                         int(self.block_r), int(self.block_c), int(self.bins),
                         int(self.refine_iters), float(self.refine_tol))

    @property
    def t_r(self) -> int:
        return (self.q.shape[0] + self.block_r - 1) // self.block_r if self.block_r > 0 else 1

    @property
    def t_c(self) -> int:
        return (self.k.shape[0] + self.block_c - 1) // self.block_c if self.block_c > 0 else 1


class Oracle:
    def __init__(self, kind: str = "port"):
        if kind not in ("port", "reference"):
            raise ValueError(kind)
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        _build_if_missing(path)
        self.lib = C.CDLL(path)
        pre = "orc_" if kind == "port" else "ref_"
        self._p = pre
        L = self.lib
        P = C.POINTER(OrcParams)
        self._fwd = getattr(L, pre + "forward")
        self._fwd.argtypes = [P, _DP, _DP, _DP, C.c_int, _DP, _DP, _DP, _U32P, _I32P,
                              C.POINTER(OrcStats)]
        self._fwd.restype = C.c_int
        self._dense = getattr(L, pre + "dense_reference")
        self._dense.argtypes = [P, _DP, _DP, _DP, _DP, _DP, _DP, _U32P, C.POINTER(OrcStats)]
        self._dense.restype = C.c_int
        self._delta = getattr(L, pre + "compute_delta")
        self._delta.argtypes = [P, _DP, _DP, _DP, _DP, _DP, _U32P, _DP, C.c_int, _DP]
        self._delta.restype = C.c_int
        self._bwd = getattr(L, pre + "backward")
        self._bwd.argtypes = [P, _DP, _DP, _DP, _DP, _DP, _U32P, _DP, C.c_int, _DP, _DP, _DP,
                              _DP, _U64P]
        self._bwd.restype = C.c_int
        self._bs = getattr(L, pre + "block_sparsity")
        self._bs.argtypes = [_U32P, C.c_int, C.c_int, C.c_int]
        self._bs.restype = C.c_double
        self._sh = getattr(L, pre + "solve_histogram")
        self._sh.argtypes = [_U32P, C.c_int, C.c_double, C.POINTER(C.c_double),
                             C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        self._sh.restype = C.c_int
        self._fe = getattr(L, pre + "f_eval")
        self._fe.argtypes = [_DP, C.c_int, C.c_double, C.c_double, C.POINTER(C.c_double),
                             C.POINTER(C.c_double), C.POINTER(C.c_double)]
        self._fe.restype = None
        self._gf = getattr(L, pre + "gaussian_fill")
        self._gf.argtypes = [C.c_uint64, C.c_double, _DP, C.c_size_t]
        self._gf.restype = None
        self._xn = getattr(L, pre + "xoshiro_next")
        self._xn.argtypes = [C.c_uint64, _U64P, C.c_size_t]
        self._xn.restype = None
        self._err = getattr(L, pre + "last_error")
        self._err.restype = C.c_char_p

    def _check(self, rc: int) -> None:
        if rc:
            raise OracleError(rc, self._err().decode())

    @staticmethod
    def _c(a):
        return np.ascontiguousarray(a, dtype=np.float64)

    def forward(self, pb: Problem, threads: int = 1) -> dict:
        n, dv = pb.q.shape[0], pb.v.shape[1]
        t_r, t_c = max(pb.t_r, 1), max(pb.t_c, 1)
        wpr = (t_c + 31) // 32
        out = np.zeros((n, dv))
        tau = np.zeros(n)
        rmax = np.zeros(n)
        mask = np.zeros((t_r, wpr), dtype=np.uint32)
        steps = np.zeros(n, dtype=np.int32)
        st = OrcStats()
        self._check(self._fwd(C.byref(pb.params()), self._c(pb.q), self._c(pb.k),
                              self._c(pb.v), int(threads), out, tau, rmax, mask, steps,
                              C.byref(st)))
        return dict(out=out, tau=tau, row_max=rmax, mask=mask, row_steps=steps,
                    block_sparsity=st.block_sparsity,
                    blocks_visited_fwd=int(st.blocks_visited_fwd), flushes=int(st.flushes))

    def forward_hist(self, pb: Problem, threads: int = 1) -> dict:
        """forward plus the per-row histogram counts and tau_h (C restatement only:
        the reference keeps them private)."""
        if self.kind != "port":
            raise NotImplementedError("the histogram state is internal to the reference")
        fn = self.lib.orc_forward_ex
        fn.argtypes = self._fwd.argtypes + [_DP, _U32P]
        fn.restype = C.c_int
        n, dv = pb.q.shape[0], pb.v.shape[1]
        t_r, t_c = max(pb.t_r, 1), max(pb.t_c, 1)
        out, tau, rmax = np.zeros((n, dv)), np.zeros(n), np.zeros(n)
        mask = np.zeros((t_r, (t_c + 31) // 32), dtype=np.uint32)
        steps = np.zeros(n, dtype=np.int32)
        tau_h = np.zeros(n)
        counts = np.zeros((n, pb.bins), dtype=np.uint32)
        st = OrcStats()
        self._check(fn(C.byref(pb.params()), self._c(pb.q), self._c(pb.k), self._c(pb.v),
                       int(threads), out, tau, rmax, mask, steps, C.byref(st), tau_h, counts))
        return dict(out=out, tau=tau, row_max=rmax, mask=mask, row_steps=steps, tau_h=tau_h,
                    counts=counts, block_sparsity=st.block_sparsity)

    def dense_reference(self, pb: Problem) -> dict:
        n, dv = pb.q.shape[0], pb.v.shape[1]
        wpr = (pb.t_c + 31) // 32
        out = np.zeros((n, dv))
        tau = np.zeros(n)
        rmax = np.zeros(n)
        mask = np.zeros((pb.t_r, wpr), dtype=np.uint32)
        st = OrcStats()
        self._check(self._dense(C.byref(pb.params()), self._c(pb.q), self._c(pb.k),
                                self._c(pb.v), out, tau, rmax, mask, C.byref(st)))
        return dict(out=out, tau=tau, row_max=rmax, mask=mask,
                    block_sparsity=st.block_sparsity)

    def compute_delta(self, pb: Problem, res: dict, dout: np.ndarray, threads: int = 1):
        delta = np.zeros(pb.q.shape[0])
        self._check(self._delta(C.byref(pb.params()), self._c(pb.q), self._c(pb.k),
                                self._c(pb.v), self._c(res["tau"]), self._c(res["row_max"]),
                                np.ascontiguousarray(res["mask"], dtype=np.uint32),
                                self._c(dout), int(threads), delta))
        return delta

    def backward(self, pb: Problem, res: dict, dout: np.ndarray, threads: int = 1) -> dict:
        n, m, d, dv = pb.q.shape[0], pb.k.shape[0], pb.q.shape[1], pb.v.shape[1]
        dq = np.zeros((n, d))
        dk = np.zeros((m, d))
        dvv = np.zeros((m, dv))
        delta = np.zeros(n)
        vis = np.zeros(1, dtype=np.uint64)
        self._check(self._bwd(C.byref(pb.params()), self._c(pb.q), self._c(pb.k),
                              self._c(pb.v), self._c(res["tau"]), self._c(res["row_max"]),
                              np.ascontiguousarray(res["mask"], dtype=np.uint32),
                              self._c(dout), int(threads), dq, dk, dvv, delta, vis))
        return dict(dq=dq, dk=dk, dv=dvv, delta=delta, blocks_visited_bwd=int(vis[0]))

    def block_sparsity(self, mask: np.ndarray, t_r: int, t_c: int, causal: bool) -> float:
        return float(self._bs(np.ascontiguousarray(mask, dtype=np.uint32), t_r, t_c,
                              int(causal)))

    def solve_histogram(self, counts, alpha: float):
        c = np.ascontiguousarray(counts, dtype=np.uint32)
        th, lo, hi = C.c_double(), C.c_double(), C.c_double()
        fl = C.c_int()
        self._check(self._sh(c, len(c), float(alpha), C.byref(th), C.byref(fl), C.byref(lo),
                             C.byref(hi)))
        return th.value, fl.value, lo.value, hi.value

    def f_eval(self, z, alpha: float, tau: float):
        zz = self._c(z)
        f, f1, f2 = C.c_double(), C.c_double(), C.c_double()
        self._fe(zz, len(zz), float(alpha), float(tau), C.byref(f), C.byref(f1), C.byref(f2))
        return f.value, f1.value, f2.value

    def gaussian(self, seed: int, count: int, scale: float = 1.0) -> np.ndarray:
        out = np.zeros(count)
        self._gf(seed, scale, out, count)
        return out

    def xoshiro_next(self, seed: int, count: int) -> np.ndarray:
        out = np.zeros(count, dtype=np.uint64)
        self._xn(seed, out, count)
        return out

    def propose_step(self, alpha, tau, f, f1, f2, sec_tau, sec_f, lo, hi):
        if self.kind != "port":
            raise NotImplementedError("propose_step is internal to the reference")
        fn = self.lib.orc_propose_step
        fn.argtypes = [C.c_double] * 9 + [C.POINTER(C.c_int)]
        fn.restype = C.c_double
        k = C.c_int()
        v = fn(alpha, tau, f, f1, f2, sec_tau, sec_f, lo, hi, C.byref(k))
        return v, k.value


def gen_attn_inputs(seed: int, n: int, d: int, qscale: float = 1.0, lib: Oracle | None = None):
    """cmd_attn input stream (atn_main.cpp:227-232): Q=qscale*N(0,1), K, V, dO."""
    lib = lib or Oracle("port")
    g = lib.gaussian(seed, 4 * n * d)
    # qscale multiplies each deviate before storage (gaussian_matrix, atn_main.cpp:73-77);
    # the elementwise IEEE product equals the reference's scalar product.
    q = (qscale * g[: n * d]).reshape(n, d)
    k = g[n * d: 2 * n * d].reshape(n, d).copy()
    v = g[2 * n * d: 3 * n * d].reshape(n, d).copy()
    do = g[3 * n * d:].reshape(n, d).copy()
    return q, k, v, do
