"""Row-wise alpha-entmax thresholds on materialised scores.

``entmax_rows`` runs the reference's per-vector solvers on every row of a
[rows, n] score matrix on the GPU (csrc/rows.cu through
``adattn_b200_entmax_rows``): histogram init + hybrid refinement (the paper's
inference variant), hybrid from the bracket midpoint, or bisection.
``solver_bench`` is the reference's convergence experiment (hybrid.cpp:108-178,
`atn bench-solver`, Fig. 3) with the GPU solvers: mean |tau_k - tau*|
per iteration over Gaussian score vectors drawn from Xoshiro256pp(seed + r).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, dense, tensor_io

_DT = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16, torch.float64: _lib.F64}
METHODS = {"histogram+hybrid": _lib.ROWS_HISTOGRAM_HYBRID, "hybrid": _lib.ROWS_HYBRID,
           "bisection": _lib.ROWS_BISECTION}


@dataclass
class RowsResult:
    tau: torch.Tensor          # [rows] fp64, centred scale
    residual: torch.Tensor     # [rows] f(tau)
    iterations: torch.Tensor   # [rows] int32
    converged: torch.Tensor    # [rows] bool
    probs: torch.Tensor | None = None   # [rows, n] fp32
    trace: torch.Tensor | None = None   # [rows, trace_len] fp64


def entmax_rows(scores: torch.Tensor, alpha: float, method: str = "histogram+hybrid",
                bins: int = 8, max_iters: int = 2, tol: float = 1e-6, mask=None,
                probs: bool = False, trace_len: int = 0) -> RowsResult:
    if scores.dim() != 2:
        raise ValueError("entmax_rows: scores must be [rows, n]")
    if not scores.is_cuda:
        raise ValueError("entmax_rows: scores must be on a CUDA device (no CPU path)")
    if scores.dtype not in _DT:
        raise ValueError(f"entmax_rows: unsupported dtype {scores.dtype}")
    if method not in METHODS:
        raise ValueError("solve: unknown --method " + method)
    s = scores.contiguous()
    rows, n = s.shape
    dev = s.device
    m = None
    if mask is not None:
        m = mask.to(device=dev, dtype=torch.uint8).contiguous()
        if m.shape != s.shape:
            raise ValueError("center_scores: mask size mismatch")
    tau = torch.empty(rows, dtype=torch.float64, device=dev)
    res = torch.empty_like(tau)
    its = torch.empty(rows, dtype=torch.int32, device=dev)
    conv = torch.empty(rows, dtype=torch.int32, device=dev)
    pr = torch.empty(rows, n, dtype=torch.float32, device=dev) if probs else None
    tr = torch.empty(rows, trace_len, dtype=torch.float64, device=dev) if trace_len > 0 else None
    pb = _lib.RowsProblem(rows, n, _DT[s.dtype], float(alpha), int(bins), int(max_iters),
                          float(tol), METHODS[method], int(trace_len))
    P = lambda t: None if t is None else C.c_void_p(t.data_ptr())
    _lib.check(_lib.load().adattn_b200_entmax_rows(
        C.byref(pb), P(s), P(m), P(tau), P(res), P(its), P(conv), P(pr), P(tr),
        C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    return RowsResult(tau, res, its, conv.bool(), pr, tr)


def solver_bench(n: int, alpha: float, bins_list, runs: int, seed: int, iters: int = 10,
                 device="cuda"):
    """[(method, iteration, mae)] as solver_bench (hybrid.cpp:108-178)."""
    if n < 2 or runs < 1 or iters < 1:
        raise ValueError("solver_bench: bad n/runs/iters")
    rows = np.stack([tensor_io.xoshiro(seed + r, 0, n)[1] for r in range(runs)])
    s = torch.from_numpy(rows).to(device)
    # tau* of every run: exact (alpha 1.5 / 2) or bisection to 1e-14 (dense.py, fp64)
    z = (alpha - 1.0) * (s - s.amax(dim=1, keepdim=True)) + 1.0
    z = torch.where(s == s.amax(dim=1, keepdim=True), torch.ones_like(z), z)
    tau_star = (dense._tau_exact(z, alpha) if alpha in (1.5, 2.0)
                else dense._tau_bisection(z, alpha)).cpu().numpy()
    out = []
    runs_m = [("bisection", dict(method="bisection", max_iters=iters + 1, tol=0.0)),
              ("hybrid", dict(method="hybrid", max_iters=iters, tol=0.0))]
    runs_m += [(f"hist-B{b}", dict(method="histogram+hybrid", bins=b, max_iters=iters, tol=0.0))
               for b in bins_list]
    for name, kw in runs_m:
        r = entmax_rows(s, alpha, trace_len=iters + 1, **kw)
        tr = r.trace.cpu().numpy()
        mae = np.abs(tr - tau_star[:, None]).mean(axis=0)
        out += [(name, k, float(mae[k])) for k in range(iters + 1)]
    return out
