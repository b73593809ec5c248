"""Host-side mirror of the reference's tiled-attention interface.

Same names, argument meaning and error behaviour as
``/root/reference/proj/include/adattn/attention.hpp:24-123``:

=======================  ===========================================  =====================
this module              reference                                    C-ABI entry
=======================  ===========================================  =====================
``AttentionProblem``     ``AttentionProblem`` (attention.hpp:24-36)   ``adattn_problem``
``forward``              ``forward`` (attention.hpp:72-76)            ``adattn_b200_forward``
``compute_delta``        ``compute_delta`` (attention.hpp:82-85)      ``..._compute_delta``
``backward``             ``backward`` (attention.hpp:87-92)           ``adattn_b200_backward``
``block_sparsity``       ``block_sparsity`` (attention.hpp:94-97)     ``adattn_b200_stats``
``PackedBlockMask``      ``PackedBlockMask`` (bitpack.hpp:72-110)     mask word layout
=======================  ===========================================  =====================

Invalid problems raise ``ValueError`` with the reference's
``std::invalid_argument`` message.  Tensors live on the GPU (torch is only
the allocator and stream provider); every number is computed by the CUDA
kernels in ``libadattn_b200.so`` -- there is no CPU path.  Inputs may be a
single head ``[n, d]`` (the reference's shape) or a batch ``[B, H, n, d]``.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field
from typing import Optional

import torch

from . import _lib

_PATHS = {"auto": _lib.PATH_AUTO, "exact": _lib.PATH_EXACT, "tc": _lib.PATH_TC}
_IN_DTYPES = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16, torch.float64: _lib.F64}
_OUT_DTYPES = {torch.float32: _lib.F32, torch.float64: _lib.F64}


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


@dataclass
class AttentionProblem:
    """Mirror of AttentionProblem (attention.hpp:24-36), batched over [B, H]."""
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    alpha: float = 1.5
    scale: float = 0.0  # 0 => 1/sqrt(d)
    causal: bool = False
    block_r: int = 64
    block_c: int = 64
    bins: int = 8
    refine_iters: int = 2
    refine_tol: float = 1e-6
    path: str = "auto"  # 'auto' | 'exact' (fp64 SIMT) | 'tc' (bf16 tcgen05)
    out_dtype: Optional[torch.dtype] = None  # default: float64 on exact, float32 on tc

    def _dims(self):
        q, k, v = self.q, self.k, self.v
        if q.dim() == 2:
            lead = ()
            B, H = 1, 1
        elif q.dim() == 4:
            lead = tuple(q.shape[:2])
            B, H = lead
        else:
            raise ValueError("attention: q must be [n, d] or [B, H, n, d]")
        if k.dim() != q.dim() or v.dim() != q.dim():
            raise ValueError("attention: q, k, v ranks differ")
        if tuple(k.shape[:-2]) != lead or tuple(v.shape[:-2]) != lead:
            raise ValueError("attention: q, k, v batch shapes differ")
        n, d = q.shape[-2:]
        m, dk = k.shape[-2:]
        mv, dv = v.shape[-2:]
        if dk != d:
            raise ValueError("attention: q/k width mismatch")
        if mv != m:
            raise ValueError("attention: k/v length mismatch")
        return lead, B, H, n, m, d, dv

    def c_problem(self, out_dtype_code: int = -1) -> _lib.Problem:
        lead, B, H, n, m, d, dv = self._dims()
        if self.q.dtype not in _IN_DTYPES:
            raise ValueError(f"attention: unsupported input dtype {self.q.dtype}")
        if self.k.dtype != self.q.dtype or self.v.dtype != self.q.dtype:
            raise ValueError("attention: q, k, v dtypes differ")
        if self.path not in _PATHS:
            raise ValueError(f"attention: unknown path {self.path!r}")
        pb = _lib.Problem(B, H, n, m, d, dv, float(self.alpha), float(self.scale),
                          int(bool(self.causal)), int(self.block_r), int(self.block_c),
                          int(self.bins), int(self.refine_iters), float(self.refine_tol),
                          _IN_DTYPES[self.q.dtype], _lib.F64, _PATHS[self.path], 0)
        if out_dtype_code >= 0:
            pb.out_dtype = out_dtype_code
        elif self.out_dtype is not None:
            pb.out_dtype = _OUT_DTYPES[self.out_dtype]
        else:
            path = resolved_path(pb)
            pb.out_dtype = _lib.F64 if path == _lib.PATH_EXACT else _lib.F32
        return pb

    @property
    def t_r(self) -> int:
        return (self.q.shape[-2] + self.block_r - 1) // self.block_r

    @property
    def t_c(self) -> int:
        return (self.k.shape[-2] + self.block_c - 1) // self.block_c


def resolved_path(pb: _lib.Problem) -> int:
    lib = _lib.load()
    r = lib.adattn_b200_resolved_path(C.byref(pb))
    if r < 0:
        _lib.check(-r)
    return r


class PackedBlockMask:
    """Reference PackedBlockMask (bitpack.hpp:72-110) over device words.

    ``words`` is ``[..., t_r, ceil(t_c/32)]`` uint32 (stored as int32 in torch),
    LSB-first, trailing bits zero -- the reference's exact word layout.
    """

    def __init__(self, words: torch.Tensor, t_r: int, t_c: int):
        self.words = words
        self.t_r, self.t_c = int(t_r), int(t_c)
        self.words_per_row = (self.t_c + 31) // 32

    def tile_rows(self) -> int:
        return self.t_r

    def tile_cols(self) -> int:
        return self.t_c

    def _host(self, head: int = 0):
        w = self.words.reshape(-1, self.t_r, self.words_per_row)[head]
        return w.to("cpu").view(torch.int32).numpy().view("uint32")

    def test(self, i: int, j: int, head: int = 0) -> bool:
        if not (0 <= i < self.t_r and 0 <= j < self.t_c):
            raise ValueError("PackedBlockMask: index out of range")
        return bool((int(self._host(head)[i, j // 32]) >> (j % 32)) & 1)

    def row_popcount(self, i: int, head: int = 0) -> int:
        return int(sum(bin(int(x)).count("1") for x in self._host(head)[i]))

    def total_popcount(self) -> int:
        w = self.words.to("cpu").view(torch.int32).numpy().view("uint32")
        import numpy as np
        return int(np.unpackbits(w.view(np.uint8)).sum())

    def serialize(self, head: int = 0) -> bytes:
        """Byte layout of PackedBlockMask::serialize (bitpack.cpp:145-158)."""
        h = self._host(head)
        return struct.pack("<II", self.t_r, self.t_c) + h.astype("<u4").tobytes()

    def __eq__(self, other) -> bool:
        return (isinstance(other, PackedBlockMask) and self.t_r == other.t_r
                and self.t_c == other.t_c and torch.equal(self.words.cpu(), other.words.cpu()))


@dataclass
class AttentionStats:
    """Mirror of AttentionStats (attention.hpp:38-43), aggregated over heads."""
    block_sparsity: float = 0.0
    blocks_visited_fwd: int = 0
    blocks_visited_bwd: int = 0
    flushes: int = 0


@dataclass
class NonzeroBlockLists:
    """The forward's per-row-block nonzero-block lists (ELL, on the device):
    ``cnt[..., i]`` active key blocks of row block i, ``cols[..., i, :cnt]`` their
    indices ascending (PackedBlockMask::for_each_set order, bitpack.hpp:85-92).
    The backward's kernels walk them (and their transpose)."""
    cnt: torch.Tensor   # int32 [..., t_r]
    cols: torch.Tensor  # int16 storage of uint16 [..., t_r, t_c]

    def row(self, i: int, head: int = 0) -> list:
        c = self.cnt.reshape(-1, self.cnt.shape[-1])[head, i].item()
        v = self.cols.reshape(-1, *self.cols.shape[-2:])[head, i, :c]
        return [int(x) & 0xFFFF for x in v.cpu().tolist()]


@dataclass
class AttentionResult:
    """Mirror of AttentionResult (attention.hpp:45-55)."""
    out: torch.Tensor
    tau: torch.Tensor
    row_max: torch.Tensor
    mask: PackedBlockMask
    row_steps: torch.Tensor
    lists: Optional[NonzeroBlockLists] = None
    # the output pass's sum_j u_ij v_j and sum_j u_ij (float32, flat: [B*H*n*dv] then
    # [B*H*n]) when the forward folded the delta accumulation; the
    # backward then forms delta = dO . Ubar / sum u instead of a delta pre-pass
    delta_aux: Optional[torch.Tensor] = field(repr=False, default=None)
    _problem: _lib.Problem = field(repr=False, default=None)
    _stats: Optional[AttentionStats] = field(repr=False, default=None)
    _bwd_done: bool = field(repr=False, default=False)

    @property
    def path(self) -> str:
        """The kernels that ran: "tc" (bf16 tcgen05) or "exact" (fp64 SIMT) --
        AUTO sends bf16 inputs outside the tensor-core envelope to "exact"."""
        return "tc" if resolved_path(self._problem) == _lib.PATH_TC else "exact"

    @property
    def stats(self) -> AttentionStats:
        """Lazily computed (one popcount kernel + a stream sync) on first access."""
        if self._stats is None:
            st = _mask_stats(self._problem, self.mask.words)
            self._stats = AttentionStats(st.block_sparsity, int(st.blocks_visited_fwd), 0,
                                         int(st.flushes))
        self._stats.blocks_visited_bwd = 2 * self._stats.blocks_visited_fwd if self._bwd_done else 0
        return self._stats


@dataclass
class AttentionGradients:
    """Mirror of AttentionGradients (attention.hpp:57-60)."""
    dq: torch.Tensor
    dk: torch.Tensor
    dv: torch.Tensor
    delta: torch.Tensor


@dataclass
class PhaseTimings:
    """Mirror of PhaseTimings (attention.hpp:62-66): ms[0..3] += row max,
    histogram, refinement, output time of a forward (attention.cpp:196-199,
    229-232, 329-332, 352), filled like the reference only when
    ``threads <= 1``.  The GPU forward runs the four phases inside one kernel;
    its CUDA-event duration is split by the share of CTA time each phase took
    (adattn_b200_forward_timed)."""
    ms: list = field(default_factory=lambda: [0.0, 0.0, 0.0, 0.0])


def _mask_stats(pb: _lib.Problem, words: torch.Tensor) -> _lib.Stats:
    lib = _lib.load()
    st = _lib.Stats()
    _lib.check(lib.adattn_b200_stats(C.byref(pb), _ptr(words), C.byref(st), _stream()))
    return st


def _check_device(*ts):
    for t in ts:
        if not t.is_cuda:
            raise ValueError("attention: tensors must live on a CUDA device (no CPU path)")
        if not t.is_contiguous():
            raise ValueError("attention: tensors must be contiguous row-major")


_torch_out = {_lib.F32: torch.float32, _lib.F64: torch.float64}


def forward(p: AttentionProblem, threads: int = 1, timings: Optional[PhaseTimings] = None,
            tau_h: Optional[torch.Tensor] = None) -> AttentionResult:
    """Tiled alpha-entmax forward (attention.cpp:157-361).  ``threads`` only
    gates ``timings`` as in the reference (work goes to the current stream)."""
    pb = p.c_problem()
    lib = _lib.load()
    _lib.check(lib.adattn_b200_validate(C.byref(pb)))
    _check_device(p.q, p.k, p.v)
    lead = tuple(p.q.shape[:-2])
    dev = p.q.device
    n, dv = pb.n, pb.dv
    t_r, t_c = p.t_r, p.t_c
    wpr = (t_c + 31) // 32
    out = torch.empty(lead + (n, dv), dtype=_torch_out[pb.out_dtype], device=dev)
    tau = torch.empty(lead + (n,), dtype=torch.float64, device=dev)
    row_max = torch.empty(lead + (n,), dtype=torch.float64, device=dev)
    words = torch.empty(lead + (t_r, wpr), dtype=torch.int32, device=dev)
    steps = torch.empty(lead + (n,), dtype=torch.int32, device=dev)
    ws_bytes = lib.adattn_b200_forward_workspace(C.byref(pb))
    ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=dev)
    args = (C.byref(pb), _ptr(p.q), _ptr(p.k), _ptr(p.v), _ptr(out), _ptr(tau), _ptr(row_max),
            _ptr(words), _ptr(steps), _ptr(ws), ws_bytes, _stream())
    timed = timings is not None and threads <= 1  # attention.cpp:170
    lists = None
    if t_c <= 65535:  # the nonzero-block lists the backward walks (uint16 indices)
        lists = NonzeroBlockLists(torch.empty(lead + (t_r,), dtype=torch.int32, device=dev),
                                  torch.empty(lead + (t_r, t_c), dtype=torch.int16, device=dev))
    # tau_h (optional, float64 like tau): each row's histogram solution
    # (solve_histogram, histogram.cpp:73-161), which the reference keeps private
    if tau_h is not None:
        if tau_h.shape != tau.shape or tau_h.dtype != torch.float64:
            raise ValueError("forward: tau_h must be float64 shaped like tau")
        _check_device(tau_h)
    ph = (C.c_double * 4)()
    aux_bytes = lib.adattn_b200_delta_aux_bytes(C.byref(pb))
    aux = torch.empty(aux_bytes // 4, dtype=torch.float32, device=dev) if aux_bytes else None
    ex = _lib.ForwardExtras(ph if timed else None, _ptr(tau_h),
                            _ptr(lists.cnt) if lists else None,
                            _ptr(lists.cols) if lists else None, _ptr(aux))
    _lib.check(lib.adattn_b200_forward_ex(*args, C.byref(ex)))
    if timed:
        for i in range(4):
            timings.ms[i] += ph[i]
    return AttentionResult(out, tau, row_max, PackedBlockMask(words, t_r, t_c), steps, lists,
                           aux, pb)


def _grad_problem(p: AttentionProblem, res: AttentionResult, dout: torch.Tensor) -> _lib.Problem:
    pb = p.c_problem(out_dtype_code=_OUT_DTYPES.get(res.out.dtype, _lib.F32))
    if tuple(dout.shape) != tuple(res.out.shape):
        raise ValueError("backward: dout shape mismatch")
    if dout.dtype != p.q.dtype:
        raise ValueError("backward: dout dtype must match q")
    _check_device(dout, res.tau, res.row_max, res.mask.words)
    return pb


def compute_delta(p: AttentionProblem, res: AttentionResult, dout: torch.Tensor,
                  threads: int = 1) -> torch.Tensor:
    """delta_i = <u_i, dP_i>/<u_i, 1>, u = P^(2-alpha) (attention.cpp:411-446)."""
    del threads
    pb = _grad_problem(p, res, dout)
    lib = _lib.load()
    delta = torch.empty_like(res.tau)
    ws_bytes = lib.adattn_b200_backward_workspace(C.byref(pb))
    ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=p.q.device)
    _lib.check(lib.adattn_b200_compute_delta(
        C.byref(pb), _ptr(p.q), _ptr(p.k), _ptr(p.v), _ptr(res.tau), _ptr(res.row_max),
        _ptr(res.mask.words), _ptr(dout), _ptr(delta), _ptr(ws), ws_bytes, _stream()))
    return delta


def backward(p: AttentionProblem, res: AttentionResult, dout: torch.Tensor,
             threads: int = 1) -> AttentionGradients:
    """Mask-guided backward (attention.cpp:448-539).  Like the reference it
    updates ``res.stats.blocks_visited_bwd`` (two visits per active block)."""
    del threads
    pb = _grad_problem(p, res, dout)
    lib = _lib.load()
    gdt = res.out.dtype
    dq = torch.empty(p.q.shape, dtype=gdt, device=p.q.device)
    dk = torch.empty(p.k.shape, dtype=gdt, device=p.q.device)
    dv = torch.empty(p.v.shape, dtype=gdt, device=p.q.device)
    delta = torch.empty_like(res.tau)
    ws_bytes = lib.adattn_b200_backward_workspace(C.byref(pb))
    ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=p.q.device)
    lists = res.lists
    ex = _lib.BackwardExtras(_ptr(lists.cnt) if lists else None,
                             _ptr(lists.cols) if lists else None, _ptr(res.delta_aux))
    _lib.check(lib.adattn_b200_backward_ex(
        C.byref(pb), _ptr(p.q), _ptr(p.k), _ptr(p.v), _ptr(res.tau), _ptr(res.row_max),
        _ptr(res.mask.words), _ptr(dout), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(delta), _ptr(ws),
        ws_bytes, _stream(), C.byref(ex)))
    res._bwd_done = True  # stats report blocks_visited_bwd = 2 * nnz (attention.cpp:537)
    return AttentionGradients(dq, dk, dv, delta)


def block_sparsity(mask: PackedBlockMask, causal: bool) -> float:
    """Zero-bit fraction over the addressable blocks (attention.cpp:541-551),
    aggregated over all heads in ``mask.words``."""
    words = mask.words.reshape(-1, mask.t_r, mask.words_per_row).contiguous()
    lib = _lib.load()
    st = _lib.Stats()
    _lib.check(lib.adattn_b200_mask_sparsity(_ptr(words), words.shape[0], mask.t_r, mask.t_c,
                                             int(bool(causal)), C.byref(st), _stream()))
    return float(st.block_sparsity)


@dataclass
class BlockLists:
    """Nonzero-block lists of a forward's mask (all heads, head-major), on the device.

    ``rowptr[h*t_r + i] .. rowptr[h*t_r + i + 1]`` indexes ``cols``: the active key
    blocks of row block i of head h, in PackedBlockMask::for_each_set order
    (bitpack.hpp:85-92); ``colptr`` / ``rows`` are the transposed lists (active
    query blocks of each key block, ascending; PackedBlockMask::transposed,
    bitpack.cpp:138-143).  Block indices are local to the head."""
    rowptr: torch.Tensor
    cols: torch.Tensor
    colptr: torch.Tensor
    rows: torch.Tensor


def block_lists(p: AttentionProblem, res: AttentionResult) -> BlockLists:
    """Per-row-block lists of the active key blocks (and their transpose) that
    the output pass and the key-major backward sweep visit (csrc/lists.cu)."""
    pb = p.c_problem()
    lib = _lib.load()
    words = res.mask.words.contiguous()
    dev = words.device
    bh = pb.batch * pb.heads
    nnz = int(res.stats.blocks_visited_fwd)  # = popcount of the mask
    rowptr = torch.empty(bh * res.mask.t_r + 1, dtype=torch.int64, device=dev)
    colptr = torch.empty(bh * res.mask.t_c + 1, dtype=torch.int64, device=dev)
    cols = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    rows = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    _lib.check(lib.adattn_b200_block_lists(C.byref(pb), _ptr(words), _ptr(rowptr), _ptr(cols),
                                           _ptr(colptr), _ptr(rows), _stream()))
    return BlockLists(rowptr, cols[:nnz], colptr, rows[:nnz])
