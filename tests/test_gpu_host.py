"""The C-ABI host entry (adattn_b200_run_host, include/adattn_b200.h): pinned or
pageable host buffers in, host buffers out, run as a copy/compute pipeline over
chunks of heads -- results identical to the device entry points."""
import ctypes as C

import pytest
import torch

import paper_2604_15180_b200 as pa
from paper_2604_15180_b200 import _lib

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.mark.parametrize("bh,pinned,N", [((2, 8), True, 1024), ((1, 3), False, 1024),
                                         ((4, 16), True, 1024), ((2, 13), True, 512)])
def test_run_host_matches_device_path(bh, pinned, N):
    """(2, 13): 26 heads -> 2-head end chunks around unequal middle chunks (5, 5, 4, 4)."""
    B, H = bh
    D = 128
    g = torch.Generator(device="cpu").manual_seed(B * 100 + H)
    q, k, v, do = ((torch.randn(B, H, N, D, generator=g)).to(torch.bfloat16) for _ in range(4))
    prob = pa.AttentionProblem(q.to(DEV), k.to(DEV), v.to(DEV), path="tc", alpha=1.5, causal=True)
    res = pa.forward(prob)
    grads = pa.backward(prob, res, do.to(DEV))
    torch.cuda.synchronize()

    lib = _lib.load()
    pb = prob.c_problem(out_dtype_code=_lib.F32)
    mk = (lambda t: t.pin_memory()) if pinned else (lambda t: t)
    hq, hk, hv, hdo = (mk(x.contiguous()) for x in (q, k, v, do))
    T = N // 64
    hout = mk(torch.empty(B, H, N, D, dtype=torch.float32))
    hdq, hdk, hdv = (mk(torch.empty(B, H, N, D, dtype=torch.float32)) for _ in range(3))
    htau, hrm, hdl = (mk(torch.empty(B, H, N, dtype=torch.float64)) for _ in range(3))
    hmask = mk(torch.empty(B, H, T, (T + 31) // 32, dtype=torch.int32))
    st = _lib.Stats()
    P = lambda t: C.c_void_p(t.data_ptr())
    _lib.check(lib.adattn_b200_run_host(C.byref(pb), P(hq), P(hk), P(hv), P(hdo), P(hout), P(htau),
                                        P(hrm), P(hmask), P(hdq), P(hdk), P(hdv), P(hdl),
                                        C.byref(st)))
    assert torch.equal(hout, res.out.float().cpu())
    assert torch.equal(htau, res.tau.cpu())
    assert torch.equal(hrm, res.row_max.cpu())
    assert torch.equal(hmask.view(torch.int32).flatten(), res.mask.words.view(torch.int32).cpu().flatten())
    assert torch.equal(hdl, grads.delta.cpu())
    for h, d in ((hdq, grads.dq), (hdk, grads.dk), (hdv, grads.dv)):
        assert torch.equal(h, d.float().cpu())
    assert abs(st.block_sparsity - res.stats.block_sparsity) < 1e-12
