"""compute-sanitizer driver (dev tool): one small call of every GPU code path --
TC list mode / sweep mode / overflow fallback / bins 32, CTA pairs, ragged and
width-padded problems, EXACT tiled and generic kernels, forward_ex extras, lists,
run_host.  python tools/sanitize_smoke.py  (under compute-sanitizer --tool memcheck)"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_15180_b200 as pa
from paper_2604_15180_b200 import _lib

g = torch.Generator(device="cpu").manual_seed(0)


def mk(B, H, n, d, dtype=torch.bfloat16):
    return torch.randn(B, H, n, d, generator=g).to(dtype).cuda()


def fb(q, k, v, do, **kw):
    p = pa.AttentionProblem(q, k, v, **kw)
    t = pa.PhaseTimings()
    th = torch.empty(q.shape[:-1], dtype=torch.float64, device=q.device)
    r = pa.forward(p, 1, t, tau_h=th)
    gr = pa.backward(p, r, do)
    pa.block_lists(p, r)
    _ = r.stats
    return r, gr


q, k, v, do = (mk(1, 2, 1024, 128) for _ in range(4))
for causal in (True, False):
    fb(q, k, v, do, path="tc", alpha=1.5, causal=causal)                 # list mode
fb(q, k, v, do, path="tc", alpha=1.25, causal=True)                      # sweep mode
fb(q, k, v, do, path="tc", alpha=1.5, causal=True, bins=32)              # bins 32
os.environ["ADATTN_CAND_CAP"] = "64"
fb(q, k, v, do, path="tc", alpha=1.5, causal=True)                       # overflow fallback
fb(q, k, v, do, path="tc", alpha=1.5, causal=True, bins=32)
del os.environ["ADATTN_CAND_CAP"]
os.environ["ADATTN_FWD_PAIRS"] = "1"
fb(q, k, v, do, path="tc", alpha=2.0, causal=True)                       # CTA pairs
del os.environ["ADATTN_FWD_PAIRS"]
q2, k2, v2, do2 = mk(1, 2, 300, 96), mk(1, 2, 300, 96), mk(1, 2, 300, 96), mk(1, 2, 300, 96)
fb(q2, k2, v2, do2, path="tc", alpha=1.5, causal=True)                   # ragged + width
q3, k3, v3, do3 = mk(1, 1, 200, 64), mk(1, 1, 333, 64), mk(1, 1, 333, 128), mk(1, 1, 200, 128)
fb(q3, k3, v3, do3, path="tc", alpha=2.0, causal=False)                  # d != dv
x = lambda n, d: mk(1, 2, n, d, torch.float32)
fb(x(150, 32), x(150, 32), x(150, 32), x(150, 32), path="exact", alpha=1.5, causal=True)
fb(x(130, 200), x(130, 200), x(130, 140), x(130, 140), path="exact", alpha=2.0, causal=True,
   block_r=100, block_c=96)                                               # generic exact
torch.cuda.synchronize()
lib = _lib.load()
B, H, N, D = 1, 4, 1024, 128
q, k, v, do = (mk(B, H, N, D) for _ in range(4))
p = pa.AttentionProblem(q, k, v, path="tc", alpha=1.5, causal=True)
pb = p.c_problem(out_dtype_code=_lib.F32)
hq, hk, hv, hdo = (t.cpu().contiguous() for t in (q, k, v, do))
T = N // 64
ho = torch.empty(B, H, N, D)
hdq, hdk, hdv = (torch.empty(B, H, N, D) for _ in range(3))
ht, hr, hd = (torch.empty(B, H, N, dtype=torch.float64) for _ in range(3))
hm = torch.empty(B, H, T, (T + 31) // 32, dtype=torch.int32)
P = lambda t: C.c_void_p(t.data_ptr())
_lib.check(lib.adattn_b200_run_host(C.byref(pb), P(hq), P(hk), P(hv), P(hdo), P(ho), P(ht),
                                    P(hr), P(hm), P(hdq), P(hdk), P(hdv), P(hd), None))
print("sanitizer run done")
