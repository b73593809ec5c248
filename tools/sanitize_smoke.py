import sys, torch, ctypes as C
sys.path.insert(0, ".")
import paper_2604_15180_b200 as pa
from paper_2604_15180_b200 import _lib
g = torch.Generator(device="cpu").manual_seed(0)
B, H, N, D = 1, 4, 1024, 128
q, k, v, do = ((torch.randn(B, H, N, D, generator=g)).to(torch.bfloat16).cuda() for _ in range(4))
for causal in (True, False):
    p = pa.AttentionProblem(q, k, v, path="tc", alpha=1.5, causal=causal)
    r = pa.forward(p); gr = pa.backward(p, r, do); bl = pa.block_lists(p, r)
torch.cuda.synchronize()
lib = _lib.load(); pb = p.c_problem(out_dtype_code=_lib.F32)
hq, hk, hv, hdo = (x.cpu().contiguous() for x in (q, k, v, do))
T = N // 64
ho = torch.empty(B, H, N, D); hdq, hdk, hdv = (torch.empty(B, H, N, D) for _ in range(3))
ht, hr, hd = (torch.empty(B, H, N, dtype=torch.float64) for _ in range(3))
hm = torch.empty(B, H, T, (T + 31) // 32, dtype=torch.int32)
P = lambda t: C.c_void_p(t.data_ptr())
_lib.check(lib.adattn_b200_run_host(C.byref(pb), P(hq), P(hk), P(hv), P(hdo), P(ho), P(ht), P(hr), P(hm), P(hdq), P(hdk), P(hdv), P(hd), None))
print("sanitizer run done")
