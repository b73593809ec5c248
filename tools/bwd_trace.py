"""Event trace of the pair dK/dV kernel's first cluster (ADATTN_PIPE_STATS build):
per unit the cycles at which warp 9 (S^T/dP^T), warp 10 (gradients) and epilogue
warp 0 pass their waits.  python tools/bwd_trace.py B H N"""
import ctypes as C, os, sys
sys.path.insert(0, ".")
import paper_2604_15180_b200._lib as L
L.LIB_PATH = os.path.abspath(os.environ.get("LIB", "paper_2604_15180_b200/libadattn_b200_stats.so"))
import torch
import paper_2604_15180_b200 as pa
from paper_2604_15180_b200 import workloads
lib = L.load()
B, H, N = (int(x) for x in sys.argv[1:4])
os.environ.setdefault("ADATTN_DELTA_FOLD", "0")
q, k, v, do = workloads.gaussian(B, H, N, 128, 1.0, seed=1)
p = pa.AttentionProblem(q, k, v, alpha=1.5, causal=True)
r = pa.forward(p); g = pa.backward(p, r, do); torch.cuda.synchronize()
g = pa.backward(p, r, do); torch.cuda.synchronize()
buf = (C.c_longlong * (3 * 512 * 4))()
lib.adattn_b200_bwd_trace(buf)
t = [[[buf[(r_ * 512 + u) * 4 + e] for e in range(4)] for u in range(512)] for r_ in range(3)]
t0 = t[0][0][0]
print("u | W9: start full grad_done issued | W10: start p_full issued | EPI: start s_full arrive")
for u in list(range(0, 8)) + list(range(200, 216)):
    w9, w10, ep = t[0][u], t[1][u], t[2][u]
    if w9[0] == 0:
        continue
    f = lambda x: x - t0 if x else -1
    print(u, "|", *[f(x) for x in w9], "|", *[f(x) for x in w10[:3]], "|", *[f(x) for x in ep[:3]])
