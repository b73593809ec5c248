"""dK/dV kernel wait fractions (ADATTN_PIPE_STATS build).  python tools/bwd_stats.py B H N  (env D=64 CAUSAL=0 for other shapes)"""
import ctypes as C, os, sys
sys.path.insert(0, ".")
import paper_2604_15180_b200._lib as L
L.LIB_PATH = os.path.abspath(os.environ.get("LIB", "paper_2604_15180_b200/libadattn_b200_stats.so"))
import torch
import paper_2604_15180_b200 as pa
from paper_2604_15180_b200 import workloads
lib = L.load()
fn = lib.adattn_b200_bwd_stats
fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
B, H, N = (int(x) for x in sys.argv[1:4])
os.environ.setdefault("ADATTN_DELTA_FOLD", "0")
D = int(os.environ.get("D", "128"))
causal = os.environ.get("CAUSAL", "1") == "1"
q, k, v, do = workloads.gaussian(B, H, N, D, 1.0, seed=1)
p = pa.AttentionProblem(q, k, v, alpha=1.5, causal=causal)
r = pa.forward(p); g = pa.backward(p, r, do); torch.cuda.synchronize()
buf = (C.c_ulonglong * 8)()
fn(buf, 1)
g = pa.backward(p, r, do); torch.cuda.synchronize()
fn(buf, 1)
st = list(buf)
mma = max(st[3], 1)
print("units", st[4], "MMA cycles/unit", mma / max(st[4], 1))
for i, n in enumerate(["mma_wait_stage(TMA)", "mma_wait_p_full(epi)", "epi_w4_wait_s_full"]):
    print(f"{n:24s} {st[i] / mma:6.3f} of MMA-warp cycles")
print("warp 9 grad_done wait per unit", st[7] / max(st[4], 1))
print("issue-blocked per unit: S/dP", st[5] / max(st[4], 1), "grads", st[6] / max(st[4], 1),
      "(pair kernel: pure MMA ~640 / 768 cycles per unit)")
