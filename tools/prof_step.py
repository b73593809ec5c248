"""One forward+backward at a given shape (for ncu captures): python tools/prof_step.py B H N D [beta]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2604_15180_b200 as pa
from paper_2604_15180_b200 import workloads
B, H, N, D = (int(x) for x in sys.argv[1:5])
beta = float(sys.argv[5]) if len(sys.argv) > 5 else None
if beta is None:
    q, k, v, do = workloads.gaussian(B, H, N, D, 1.0, seed=1)
else:
    q, k, v, do = workloads.anchored(B, H, N, D, beta, True, seed=1)
p = pa.AttentionProblem(q, k, v, alpha=1.5, causal=True)
r = pa.forward(p)
g = pa.backward(p, r, do)
torch.cuda.synchronize()
print("sparsity", r.stats.block_sparsity)
