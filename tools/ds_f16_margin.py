"""Dev check: fp16 dS (ADATTN_DS_F16=1) vs bf16 hi/lo dS gradients at long
context (the hi/lo path is within ~1e-4 of the reference, tests/test_gpu_oracle_tc.py).
    python tools/ds_f16_margin.py N alpha [beta]"""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2604_15180_b200 as pa
from paper_2604_15180_b200 import workloads
N, alpha = int(sys.argv[1]), float(sys.argv[2])
beta = float(sys.argv[3]) if len(sys.argv) > 3 else None
H = int(os.environ.get("H", "2"))
if beta is None:
    q, k, v, do = workloads.gaussian(1, H, N, 128, seed=5)
else:
    q, k, v, do = workloads.anchored(1, H, N, 128, beta, True, seed=5)
p = pa.AttentionProblem(q, k, v, alpha=alpha, causal=True)
r = pa.forward(p)
os.environ["ADATTN_DS_F16"] = "0"
g0 = pa.backward(p, r, do)
os.environ["ADATTN_DS_F16"] = "1"
g1 = pa.backward(p, r, do)
torch.cuda.synchronize()
for n in ("dq", "dk"):
    a, b = getattr(g0, n), getattr(g1, n)
    print(N, alpha, beta, n, "max|diff| %.2e" % (a - b).abs().max().item(), "max|g| %.1f" % a.abs().max().item(),
          "sparsity %.3f" % r.stats.block_sparsity)
