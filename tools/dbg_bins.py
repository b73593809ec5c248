"""Dev check: TC vs EXACT tau for one (bins, alpha) case, optional library path."""
import os, sys
sys.path.insert(0, ".")
import paper_2604_15180_b200._lib as L
if len(sys.argv) > 3:
    L.LIB_PATH = os.path.abspath(sys.argv[3])
import torch
import paper_2604_15180_b200 as pa
bins, alpha = int(sys.argv[1]), float(sys.argv[2])
g = torch.Generator(device="cpu").manual_seed(100 + bins)
q, k, v = ((torch.randn(1, 2, 1024, 128, generator=g)).to(torch.bfloat16).cuda() for _ in range(3))
rx = pa.forward(pa.AttentionProblem(q, k, v, alpha=alpha, causal=True, bins=bins, path="exact"))
rt = pa.forward(pa.AttentionProblem(q, k, v, alpha=alpha, causal=True, bins=bins, path="tc"))
torch.cuda.synchronize()
d = (rt.tau - rx.tau).abs()
print(L.LIB_PATH[-30:], bins, alpha, "max", d.max().item(), "rows>1e-5", int((d > 1e-5).sum()),
      "first", torch.nonzero(d > 1e-5)[:5].tolist())
