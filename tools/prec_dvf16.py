"""Dev check: fp16 gradient products (ADATTN_DV_F16 / ADATTN_DS_F16) vs the bf16
hi/lo products and vs the exact path (max-abs), at N=32K and N=4096."""
import os, sys, torch
sys.path.insert(0, ".")
import paper_2604_15180_b200 as pa
from paper_2604_15180_b200 import workloads
for (B, H, N, alpha) in [(1, 4, 32768, 1.5), (1, 4, 32768, 2.0), (1, 2, 32768, 1.25), (1, 2, 32768, 1.75)]:
    q, k, v, do = workloads.gaussian(B, H, N, 128, 1.0, seed=3)
    p = pa.AttentionProblem(q, k, v, alpha=alpha, causal=True)
    r = pa.forward(p)
    os.environ["ADATTN_DV_F16"] = "0"; os.environ["ADATTN_DS_F16"] = "0"; g0 = pa.backward(p, r, do)
    os.environ["ADATTN_DV_F16"] = "1"; os.environ["ADATTN_DS_F16"] = "1"; g1 = pa.backward(p, r, do)
    torch.cuda.synchronize()
    for n in ("dv", "dk", "dq"):
        a, b = getattr(g0, n), getattr(g1, n)
        print(B, H, N, alpha, n, "f16 vs hilo maxabs", f"{(a - b).abs().max().item():.3e}", "max|x|", f"{a.abs().max().item():.2f}")
