"""Dev check: single-CTA vs CTA-pair forward on one case (diff rows, steps)."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2604_15180_b200 as pa
B, H, N = 1, 2, int(os.environ.get("N", "2048"))
g = torch.Generator(device="cpu").manual_seed(int(os.environ.get("SEED", "5")))
q, k, v = ((torch.randn(B, H, N, 128, generator=g)).to(torch.bfloat16).cuda() for _ in range(3))
res = {}
for pairs in ("0", "1"):
    os.environ["ADATTN_FWD_PAIRS"] = pairs
    p = pa.AttentionProblem(q, k, v, alpha=1.5, causal=True, path="tc")
    r = pa.forward(p); torch.cuda.synchronize()
    res[pairs] = r
rx = pa.forward(pa.AttentionProblem(q, k, v, alpha=1.5, causal=True, path="exact"))
a, b = res["0"], res["1"]
d = (a.tau - b.tau).abs()
print("single vs exact tau", (a.tau - rx.tau).abs().max().item(), "pair vs exact", (b.tau - rx.tau).abs().max().item())
bad = torch.nonzero(d > 1e-9)
print("rows differing", bad.shape[0], bad[:20].tolist())
if bad.shape[0]:
    r0 = bad[:, 2]
    print("rows mod 512", sorted(set((r0 % 512).tolist()))[:40])
    print("steps single", a.row_steps[0, 0][r0[:10]].tolist(), "pair", b.row_steps[0, 0][r0[:10]].tolist())
    print("tau single", a.tau[0, 0][r0[:10]].tolist(), "pair", b.tau[0, 0][r0[:10]].tolist())
print("mask equal", torch.equal(a.mask.words, b.mask.words), "out diff", (a.out - b.out).abs().max().item())
