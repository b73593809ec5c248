"""Dev timing of a BASELINE config shape (fwd+bwd, per-kernel medians).
    python tools/cfg_time.py B H N D causal(0/1) [alpha]"""
import sys, statistics, torch
sys.path.insert(0, ".")
import paper_2604_15180_b200 as pa
import paper_2604_15180_b200._lib as L
from paper_2604_15180_b200 import workloads
B, H, N, D, causal = (int(x) for x in sys.argv[1:6])
alpha = float(sys.argv[6]) if len(sys.argv) > 6 else 1.5
q, k, v, do = workloads.gaussian(B, H, N, D, 1.0, seed=1)
p = pa.AttentionProblem(q, k, v, alpha=alpha, causal=bool(causal))
r = g = None
for _ in range(3):
    r = pa.forward(p); g = pa.backward(p, r, do)
torch.cuda.synchronize()
ts, kts = [], {}
for _ in range(5):
    L.profile_read(); L.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); r = pa.forward(p); g = pa.backward(p, r, do); e1.record(); e1.synchronize()
    L.profile_enable(False)
    for n, ms in L.profile_read(): kts.setdefault(n, []).append(ms)
    ts.append(e0.elapsed_time(e1))
T = N // 64
nnz = r.stats.blocks_visited_fwd
feff = 14.0 * D * 4096 * nnz
m = statistics.median(ts)
print(f"B={B} H={H} N={N} d={D} causal={causal} alpha={alpha}: {m:.2f} ms, eff {feff / m / 1e9:.0f} TFLOP/s, sparsity {r.stats.block_sparsity:.3f}",
      {n: round(statistics.median(v), 2) for n, v in kts.items()})
