"""TC path vs EXACT path (bit-exact to the reference) on identical bf16 inputs."""
import sys, json, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import paper_2604_15180_b200 as pa
from test_gpu_tc import inputs, run

def scan(N, alpha, D=128, causal=True, qs=1.0, seed=3):
    q, k, v, do = inputs(seed, 1, 1, N, D, qs)
    t0 = time.time()
    _, rx, gx = run(q, k, v, do, "exact", alpha=alpha, causal=causal)
    tx = time.time() - t0
    _, rt, gt = run(q, k, v, do, "tc", alpha=alpha, causal=causal)
    e = {n: (getattr(rt, n) - getattr(rx, n)).abs().max().item() for n in ("out", "tau")}
    e.update({n: (getattr(gt, n) - getattr(gx, n)).abs().max().item() for n in ("dq", "dk", "dv")})
    mags = {n: getattr(gx, n).abs().max().item() for n in ("dq", "dk", "dv")}
    print(json.dumps(dict(N=N, alpha=alpha, qs=qs, exact_s=round(tx, 2), err=e, mags=mags,
                          sparsity=rx.stats.block_sparsity)), flush=True)

def time_bwd(B=2, H=32, N=32768, D=128, alpha=1.5):
    q, k, v, do = inputs(1, B, H, N, D, 1.0)
    prob = pa.AttentionProblem(q, k, v, alpha=alpha, causal=True, path="tc")
    res = pa.forward(prob); g = pa.backward(prob, res, do); torch.cuda.synchronize()
    for _ in range(2):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(); res = pa.forward(prob); e1.record(); g = pa.backward(prob, res, do); e2.record()
        e2.synchronize()
        print("C3 fwd ms", e0.elapsed_time(e1), "bwd ms", e1.elapsed_time(e2), flush=True)

if __name__ == "__main__":
    time_bwd()
    for N in (2048, 8192):
        for alpha in (1.25, 1.5, 2.0):
            scan(N, alpha)
    scan(32768, 1.5)
    scan(32768, 2.0)
