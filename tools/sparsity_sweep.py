"""F_eff against block sparsity for alpha in {1.25, 1.5, 2} at the C3 per-head
shape (SURVEY 7.7 / VERDICT r1 item 6): for each alpha and target sparsity,
beta of the anchored generator is calibrated by bisection on the MEASURED mask
sparsity (forward only, B=1 H=2), then the full C3 batch (B=2 H=32 N=32768 d=128,
causal) is timed fwd+bwd (CUDA events, median of --reps after 2 warm-ups).
    python tools/sparsity_sweep.py [--out profiles/r2_sparsity_sweep.json]"""
import argparse, json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15180_b200 as pa
from paper_2604_15180_b200 import workloads

N, D = 32768, 128


def sparsity_at(alpha, beta, heads=2):
    if beta is None:
        q, k, v, _ = workloads.gaussian(1, heads, N, D, 1.0, seed=7)
    else:
        q, k, v, _ = workloads.anchored(1, heads, N, D, beta, True, seed=7)
    r = pa.forward(pa.AttentionProblem(q, k, v, alpha=alpha, causal=True))
    return r.stats.block_sparsity


def calibrate(alpha, target, lo=0.0, hi=2.0, iters=9):
    s_lo = sparsity_at(alpha, lo)
    if target <= s_lo + 0.02:
        return lo, s_lo
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        s = sparsity_at(alpha, mid)
        if s < target:
            lo = mid
        else:
            hi = mid
    b = 0.5 * (lo + hi)
    return b, sparsity_at(alpha, b)


def timed(alpha, beta, reps):
    q, k, v, do = workloads.anchored(2, 32, N, D, beta, True, seed=11)
    p = pa.AttentionProblem(q, k, v, alpha=alpha, causal=True)
    for _ in range(2):
        r = pa.forward(p)
        pa.backward(p, r, do)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = pa.forward(p)
        pa.backward(p, r, do)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    st = r.stats
    ms = statistics.median(ts)
    f_eff = 14.0 * D * 4096 * st.blocks_visited_fwd
    exe = workloads.executed_flops(r.mask.words, N, D, True, alpha=alpha, row_steps=r.row_steps)
    return dict(alpha=alpha, beta=beta, block_sparsity=st.block_sparsity, ms=ms,
                tflops_eff=f_eff / (ms * 1e-3) / 1e12,
                tflops_executed=sum(exe.values()) / (ms * 1e-3) / 1e12,
                tau_iters_avg=r.row_steps.float().mean().item(), reps=reps)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r2_sparsity_sweep.json")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--alphas", default="1.25,1.5,2")
    ap.add_argument("--targets", default="0,0.2,0.4,0.6,0.8,0.95")
    a = ap.parse_args()
    rows = []
    for alpha in (float(x) for x in a.alphas.split(",")):
        for tgt in (float(x) for x in a.targets.split(",")):
            beta, s_cal = calibrate(alpha, tgt)
            row = timed(alpha, beta, a.reps)
            row.update(target=tgt, calibrated_sparsity=s_cal)
            rows.append(row)
            print(json.dumps(row), flush=True)
    with open(a.out, "w") as f:
        json.dump({"shape": "C3: B=2 H=32 N=32768 d=128 causal bf16, anchored inputs (SURVEY 7.7)",
                   "note": "beta calibrated per alpha by bisection on the measured sparsity (B=1 H=2, "
                           "forward only); F_eff = 14 d 4096 nnz (SURVEY 8d)", "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
