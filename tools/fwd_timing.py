"""Dev timing of the TC forward alone (CUDA events); not the bench contract."""
import sys, time, json
import torch
sys.path.insert(0, ".")
import paper_2604_15180_b200 as pa

def run(B, H, N, D, alpha=1.5, causal=True, qscale=1.0, reps=3):
    torch.manual_seed(0)
    q = (qscale * torch.randn(B, H, N, D, device="cuda")).bfloat16()
    k = torch.randn(B, H, N, D, device="cuda").bfloat16()
    v = torch.randn(B, H, N, D, device="cuda").bfloat16()
    prob = pa.AttentionProblem(q, k, v, alpha=alpha, causal=causal, path="tc")
    res = pa.forward(prob)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); res = pa.forward(prob); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    T = N // 64
    A = T * (T + 1) // 2 if causal else T * T
    st = res.stats
    nnz = st.blocks_visited_fwd
    steps = res.row_steps.float().mean().item()
    # fwd flops: (2 + R) dense QK passes over A blocks + QK + PV over nnz
    R = 3
    f_dense = 2 * D * 4096 * (2 + R) * A * B * H
    f_out = 4 * D * 4096 * nnz
    ms = min(ts)
    print(json.dumps(dict(B=B, H=H, N=N, D=D, alpha=alpha, ms=ms, sparsity=st.block_sparsity,
                          steps=steps, tflops_alg=(f_dense + f_out) / ms / 1e9)))

if __name__ == "__main__":
    run(4, 16, 8192, 128)
    run(2, 32, 32768, 128)
    run(2, 32, 32768, 128, qscale=8.0)
