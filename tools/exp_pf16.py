import sys, os
sys.path.insert(0, ".")
import torch
lib = sys.argv[1]
import paper_2604_15180_b200._lib as L
L.LIB_PATH = os.path.abspath(lib)
import paper_2604_15180_b200 as pa
sys.path.insert(0, "tests")
from test_gpu_tc import inputs, run
for case in [(1, 2, 512, 128, 1.5, True, 1.0), (2, 1, 768, 64, 2.0, True, 1.0), (1,1,2048,128,1.5,True,1.0)]:
    B, H, N, D, alpha, causal, qs = case
    q, k, v, do = inputs(7, B, H, N, D, qs)
    _, rx, _ = run(q, k, v, None, "exact", alpha=alpha, causal=causal)
    _, rt, _ = run(q, k, v, None, "tc", alpha=alpha, causal=causal)
    print(lib, case, "out err", (rt.out - rx.out).abs().max().item(), "tau err", (rt.tau-rx.tau).abs().max().item())
