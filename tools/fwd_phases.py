"""Per-phase forward timings (PhaseTimings via adattn_b200_forward_timed) of
library variants at C3, interleaved (dev tool).
    python tools/fwd_phases.py LIB [LIB ...]"""
import os, sys, statistics
sys.path.insert(0, ".")
import paper_2604_15180_b200._lib as L
import torch
import paper_2604_15180_b200 as pa
from paper_2604_15180_b200 import workloads

B, H, N = (int(x) for x in os.environ.get("SHAPE", "2,32,32768").split(","))
alpha = float(os.environ.get("ALPHA", "1.5"))
beta = os.environ.get("BETA")
reps = int(os.environ.get("REPS", "5"))
libs = []
for path in sys.argv[1:]:
    L.LIB_PATH = os.path.abspath(path)
    L._lib = None
    libs.append((path, L.load()))
q, k, v, do = (workloads.gaussian(B, H, N, 128, 1.0, seed=1) if beta is None
               else workloads.anchored(B, H, N, 128, float(beta), True, seed=1))
p = pa.AttentionProblem(q, k, v, alpha=alpha, causal=True)
res = {a: [] for a, _ in libs}
for rep in range(reps + 1):
    for a, lib in libs:
        L._lib = lib
        t = pa.PhaseTimings()
        pa.forward(p, timings=t)
        torch.cuda.synchronize()
        if rep:
            res[a].append(t.ms)
for a, _ in libs:
    ms = [statistics.median(x[i] for x in res[a]) for i in range(4)]
    print(f"{a:50s} total {sum(ms):7.2f} ms  max {ms[0]:6.2f}  hist/cand {ms[1]:6.2f}  "
          f"refine {ms[2]:6.2f}  out {ms[3]:6.2f}")
