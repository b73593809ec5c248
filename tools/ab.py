"""A/B timing of library variants / env settings, interleaved (dev tool).
    python tools/ab.py VARIANT [VARIANT ...]   VARIANT = path/to/lib.so[:ENV=VAL[,ENV=VAL]]
Runs the C3 forward (+backward with BWD=1; SHAPE=B,H,N D=.. CAUSAL=0/1 for other shapes) of each variant in turn, REPS rounds,
and prints the median ms per variant: interleaving cancels clock drift."""
import os, sys, statistics
sys.path.insert(0, ".")
import paper_2604_15180_b200._lib as L
import torch
import paper_2604_15180_b200 as pa
from paper_2604_15180_b200 import workloads

B, H, N = (int(x) for x in os.environ.get("SHAPE", "2,32,32768").split(","))
alpha = float(os.environ.get("ALPHA", "1.5"))
beta = os.environ.get("BETA")
reps = int(os.environ.get("REPS", "7"))
bwd = os.environ.get("BWD", "0") == "1"
D = int(os.environ.get("D", "128"))
causal = os.environ.get("CAUSAL", "1") == "1"
vars_ = []
for a in sys.argv[1:]:
    path, _, envs = a.partition(":")
    env = dict(kv.split("=", 1) for kv in envs.split(",") if kv)
    L.LIB_PATH = os.path.abspath(path)
    L._lib = None
    vars_.append((a, L.load(), env))
q, k, v, do = (workloads.gaussian(B, H, N, D, 1.0, seed=1) if beta is None
               else workloads.anchored(B, H, N, D, float(beta), causal, seed=1))
p = pa.AttentionProblem(q, k, v, alpha=alpha, causal=causal)
ts = {a: [] for a, _, _ in vars_}
kts = {a: {} for a, _, _ in vars_}
for rep in range(reps + 1):
    for a, lib, env in vars_:
        L._lib = lib
        old = {kk: os.environ.get(kk) for kk in env}
        os.environ.update(env)
        L.profile_read()
        L.profile_enable(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = pa.forward(p)
        if bwd:
            pa.backward(p, r, do)
        e1.record()
        e1.synchronize()
        L.profile_enable(False)
        kt = L.profile_read()
        if rep:
            for name, ms in kt:
                kts[a].setdefault(name, []).append(ms)
        for kk, vv in old.items():
            if vv is None:
                os.environ.pop(kk, None)
            else:
                os.environ[kk] = vv
        if rep:
            ts[a].append(e0.elapsed_time(e1))
base = None
for a, _, _ in vars_:
    m = statistics.median(ts[a])
    base = base or m
    print(f"{a:60s} median {m:8.2f} ms  ({m / base:.3f})  min {min(ts[a]):.2f} max {max(ts[a]):.2f}")
    print("    " + "  ".join(f"{k} {statistics.median(v):.2f}" for k, v in kts[a].items()))
