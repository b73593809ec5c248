"""Bitwise comparison of one library under two env settings (dev tool).
    ENV_A=K=V ENV_B=K=V [LIB_B=path.so] python tools/bitcmp.py
Runs forward + backward (SHAPE=B,H,N D=.. ALPHA=.. CAUSAL=..) under each setting and reports
whether out / dq / dk / dv are bit-identical."""
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2604_15180_b200._lib as L
import paper_2604_15180_b200 as pa
from paper_2604_15180_b200 import workloads

B, H, N = (int(x) for x in os.environ.get("SHAPE", "1,8,32768").split(","))
D = int(os.environ.get("D", "128"))
alpha = float(os.environ.get("ALPHA", "1.5"))
causal = os.environ.get("CAUSAL", "1") == "1"
q, k, v, do = workloads.gaussian(B, H, N, D, 1.0, seed=3)
p = pa.AttentionProblem(q, k, v, alpha=alpha, causal=causal)
outs = []
for tag in ("ENV_A", "ENV_B"):
    kv = os.environ.get(tag, "")
    if tag == "ENV_B" and os.environ.get("LIB_B"):
        L.LIB_PATH = os.path.abspath(os.environ["LIB_B"])
        L._lib = None
    old = {}
    for item in filter(None, kv.split(",")):
        kk, vv = item.split("=", 1)
        old[kk] = os.environ.get(kk)
        os.environ[kk] = vv
    r = pa.forward(p)
    g = pa.backward(p, r, do)
    torch.cuda.synchronize()
    outs.append([r.out.clone()] + [t.clone() for t in (g.dq, g.dk, g.dv)])
    for kk, vv in old.items():
        if vv is None:
            os.environ.pop(kk, None)
        else:
            os.environ[kk] = vv
for name, a, b in zip(("out", "dq", "dk", "dv"), outs[0], outs[1]):
    print(name, "bit-identical" if torch.equal(a, b) else f"DIFFERENT max {(a - b).abs().max().item():.3e}")
