"""Event timeline of the forward's first CTA pair (build: make -C paper_2604_15180_b200
stats EXTRA=-DADATTN_PIPE_TRACE; dev tool).  python tools/trace.py LIB"""
import ctypes as C, os, sys, statistics
sys.path.insert(0, ".")
import paper_2604_15180_b200._lib as L
L.LIB_PATH = os.path.abspath(sys.argv[1])
import torch
import paper_2604_15180_b200 as pa
from paper_2604_15180_b200 import workloads
lib = L.load()
rd = lib.adattn_b200_trace_read
rd.restype = C.c_uint
rd.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
B, H, N = 2, 32, 32768
q, k, v, do = workloads.gaussian(B, H, N, 128, 1.0, seed=1)
p = pa.AttentionProblem(q, k, v, alpha=1.5, causal=True)
pa.forward(p); torch.cuda.synchronize()
rd(None, 1)
pa.forward(p); torch.cuda.synchronize()
n = rd(None, 0)
buf = (C.c_ulonglong * n)()
rd(buf, 1)
ev = []  # (t, role, type, J)
for i, x in enumerate(buf):
    if x:
        ev.append((x & 0xFFFFFFFFFF, i >> 12, x >> 56, (x >> 40) & 0xFFFF))
ev.sort()
t0 = ev[0][0]
# release lag: per tile J of the HIST sweep (2nd pass over J), per (cta, warp) release time
# relative to the earliest release of that J by any warp of that row group
sweep = int(os.environ.get("SWEEP", "1"))
rel = {}
for t, role, ty, j in ev:
    if ty in (8, 9):
        rel.setdefault((ty - 8, j), []).append((t, role))
# keep only the sweep-th occurrence block: each (rg, J) appears once per sweep per warp
lags = {}
for (rg, j), lst in rel.items():
    per = {}
    for t, role in lst:
        per.setdefault(role, []).append(t)
    for role, ts in per.items():
        if len(ts) > sweep:
            lags.setdefault((rg, j), {})[role] = ts[sweep]
agg = {}
for key, d in lags.items():
    if len(d) < 8:
        continue
    m = min(d.values())
    for role, t in d.items():
        agg.setdefault(role, []).append(t - m)
print("median release lag (ns) behind the first releasing warp, per warp (role: cta*32 + 2 + warp)")
for role in sorted(agg):
    print(f"  cta {role // 32} warp {role % 32 - 2:2d}: {statistics.median(agg[role]):7.0f}  max {max(agg[role]):7.0f}")
# MMA: s_empty-ready minus ring-ready per tile (ns), sweep-th occurrence
def occ(ty, role):
    d = {}
    for t, r, tt, j in ev:
        if tt == ty and r == role:
            d.setdefault(j, []).append(t)
    return {j: ts[sweep] for j, ts in d.items() if len(ts) > sweep}
ring, semp = occ(2, 1), occ(3, 1)
w = [semp[j] - ring[j] for j in ring if j in semp]
print("MMA s_empty wait after ring ready: median", statistics.median(w), "ns")
iv = sorted(ring.values())
print("tile interval median", statistics.median([b - a for a, b in zip(iv, iv[1:])]), "ns")
# latency from the last release of tile J (any warp, either CTA, both row groups)
# to the MMA warp passing its s_empty wait for tile J+2
last_rel = {}
for (rg, j), d in lags.items():
    last_rel[j] = max(last_rel.get(j, 0), max(d.values()))
lat = [semp[j + 2] - last_rel[j] for j in last_rel if j + 2 in semp]
print("s_empty(J+2) pass - last release(J): median", statistics.median(lat), "ns  p10", sorted(lat)[len(lat)//10], "p90", sorted(lat)[9*len(lat)//10])
# per-CTA last release
for c in (0, 1):
    lr = {}
    for (rg, j), d in lags.items():
        v = [t for r, t in d.items() if r // 32 == c]
        if v:
            lr[j] = max(lr.get(j, 0), max(v))
    lat = [semp[j + 2] - lr[j] for j in lr if j + 2 in semp]
    print(f"  vs CTA {c} last release: median", statistics.median(lat))
iss0, iss1, prod = occ(4, 1), occ(5, 1), occ(1, 0)
sf = {}
for (rg, j), d in lags.items():
    pass
full0 = {}
for t, r, tt, j in ev:
    if tt in (6, 7):
        full0.setdefault((tt - 6, j, r), []).append(t)
print("   J   ring  sempty  iss0  iss1 | rel(J-2) min..max rg0 / rg1 | sfull(J) rg0 rg1 (cta0 warp0/8)")
js = sorted(ring)
mid = js[len(js) // 3: len(js) // 3 + 12]
base = ring[mid[0]]
for j in mid:
    r0 = lags.get((0, j - 2), {}); r1 = lags.get((1, j - 2), {})
    f0 = full0.get((0, j, 2), [None] * 9); f1 = full0.get((1, j, 10), [None] * 9)
    f0 = f0[sweep] - base if len(f0) > sweep and f0[sweep] else -1
    f1 = f1[sweep] - base if len(f1) > sweep and f1[sweep] else -1
    print(f"{j:4d} {ring[j]-base:6d} {semp.get(j,0)-base:6d} {iss0.get(j,0)-base:6d} {iss1.get(j,0)-base:6d} | "
          f"{min(r0.values())-base if r0 else 0:6d}..{max(r0.values())-base if r0 else 0:6d} / "
          f"{min(r1.values())-base if r1 else 0:6d}..{max(r1.values())-base if r1 else 0:6d} | {f0:6d} {f1:6d}")

pre0, pre1, post0, post1 = occ(12, 1), occ(13, 1), occ(14, 1), occ(15, 1)
print("   J   ring  pre0  post0  pre1  post1  sempty")
for j in mid:
    print(f"{j:4d} {ring[j]-base:6d} {pre0.get(j,0)-base:6d} {post0.get(j,0)-base:6d} {pre1.get(j,0)-base:6d} {post1.get(j,0)-base:6d} {semp.get(j,0)-base:6d}")
