"""Loads the ADATTN_PIPE_STATS build (make -C paper_2604_15180_b200 stats) and
prints per-role wait fractions and per-phase cycle shares of the forward.
    python tools/pipe_stats.py B H N [beta]"""
import ctypes as C, os, sys
sys.path.insert(0, ".")
import paper_2604_15180_b200._lib as L
L.LIB_PATH = os.path.abspath(os.environ.get("LIB", "paper_2604_15180_b200/libadattn_b200_stats.so"))
import torch
import paper_2604_15180_b200 as pa
from paper_2604_15180_b200 import workloads
lib = L.load()
fn = lib.adattn_b200_pipe_stats
fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
B, H, N = (int(x) for x in sys.argv[1:4])
beta = float(sys.argv[4]) if len(sys.argv) > 4 else None
alpha = float(os.environ.get("ALPHA", "1.5"))
q, k, v, do = (workloads.gaussian(B, H, N, 128, 1.0, seed=1) if beta is None
               else workloads.anchored(B, H, N, 128, beta, True, seed=1))
p = pa.AttentionProblem(q, k, v, alpha=alpha, causal=True)
r = pa.forward(p); torch.cuda.synchronize()
buf = (C.c_ulonglong * 64)()
fn(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); r = pa.forward(p); e1.record(); e1.synchronize()
fn(buf, 1)
st = list(buf)
mma = max(st[6], 1)
names = ["mma_wait_full(TMA)", "mma_wait_s_empty(epi)", "mma_wait_p_full", "prod_wait_empty", "epi_w4_wait_s_full"]
print("fwd ms", e0.elapsed_time(e1), "sparsity", r.stats.block_sparsity, "ring items", st[7])
for i, n in enumerate(names):
    print(f"{n:26s} {st[i] / mma:6.3f} of MMA-warp cycles")
ph = ["MAX", "HIST", "CAND sweep", "list REF+mask", "REF sweeps", "OUT (S+PV)", "O/tau store"]
tot = sum(st[8:15]) or 1
for i, n in enumerate(ph):
    print(f"phase {n:16s} {100.0 * st[8 + i] / tot:5.1f}%")
for s, n in enumerate(["MAX", "HIST", "CAND", "REF/decision", "OUT (S+PV)"]):
    cyc, tiles = st[16 + 2 * s], st[17 + 2 * s]
    ideal = 1024 if s == 4 else 512
    if tiles:
        print(f"MMA sweep {n:13s} cycles/rg-tile {cyc / tiles:8.1f}  (ideal {ideal}) tiles {tiles}"
              f"  ring-wait/tile {st[32 + 2 * s] / tiles:7.1f}  S-buffer-wait/tile {st[33 + 2 * s] / tiles:7.1f}")
    else:
        print(f"MMA sweep {n:13s} cycles {cyc}")
print("MMA issue+commit cycles per rg-tile: MAX", st[44] / max(st[17], 1), "HIST+CAND", st[45] / max(st[19] + st[21], 1))
print("epilogue thread 0: TMEM ld32+wait cycles per load", st[46] / max(st[47], 1), "loads", st[47])
if st[27]:
    print(f"candidate lists: mean {st[26] / st[27]:.1f} entries/thread, longest {st[28]}, "
          f"overflowed threads {st[29]} of {st[27]}")
lm = ["wait all CAND", "staging+hist", "solve", "refine rounds", "mask", "tiles+decision"]
tl = sum(st[48:54]) or 1
print("list phase (thread 0 cycles per CTA):", "  ".join(f"{n} {st[48 + i] / max(st[27] / 512, 1):.0f}" for i, n in enumerate(lm)))
print("raw sweep waits [32..41]:", st[32:42])
