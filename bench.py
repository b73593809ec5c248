#!/usr/bin/env python
"""Benchmark of the alpha-entmax attention hot path (fwd + bwd) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--gpus N` (N > 1) re-executes itself under torch.distributed.run with N local
ranks when it is not already running under torchrun (the driver's launch).

Workload (BASELINE.json configs[2], the config the metric is quoted on): alpha=1.5,
causal, B=2 H=32 N=32768 d=128, bf16 inputs (synthetic, cmd_attn's N(0,1)
distribution, one generator seed per head).  The B*H = 64 heads are independent
problems: rank r of N runs the contiguous head shard
parallel.shard_heads(64, N, r) with no collective on the path (fixed total work
-> "scaling": "strong").  A "step" = forward + backward over the rank's heads.
`value` = effective TFLOP/s over the non-zero 64x64 blocks of all heads
(F_eff = 14 d 4096 nnz) / max-over-ranks step time.  Inputs
(4 x 512 MiB at N=1) exceed the 126 MB L2, so no explicit flush.
`e2e` = the same metric through the C-ABI host entry (adattn_b200_run_host) with
pinned host buffers: H2D of q/k/v/dO and D2H of out/dq/dk/dv/tau/row_max/delta/mask
inside the timed region, over --steps steps.  `validation` = per-head digests
gathered once over NVLink and compared with a 1-GPU run of all heads on rank 0.
`sweep` / `alpha_sweep` = the same step on the anchored generator (block
sparsity 0..~99%) and at alpha 1.25 / 2.
`--impl reference` = the reference's own CPU forward+backward (oracle/_ref) on
one head of the same per-head shape per step, all host threads.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("entmax attn fwd+bwd ms & effective TFLOP/s vs block sparsity (N=32K); "
          "avg τ iters")
UNIT = "TFLOP/s"


def peaks():
    """Roofline denominators (B200_PROFILING.md / MEASURED_PEAKS.json): the burst
    dense-bf16 figure (the larger of the two measured peaks, so `frac` is the
    conservative reading -- several of these kernels exceed the 4-second sustained
    matmul figure inside the ~0.1 s step), else the sustained one, else the
    recipe's fallback (1.59 PF burst)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        bw = float(p.get("hbm_gbs", 6542.4))
        if p.get("bf16_tflops"):
            return float(p["bf16_tflops"]), bw, "measured burst"
        return float(p["bf16_tflops_sustained"]), bw, "measured sustained"
    except Exception:
        return 1590.0, 6650.0, "fallback burst"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for i, nm in enumerate(names):
                if len(s) > 3 + i and s[3 + i].lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ launcher
def self_launch(args) -> None:
    """`bench.py --gpus N` (N > 1) outside torchrun: re-exec under
    torch.distributed.run with N local ranks (127.0.0.1 rendezvous)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def nccl_init_lines(path_pattern: str):
    """The communicator-init lines NCCL_DEBUG=INFO wrote for this process (proof of
    the rank count)."""
    import glob
    out = []
    for p in glob.glob(path_pattern):
        try:
            with open(p) as f:
                out += [ln.strip() for ln in f if "Init COMPLETE" in ln or "nRanks" in ln]
        except OSError:
            pass
    return out[:4]


# ------------------------------------------------------------------ CPU side
def cpu_reference_step(n, d, alpha, causal, head=0, threads=None, kind="reference"):
    """One fwd+bwd of the reference CPU implementation (oracle/_ref, compiled from the
    reference sources, stock adattn::forward / adattn::backward) on ONE head of the
    workload: cmd_attn's inputs (atn_main.cpp:227-232) for seed 1 + head, rounded to
    bf16 like the GPU arm's, promoted to double.  Timed like cmd_attn times it
    (atn_main.cpp:239-247: forward and backward back to back)."""
    import numpy as np
    from oracle.oracle import Oracle, Problem, gen_attn_inputs
    orc = Oracle(kind)
    threads = threads or os.cpu_count() or 1
    q, k, v, do = gen_attn_inputs(1 + head, n, d, 1.0, orc)

    def bf16(x):  # round-to-nearest-even to bf16, as torch does for the GPU arm
        u = x.astype(np.float32).view(np.uint32)
        u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
        return u.view(np.float32).astype(np.float64)

    q, k, v, do = (bf16(x) for x in (q, k, v, do))
    pb = Problem(q, k, v, alpha=alpha, causal=causal)
    t0 = time.perf_counter()
    f = orc.forward(pb, threads)
    orc.backward(pb, f, do, threads)
    dt = time.perf_counter() - t0
    nnz = f["blocks_visited_fwd"]
    return dict(seconds=dt, nnz=nnz, tflops=14.0 * d * 4096 * nnz / dt / 1e12, threads=threads,
                sparsity=f["block_sparsity"])


def run_reference_arm(args):
    """The reference's own CPU implementation on the GPU arm's per-head workload
    (BASELINE config 3 head: N=32768, d=128, alpha=1.5, causal, bf16-valued
    N(0,1) inputs), all host threads.  One step = forward + backward of one
    head (a bounded sample of the 64-head job; throughput = the same
    effective-TFLOP/s metric, which is per-unit-work and so like-for-like)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    from paper_2604_15180_b200 import workloads
    cfg = dict(workloads.CONFIGS[args.config])
    if args.alpha is not None:
        cfg["alpha"] = args.alpha
    n = args.ref_n or cfg["N"]
    kw = dict(n=n, d=cfg["D"], alpha=cfg["alpha"], causal=cfg["causal"])
    heads = cfg["B"] * cfg["H"]
    budget = float(os.environ.get("ADATTN_REF_BUDGET_S", "1500"))
    t_start = time.perf_counter()
    # warm-up steps on other heads; if the projected run would overrun the arm's
    # time budget (ADATTN_REF_BUDGET_S), fewer warm-up / timed steps run and the line
    # says so (warmup / steps vs *_requested)
    warm = []
    for w in range(args.warmup):
        warm.append(cpu_reference_step(head=heads - 1 - (w % heads), **kw)["seconds"])
        left = budget - (time.perf_counter() - t_start)
        if left < (args.steps + 1) * warm[-1]:
            break
    per = warm[-1] if warm else None
    steps = args.steps
    if per:
        steps = max(1, min(args.steps, int((budget - (time.perf_counter() - t_start)) / per)))
    vals, secs, rs = [], [], []
    for s in range(steps):
        r = cpu_reference_step(head=s % heads, **kw)
        vals.append(r["tflops"])
        secs.append(r["seconds"])
        rs.append(r)
    tot_flops = sum(14.0 * kw["d"] * 4096 * r["nnz"] for r in rs)
    v = tot_flops / sum(secs) / 1e12
    sample = (f"{steps} of the {heads} heads of {args.config} (one head per step: N={n}, "
              f"d={kw['d']}, alpha={kw['alpha']}, causal={kw['causal']}, bf16-valued N(0,1) "
              f"inputs), the reference's forward+backward (oracle/_ref, -O3) on "
              f"{rs[0]['threads']} threads, {sum(secs) / steps:.1f} s per head")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
            "n_gpus": args.gpus, "steps": steps, "steps_requested": args.steps,
            "warmup": len(warm), "warmup_requested": args.warmup,
            "ms_per_step": 1000.0 * sum(secs) / steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} per-head sample", "B": cfg["B"],
                       "H": cfg["H"], "N": n, "d": kw["d"], "alpha": kw["alpha"],
                       "causal": kw["causal"], "heads_per_step": 1,
                       "same_per_head_config_as_gpu_arm": n == cfg["N"]},
            "block_sparsity": sum(r["sparsity"] for r in rs) / steps,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": rs[0]["threads"],
                             "kind": "reference", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU side
def head_digest(res, g):
    """Per-head fingerprint of a fwd+bwd result: [heads, 8] fp64 --
    sum tau, mask popcount, sum|out|, sum|dq|, sum|dk|, sum|dv|, sum delta, sum row_max."""
    import torch
    hc = res.tau.shape[0] * res.tau.shape[1]
    w = res.mask.words.reshape(hc, -1).view(torch.int32)
    pop = ((w.unsqueeze(-1) >> torch.arange(32, device=w.device)) & 1).sum(dim=(1, 2))
    f = lambda t: t.reshape(hc, -1).double()
    return torch.stack([f(res.tau).sum(1), pop.double(), f(res.out).abs().sum(1),
                        f(g.dq).abs().sum(1), f(g.dk).abs().sum(1), f(g.dv).abs().sum(1),
                        f(g.delta).sum(1), f(res.row_max).sum(1)], dim=1)


def gather_digests(dig, total, world, rank):
    """All ranks' per-head digests in global head order on rank 0 (one collective,
    outside the timed region); shards differ in size by at most one head."""
    import torch
    from paper_2604_15180_b200 import parallel
    width = -(-total // world)
    pad = torch.full((width, dig.shape[1]), float("nan"), dtype=torch.float64,
                     device=dig.device)
    pad[:dig.shape[0]] = dig
    allp = parallel.gather_to_rank0(pad.unsqueeze(0))
    if rank != 0:
        return None
    rows = []
    for r in range(world):
        _, c = parallel.shard_heads(total, world, r)
        rows.append(allp[r, :c])
    return torch.cat(rows, 0)


def compare_digests(sharded, single):
    import torch
    same = bool(torch.equal(sharded, single))
    rel = ((sharded - single).abs() / single.abs().clamp_min(1e-30)).max().item()
    return {"heads": int(sharded.shape[0]), "bitwise_equal_to_1gpu_run": same,
            "max_rel_diff": rel}


def plumbing_check(args, world, rank):
    """--plumbing-check: the multi-rank host path (sharding, per-head inputs,
    digest gather, comparison with a single-rank recomputation, max-over-ranks
    timing) with a stand-in per-head digest of the INPUTS instead of the GPU
    kernels -- runs under gloo on a CPU-only box (tests/test_parallel.py)."""
    import torch
    from paper_2604_15180_b200 import parallel, workloads
    B, H, N, D = 2, 3, 128, 16
    total = B * H
    h0, hc = parallel.shard_heads(total, world, rank)
    q, k, v, do = workloads.gaussian_heads(range(h0, h0 + hc), N, D, seed=7, device="cpu",
                                           dtype=torch.float32)
    dig = torch.stack([q.reshape(hc, -1).double().sum(1), k.reshape(hc, -1).double().sum(1),
                       v.reshape(hc, -1).double().abs().sum(1),
                       do.reshape(hc, -1).double().abs().sum(1)], 1)
    allg = gather_digests(dig, total, world, rank)
    ms = parallel.max_over_ranks(1.0 + rank)
    if rank == 0:
        q1, k1, v1, d1 = workloads.gaussian_heads(range(total), N, D, seed=7, device="cpu",
                                                  dtype=torch.float32)
        ref = torch.stack([q1.reshape(total, -1).double().sum(1),
                           k1.reshape(total, -1).double().sum(1),
                           v1.reshape(total, -1).double().abs().sum(1),
                           d1.reshape(total, -1).double().abs().sum(1)], 1)
        print(json.dumps({"plumbing_check": True, "n_ranks": world, "max_over_ranks": ms,
                          "shards": [parallel.shard_heads(total, world, r) for r in range(world)],
                          "validation": compare_digests(allg, ref)}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--alpha", type=float, default=None)
    ap.add_argument("--qscale", type=float, default=1.0)
    ap.add_argument("--sweep", default="0.6,0.7,0.8,1.0",
                    help="anchored-generator betas ('' to skip)")
    ap.add_argument("--alphas", default="1.25,2.0",
                    help="extra alphas timed on the headline shape (comma list, '' = none)")
    ap.add_argument("--sweep-steps", type=int, default=None,
                    help="timed steps per sweep point (default: --steps)")
    ap.add_argument("--ref-n", type=int, default=0, help="CPU sample rows (0: the config's N)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-validate", action="store_true")
    ap.add_argument("--plumbing-check", action="store_true",
                    help="multi-rank host path only (gloo, no GPU kernels)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)  # does not return
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.plumbing_check:
        if world > 1:
            dist.init_process_group("gloo")
        try:
            return plumbing_check(args, world, rank)
        finally:
            if world > 1:
                dist.destroy_process_group()

    import paper_2604_15180_b200 as pa
    from paper_2604_15180_b200 import _lib, parallel, workloads

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl_log = None
    if world > 1:
        if "NCCL_DEBUG" not in os.environ:
            import tempfile
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
            nccl_log = os.path.join(tempfile.gettempdir(), f"adattn_nccl.{os.getpid()}.log")
            os.environ["NCCL_DEBUG_FILE"] = nccl_log
        dist.init_process_group("nccl", device_id=dev)
        dist.barrier()

    cfg = dict(workloads.CONFIGS[args.config])
    if args.alpha is not None:
        cfg["alpha"] = args.alpha
    B, H, N, D = cfg["B"], cfg["H"], cfg["N"], cfg["D"]
    alpha, causal, dtype = cfg["alpha"], cfg["causal"], cfg["dtype"]
    total = B * H
    # B x H heads are independent problems: contiguous shards, no collective on the path
    h0, hc = parallel.shard_heads(total, world, rank)
    heads = range(h0, h0 + hc)
    q, k, v, do = workloads.gaussian_heads(heads, N, D, args.qscale, seed=1000, device=dev,
                                           dtype=dtype)
    prob = pa.AttentionProblem(q, k, v, alpha=alpha, causal=causal)
    resolved = {_lib.PATH_TC: "tc", _lib.PATH_EXACT: "exact"}[
        pa.attention.resolved_path(prob.c_problem())]

    def step(p, dout):
        r = pa.forward(p)
        g = pa.backward(p, r, dout)
        return r, g

    def timed(p, dout, warm, steps, profile=False):
        # warm-up holds the previous step's results exactly like the timed loop, so the
        # caching allocator owns both result sets before timing
        res = g = None
        for _ in range(warm):
            res, g = step(p, dout)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        if profile:
            _lib.profile_read()  # clear
            _lib.profile_enable(True)
        l0 = _lib.load().adattn_b200_launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            res, g = step(p, dout)
        e1.record()
        torch.cuda.synchronize()
        launches = _lib.load().adattn_b200_launch_count() - l0
        kt = []
        if profile:
            _lib.profile_enable(False)
            kt = _lib.profile_read()
        if world > 1:
            dist.barrier()
        ms = parallel.max_over_ranks(e0.elapsed_time(e1) / steps, device=dev)
        return ms, res, g, launches, kt

    clk = ClockSampler(local)
    clk.start()
    ms, res, grads, launches, ktimes = timed(prob, do, args.warmup, args.steps, profile=True)
    clocks = clk.stop()

    st = res.stats
    T = N // 64
    A_head = T * (T + 1) // 2 if causal else T * T
    nnz_rank = st.blocks_visited_fwd
    nnz_all = int(parallel.sum_over_ranks(nnz_rank, device=dev))
    steps_sum = parallel.sum_over_ranks(res.row_steps.double().sum().item(), device=dev)
    tau_iters = steps_sum / (total * N)
    fl = workloads.flops(D, nnz_all, A_head * total)
    value = fl["f_eff"] / (ms * 1e-3) / 1e12
    tflops_alg = fl["f_alg"] / (ms * 1e-3) / 1e12
    sparsity = 1.0 - nnz_all / (A_head * total)

    # ---- validation (outside the timed region): per-head digests gathered once over
    # NVLink, compared with a single-GPU run of all heads on rank 0
    validation = None
    if not args.no_validate:
        dig = head_digest(res, grads)
        allg = gather_digests(dig, total, world, rank)
        if rank == 0:
            if world > 1:
                q1, k1, v1, d1 = workloads.gaussian_heads(range(total), N, D, args.qscale,
                                                          seed=1000, device=dev, dtype=dtype)
                p1 = pa.AttentionProblem(q1, k1, v1, alpha=alpha, causal=causal)
                r1, g1 = step(p1, d1)
                validation = compare_digests(allg, head_digest(r1, g1))
                del q1, k1, v1, d1, p1, r1, g1
            else:
                validation = {"heads": int(allg.shape[0]), "all_finite":
                              bool(torch.isfinite(allg).all())}
            validation["tau_sum"] = float(allg[:, 0].sum())
            validation["mask_popcount"] = int(allg[:, 1].sum())

    # ---- per-kernel breakdown (CUDA events on the launching stream, timed region)
    agg = {}
    for name, t in ktimes:
        a = agg.setdefault(name, [0.0, 0])
        a[0] += t
        a[1] += 1
    kern = {n: {"ms_avg": a[0] / a[1], "launches": a[1]} for n, a in agg.items()}
    peak_tf, peak_bw, peak_kind = peaks()
    fl_rank = workloads.flops(D, nnz_rank, A_head * hc)
    # per launch of each tensor-core kernel: (a) the tcgen05 MMA flops it executes
    # (roofline numerator, workloads.executed_flops) and (b) the algorithmic count of
    # SURVEY 8(d) (reference algorithm: 2+R dense passes, no hi/lo halves)
    exe = workloads.executed_flops(res.mask.words, N, D, causal, alpha=alpha,
                                   row_steps=res.row_steps)
    per_alg = {"tc_fwd": fl_rank["f_fwd"], "tc_delta": 4.0 * D * 4096 * nnz_rank,
               "tc_dq": 6.0 * D * 4096 * nnz_rank, "tc_dkdv": 8.0 * D * 4096 * nnz_rank}
    dom = max(kern, key=lambda n: kern[n]["ms_avg"] * kern[n]["launches"]) if kern else None
    roofline = None
    for n in kern:
        if n in exe and exe[n] > 0:
            kern[n]["tflops_executed"] = exe[n] / (kern[n]["ms_avg"] * 1e-3) / 1e12
            kern[n]["frac_executed"] = kern[n]["tflops_executed"] / peak_tf
            kern[n]["tflops_alg"] = per_alg[n] / (kern[n]["ms_avg"] * 1e-3) / 1e12
        elif n == "tc_delta" and n in exe and res.delta_aux is not None:
            if alpha == 2.0 and os.environ.get("ADATTN_DELTA_SUPP", "1") == "0":
                # delta fold: delta = dO . Ubar / sum u, one HBM-bound pass per row -- reads
                # dO (bf16), Ubar (fp32), sum u, tau, m; writes delta (fp64), rowc (2 x fp32)
                b = hc * N * (2 * D + 4 * D + 4 + 8 + 8 + 8 + 8)
                kern[n]["kind"] = "delta fold row kernel (HBM)"
            else:
                # support lists (sparse_rows_kernel: delta and dQ): per row dO (bf16),
                # (count, offset), ~30 (key, t) entries, tau, m in; delta (fp64), rowc, dQ
                # (fp32) and ~30 scattered (row, p, dS) out; the V and K rows it gathers
                # (2 x 256 B per entry) stay L2-resident (one head at a time), not counted
                b = hc * N * (2 * D + 16 + 30 * 8 + 8 + 8 + 8 + 8 + 4 * D + 30 * 12)
                kern[n]["kind"] = "delta and dQ from support lists (SIMT gather, no MMA)"
            kern[n]["hbm_bytes"] = b
            kern[n]["gbps"] = b / (kern[n]["ms_avg"] * 1e-3) / 1e9
            kern[n]["frac_hbm"] = kern[n]["gbps"] / peak_bw
        elif n == "tc_dkdv" and n in exe and exe[n] == 0:
            # sparse_keys_kernel: per key its (row, p, dS) list (~30 x 12 B) and offsets
            # in, dK and dV (fp32) out; the dO / Q rows it gathers stay L2-resident
            b = hc * N * (30 * 12 + 8 + 2 * 4 * D)
            kern[n]["kind"] = "dK and dV from support lists (SIMT gather, no MMA)"
            kern[n]["hbm_bytes"] = b
            kern[n]["gbps"] = b / (kern[n]["ms_avg"] * 1e-3) / 1e9
            kern[n]["frac_hbm"] = kern[n]["gbps"] / peak_bw
    if dom in exe:
        ach = kern[dom]["tflops_executed"]
        roofline = {"kernel": dom, "bound": "tensor", "achieved": ach, "peak": peak_tf,
                    "unit": "TFLOP/s", "frac": ach / peak_tf, "traffic": None,
                    "basis": "executed tcgen05 MMA flops per launch (incl. hi/lo halves), "
                             "workloads.executed_flops; tflops_alg = SURVEY 8(d) count",
                    "achieved_alg": kern[dom]["tflops_alg"],
                    "peak_kind": f"{peak_kind} bf16 (frac is 'of {peak_kind.split()[0]}')",
                    "share_of_step": kern[dom]["ms_avg"] * kern[dom]["launches"] /
                    (ms * args.steps)}
    prof_file = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if roofline and os.path.exists(prof_file):
        try:
            with open(prof_file) as f:
                tr = json.load(f).get(dom)
            if tr:
                roofline["traffic"] = tr.get("dram_bytes_per_launch", 0) * hc / 64
                roofline["traffic_note"] = tr.get("note")
        except Exception:
            pass

    # ---- e2e through the C-ABI host entry with pinned host buffers, over --steps
    e2e = None
    if not args.no_e2e:
        lib = _lib.load()
        pb = prob.c_problem(out_dtype_code=_lib.F32)
        hq, hk, hv, hdo = (x.cpu().pin_memory() for x in (q, k, v, do))
        shp = tuple(q.shape)
        hout = torch.empty(shp, dtype=torch.float32).pin_memory()
        hdq, hdk, hdv = (torch.empty(shp, dtype=torch.float32).pin_memory() for _ in range(3))
        htau = torch.empty(shp[:-1], dtype=torch.float64).pin_memory()
        hrm = torch.empty(shp[:-1], dtype=torch.float64).pin_memory()
        hdl = torch.empty(shp[:-1], dtype=torch.float64).pin_memory()
        hmask = torch.empty(shp[:2] + (T, (T + 31) // 32), dtype=torch.int32).pin_memory()
        P = lambda t: C.c_void_p(t.data_ptr())

        def e2e_call():
            _lib.check(lib.adattn_b200_run_host(C.byref(pb), P(hq), P(hk), P(hv), P(hdo),
                                                P(hout), P(htau), P(hrm), P(hmask), P(hdq),
                                                P(hdk), P(hdv), P(hdl), None))
        for _ in range(max(1, min(args.warmup, 3))):
            e2e_call()  # the first call allocates the cached device buffers
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_call()
        e_local = 1000.0 * (time.perf_counter() - t0) / args.steps
        if world > 1:
            dist.barrier()
        e_ms = parallel.max_over_ranks(e_local, device=dev)
        h2d = sum(x.numel() * x.element_size() for x in (hq, hk, hv, hdo))
        d2h = sum(x.numel() * x.element_size() for x in (hout, hdq, hdk, hdv, htau, hrm, hdl,
                                                         hmask))
        h2d = int(parallel.sum_over_ranks(h2d, device=dev))
        d2h = int(parallel.sum_over_ranks(d2h, device=dev))
        e2e = {"value": fl["f_eff"] / (e_ms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": e_ms,
               "steps": args.steps, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": "adattn_b200_run_host (C-ABI, pinned host buffers; wall clock, "
                       "max over ranks)"}
        del hq, hk, hv, hdo, hout, hdq, hdk, hdv

    sweep_steps = args.sweep_steps or args.steps
    sweep_warm = max(1, min(args.warmup, 3))

    # ---- sparsity sweep (anchored generator), same sharding
    sweep = []
    for bs in [x for x in args.sweep.split(",") if x.strip()]:
        beta = float(bs)
        qa, ka, va, da = workloads.anchored_heads(heads, N, D, beta, causal, seed=2000,
                                                  device=dev, dtype=dtype)
        pa_ = pa.AttentionProblem(qa, ka, va, alpha=alpha, causal=causal)
        sms, sres, _, _, _ = timed(pa_, da, sweep_warm, sweep_steps)
        snnz = int(parallel.sum_over_ranks(sres.stats.blocks_visited_fwd, device=dev))
        sfl = workloads.flops(D, snnz, A_head * total)
        sit = parallel.sum_over_ranks(sres.row_steps.double().sum().item(), device=dev)
        sweep.append({"beta": beta, "block_sparsity": 1.0 - snnz / (A_head * total),
                      "ms": sms, "steps": sweep_steps,
                      "tflops_eff": sfl["f_eff"] / (sms * 1e-3) / 1e12,
                      "tflops_alg": sfl["f_alg"] / (sms * 1e-3) / 1e12,
                      "tau_iters_avg": sit / (total * N)})
        del qa, ka, va, da, pa_, sres

    # ---- alpha sweep of the same shape (N(0,1) inputs)
    alpha_sweep = []
    for a_s in [x for x in args.alphas.split(",") if x.strip()]:
        pa_ = pa.AttentionProblem(q, k, v, alpha=float(a_s), causal=causal)
        sms, sres, _, _, _ = timed(pa_, do, sweep_warm, sweep_steps)
        snnz = int(parallel.sum_over_ranks(sres.stats.blocks_visited_fwd, device=dev))
        sfl = workloads.flops(D, snnz, A_head * total)
        sit = parallel.sum_over_ranks(sres.row_steps.double().sum().item(), device=dev)
        alpha_sweep.append({"alpha": float(a_s), "block_sparsity": 1.0 - snnz / (A_head * total),
                            "ms": sms, "steps": sweep_steps,
                            "tflops_eff": sfl["f_eff"] / (sms * 1e-3) / 1e12,
                            "tau_iters_avg": sit / (total * N)})
        del pa_, sres

    # ---- CPU baseline (rank 0 at N=1 only): the reference on one head of this workload
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            n_cpu = args.ref_n or N
            r = cpu_reference_step(n_cpu, D, alpha, causal, head=0)
            cpu = {"value": r["tflops"], "unit": UNIT, "cores": r["threads"], "kind": "reference",
                   "sample": f"1 of the {total} heads (N={n_cpu}, d={D}, alpha={alpha}, "
                             f"causal={causal}, bf16-valued N(0,1) inputs): the reference's "
                             f"forward+backward (oracle/_ref, -O3) on {r['threads']} threads, "
                             f"{r['seconds']:.1f} s"}
        except Exception as ex:  # the checker is optional for the GPU number
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    nccl = None
    if world > 1 and nccl_log:
        nccl = nccl_init_lines(nccl_log + "*")

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic N(0,1) (cmd_attn distribution, qscale=%g), one generator "
                    "seed per head" % args.qscale,
            "config": {"workload": f"{args.config}: alpha={alpha} causal={causal} B={B} H={H} "
                                   f"N={N} d={D}, {total} heads split over {world} GPU(s)",
                       "alpha": alpha, "causal": causal, "B": B, "H": H, "N": N, "d": D,
                       "parallelism": f"heads/{world} (B*H={total} fixed; no collective)",
                       "heads_per_gpu": [parallel.shard_heads(total, world, r)[1]
                                         for r in range(world)],
                       "path": resolved,
                       "l2": "inputs 4x%d MiB per GPU > L2, no flush" % (hc * N * D * 2 >> 20)},
            "block_sparsity": sparsity, "nnz_blocks": nnz_all,
            "tau_iters_avg": tau_iters, "tflops_alg": tflops_alg,
            "gpu_launches": int(launches), "kernels": kern, "roofline": roofline,
            "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu, "sweep": sweep,
            "alpha_sweep": alpha_sweep, "validation": validation, "nccl_init": nccl,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
