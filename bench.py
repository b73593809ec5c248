#!/usr/bin/env python
"""Benchmark of the alpha-entmax attention hot path (fwd + bwd) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (BASELINE.json configs[2], the config the metric is quoted on): alpha=1.5,
causal, B=2 H=32 N=32768 d=128, bf16 inputs (synthetic, cmd_attn's N(0,1)
distribution, qscale=1), per GPU (weak scaling: every rank runs its own B x H heads).
A "step" = forward + backward over the whole batch.  `value` = effective TFLOP/s over
the non-zero 64x64 blocks (F_eff = 14 d 4096 nnz) of all ranks / max
rank time.  Inputs (4 x 512 MiB) exceed the 126 MB L2, so no explicit flush.
`e2e` = the same metric through the C-ABI host entry (adattn_b200_run_host) with
pinned host buffers: H2D of q/k/v/dO and D2H of out/dq/dk/dv/tau/row_max/mask
inside the timed region.  `sweep` = the same step on the "anchored" generator at
several temperatures (block sparsity 0..~95%, measured).
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
    """Roofline denominators (B200_PROFILING.md): the kernels are timed inside the
    fwd+bwd step (~0.1 s of back-to-back kernels under the power cap), so the
    sustained bf16 figure of MEASURED_PEAKS.json is the one that applies; the burst
    figure when only that is present; else the recipe's fallback (1.59 PF burst)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        bw = float(p.get("hbm_gbs", 6542.4))
        if p.get("bf16_tflops_sustained"):
            return float(p["bf16_tflops_sustained"]), bw, "measured sustained"
        return float(p["bf16_tflops"]), bw, "measured burst"
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


# ------------------------------------------------------------------ CPU side
def cpu_reference_step(n=4096, d=128, alpha=1.5, seed=1, threads=None, kind="reference"):
    """One fwd+bwd of the reference CPU implementation (oracle/_ref, compiled from the
    reference sources) on one head of the workload's shape at n rows."""
    from oracle.oracle import Oracle, Problem, gen_attn_inputs
    orc = Oracle(kind)
    threads = threads or os.cpu_count() or 1
    q, k, v, do = gen_attn_inputs(seed, n, d, 1.0, orc)
    q, k, v, do = (x.astype("float32").astype("float64") for x in (q, k, v, do))
    pb = Problem(q, k, v, alpha=alpha, causal=True)
    t0 = time.perf_counter()
    f = orc.forward(pb, threads)
    orc.backward(pb, f, do, threads)
    dt = time.perf_counter() - t0
    nnz = f["blocks_visited_fwd"]
    return dict(seconds=dt, nnz=nnz, tflops=14.0 * d * 4096 * nnz / dt / 1e12, threads=threads,
                sparsity=f["block_sparsity"])


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = dict(n=args.ref_n, d=128, alpha=1.5)
    for _ in range(args.warmup):
        cpu_reference_step(**cfg)
    vals, secs = [], []
    for s in range(args.steps):
        r = cpu_reference_step(seed=1 + s, **cfg)
        vals.append(r["tflops"])
        secs.append(r["seconds"])
    v = sum(vals) / len(vals)
    sample = (f"1 head of the C3 shape at N={args.ref_n} (d=128, alpha=1.5, causal, fp32-valued "
              f"N(0,1) inputs), reference forward+backward with {r['threads']} threads")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * sum(secs) / len(secs), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c3-sample", "n": args.ref_n, "d": 128, "alpha": 1.5,
                       "causal": True, "heads": 1},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": r["threads"], "kind": "reference",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU side
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
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--alphas", default="1.25,2.0",
                    help="extra alphas timed on the headline shape (comma list, '' = none)")
    ap.add_argument("--ref-n", type=int, default=4096)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist
    import paper_2604_15180_b200 as pa
    from paper_2604_15180_b200 import _lib, parallel, workloads

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg = dict(workloads.CONFIGS[args.config])
    if args.alpha is not None:
        cfg["alpha"] = args.alpha
    B, H, N, D = cfg["B"], cfg["H"], cfg["N"], cfg["D"]
    alpha, causal, dtype = cfg["alpha"], cfg["causal"], cfg["dtype"]
    q, k, v, do = workloads.gaussian(B, H, N, D, args.qscale, seed=1000 + rank, device=dev,
                                     dtype=dtype)
    prob = pa.AttentionProblem(q, k, v, alpha=alpha, causal=causal)

    def step(p, dout):
        r = pa.forward(p)
        g = pa.backward(p, r, dout)
        return r, g

    def timed(p, dout, warm, steps, profile=False):
        # warm-up holds the previous step's results exactly like the timed loop, so the
        # caching allocator owns both result sets before timing (a cudaMalloc of a few
        # GB inside the first timed step stalled it by up to ~10 ms)
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
        ms = parallel.max_over_ranks(e0.elapsed_time(e1) / steps, device=dev)
        return ms, res, launches, kt

    clk = ClockSampler(local)
    clk.start()
    ms, res, launches, ktimes = timed(prob, do, args.warmup, args.steps, profile=True)
    clocks = clk.stop()

    # one validation gather over NVLink, outside the timed region: per-rank checksums
    chk = torch.stack([res.tau.double().sum(), res.out.double().abs().sum(),
                       torch.tensor(float(torch.isfinite(res.out).all()), device=dev,
                                    dtype=torch.float64)])
    gathered = parallel.gather_to_rank0(chk.unsqueeze(0))
    validation = None
    if rank == 0:
        gathered = gathered.cpu()
        validation = {"ranks": int(gathered.shape[0]),
                      "all_finite": bool((gathered[:, 2] == 1).all()),
                      "tau_sums": [round(float(x), 3) for x in gathered[:, 0]]}
    st = res.stats
    T = N // 64
    A_head = T * (T + 1) // 2 if causal else T * T
    nnz_rank = st.blocks_visited_fwd
    tau_iters = res.row_steps.float().mean().item()
    nnz_all = nnz_rank * world
    fl = workloads.flops(D, nnz_all, A_head * B * H * world)
    value = fl["f_eff"] / (ms * 1e-3) / 1e12
    tflops_alg = fl["f_alg"] / (ms * 1e-3) / 1e12

    # ---- per-kernel breakdown (CUDA events on the launching stream, timed region)
    agg = {}
    for name, t in ktimes:
        a = agg.setdefault(name, [0.0, 0])
        a[0] += t
        a[1] += 1
    kern = {n: {"ms_avg": a[0] / a[1], "launches": a[1]} for n, a in agg.items()}
    peak_tf, peak_bw, peak_kind = peaks()
    fl_rank = workloads.flops(D, nnz_rank, A_head * B * H)
    # per launch of each tensor-core kernel: (a) the tcgen05 MMA flops it executes
    # (roofline numerator, workloads.executed_flops) and (b) the algorithmic count of
    # SURVEY 8(d) (reference algorithm: 2+R dense passes, no hi/lo halves)
    exe = workloads.executed_flops(res.mask.words, N, D, causal)
    per_alg = {"tc_fwd": fl_rank["f_fwd"], "tc_delta": 4.0 * D * 4096 * nnz_rank,
               "tc_dq": 6.0 * D * 4096 * nnz_rank, "tc_dkdv": 8.0 * D * 4096 * nnz_rank}
    dom = max(kern, key=lambda n: kern[n]["ms_avg"] * kern[n]["launches"]) if kern else None
    roofline = None
    for n in kern:
        if n in exe:
            kern[n]["tflops_executed"] = exe[n] / (kern[n]["ms_avg"] * 1e-3) / 1e12
            kern[n]["frac_executed"] = kern[n]["tflops_executed"] / peak_tf
            kern[n]["tflops_alg"] = per_alg[n] / (kern[n]["ms_avg"] * 1e-3) / 1e12
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
                roofline["traffic"] = tr.get("dram_bytes_per_launch")
                roofline["traffic_note"] = tr.get("note")
        except Exception:
            pass

    # ---- e2e through the C-ABI host entry with pinned host buffers
    e2e = None
    if args.e2e_steps > 0:
        lib = _lib.load()
        pb = prob.c_problem(out_dtype_code=_lib.F32)
        hq, hk, hv, hdo = (x.cpu().pin_memory() for x in (q, k, v, do))
        hout = torch.empty(B, H, N, D, dtype=torch.float32).pin_memory()
        hdq, hdk, hdv = (torch.empty(B, H, N, D, dtype=torch.float32).pin_memory() for _ in range(3))
        htau = torch.empty(B, H, N, dtype=torch.float64).pin_memory()
        hrm = torch.empty(B, H, N, dtype=torch.float64).pin_memory()
        hdl = torch.empty(B, H, N, dtype=torch.float64).pin_memory()
        hmask = torch.empty(B, H, T, (T + 31) // 32, dtype=torch.int32).pin_memory()
        P = lambda t: C.c_void_p(t.data_ptr())
        hst = _lib.Stats()

        def e2e_call():
            _lib.check(lib.adattn_b200_run_host(C.byref(pb), P(hq), P(hk), P(hv), P(hdo), P(hout),
                                                P(htau), P(hrm), P(hmask), P(hdq), P(hdk), P(hdv),
                                                P(hdl), None))
        e2e_call()  # warm (allocates the cached device buffers)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_call()
        e_ms = parallel.max_over_ranks(1000.0 * (time.perf_counter() - t0) / args.e2e_steps,
                                       device=dev)
        h2d = sum(x.numel() * x.element_size() for x in (hq, hk, hv, hdo))
        d2h = sum(x.numel() * x.element_size() for x in (hout, hdq, hdk, hdv, htau, hrm, hdl, hmask))
        e2e = {"value": fl["f_eff"] / (e_ms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": "adattn_b200_run_host (C-ABI, pinned host buffers)"}
        del hq, hk, hv, hdo, hout, hdq, hdk, hdv

    # ---- sparsity sweep (anchored generator), per-rank inputs
    sweep = []
    for bs in [x for x in args.sweep.split(",") if x.strip()]:
        beta = float(bs)
        qa, ka, va, da = workloads.anchored(B, H, N, D, beta, causal, seed=2000 + rank,
                                            device=dev, dtype=dtype)
        pa_ = pa.AttentionProblem(qa, ka, va, alpha=alpha, causal=causal)
        sms, sres, _, _ = timed(pa_, da, 1, 2)
        sst = sres.stats
        sfl = workloads.flops(D, sst.blocks_visited_fwd * world, A_head * B * H * world)
        sweep.append({"beta": beta, "block_sparsity": sst.block_sparsity, "ms": sms,
                      "tflops_eff": sfl["f_eff"] / (sms * 1e-3) / 1e12,
                      "tflops_alg": sfl["f_alg"] / (sms * 1e-3) / 1e12,
                      "tau_iters_avg": sres.row_steps.float().mean().item()})
        del qa, ka, va, da, pa_, sres

    # ---- alpha sweep of BASELINE config 3 (same shape, N(0,1) inputs): alpha = 1.25 runs
    # the refinement sweeps (candidate lists would overflow), alpha = 2 the lists
    alpha_sweep = []
    for a_s in [x for x in args.alphas.split(",") if x.strip()]:
        pa_ = pa.AttentionProblem(q, k, v, alpha=float(a_s), causal=causal)
        sms, sres, _, _ = timed(pa_, do, 1, 2)
        sst = sres.stats
        sfl = workloads.flops(D, sst.blocks_visited_fwd * world, A_head * B * H * world)
        alpha_sweep.append({"alpha": float(a_s), "block_sparsity": sst.block_sparsity, "ms": sms,
                            "tflops_eff": sfl["f_eff"] / (sms * 1e-3) / 1e12,
                            "tau_iters_avg": sres.row_steps.float().mean().item()})
        del pa_, sres

    # ---- CPU baseline (rank 0 at N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            r = cpu_reference_step(n=args.ref_n)
            cpu = {"value": r["tflops"], "unit": UNIT, "cores": r["threads"], "kind": "reference",
                   "sample": f"1 head, N={args.ref_n}, d=128, alpha=1.5, causal: the reference's "
                             f"forward+backward (oracle/_ref, -O3) on {r['threads']} threads, "
                             f"{r['seconds']:.2f} s"}
        except Exception as ex:  # the checker is optional for the GPU number
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic N(0,1) (cmd_attn distribution, qscale=%g)" % args.qscale,
            "config": {"workload": f"{args.config}: alpha={alpha} causal={causal} B={B} H={H} "
                                   f"N={N} d={D} per GPU", "alpha": alpha, "causal": causal,
                       "B": B, "H": H, "N": N, "d": D, "parallelism": f"heads x{world} (weak)",
                       "l2": "inputs 4x%d MiB > L2, no flush" % (B * H * N * D * 2 >> 20)},
            "block_sparsity": st.block_sparsity, "nnz_blocks": nnz_all,
            "tau_iters_avg": tau_iters, "tflops_alg": tflops_alg,
            "gpu_launches": int(launches), "kernels": kern, "roofline": roofline,
            "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu, "sweep": sweep,
            "alpha_sweep": alpha_sweep,
            "validation_gather": validation,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
