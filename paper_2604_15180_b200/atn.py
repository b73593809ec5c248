"""`atn` -- the reference's experiment driver with the B200 backend
(/root/reference/proj/tools/atn_main.cpp).

    python -m paper_2604_15180_b200.atn attn --n 2048 --d 128 --causal --out json
    python -m paper_2604_15180_b200.atn gen --n 4 --d 3 --seed 7 --out x.atn
    python -m paper_2604_15180_b200.atn dump x.atn

``attn`` reproduces cmd_attn (atn_main.cpp:224-328): the same input stream
(Q = qscale N(0,1), then K, V, dO from Xoshiro256pp(seed)), forward + backward
(here on the GPU), and one BenchRecord with the same experiment/seed/params/
metrics keys, emitted as one JSON object per line (sorted keys, compact, like
nlohmann::json::dump) or CSV with the frozen column order (README.md:122-138).
Timings are CUDA-event device times of the two calls; the four phase timers are
0 because the phases run inside one fused kernel (the reference also reports 0
when its phases are not timed, attention.cpp:170).  ``--verify`` compares with
the dense fp64 reference on the GPU (paper_2604_15180_b200.dense, n <= 4096).
``--dtype`` picks the device input precision: f32/f64 run the exact path
(bit-identical to the reference), bf16 the tensor-core path.
Errors print {"error": ...} on stderr and exit 1 (atn_main.cpp:416-419).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

PARAM_COLS = ["n", "d", "alpha", "block_r", "block_c", "bins", "causal", "qscale", "threads"]
METRIC_COLS = ["block_sparsity", "blocks_visited_fwd", "blocks_visited_bwd", "flushes",
               "t_phase1_ms", "t_phase2_ms", "t_phase3_ms", "t_phase4_ms", "t_forward_ms",
               "t_backward_ms", "max_abs_err_out", "max_abs_err_tau", "fd_max_abs_err"]


def _dump(v) -> str:
    return json.dumps(v, sort_keys=True, separators=(",", ":"))


def emit_records(records, fmt, param_cols, metric_cols, out=None):
    """emit_records (atn_main.cpp:56-71)."""
    out = out or sys.stdout
    if fmt == "json":
        for r in records:
            out.write(_dump(r) + "\n")
        return
    out.write(",".join(["experiment", "seed"] + param_cols + metric_cols) + "\n")
    for r in records:
        cells = [r["experiment"], str(r["seed"])]
        for key, cols in (("params", param_cols), ("metrics", metric_cols)):
            for c in cols:
                v = r[key].get(c)
                cells.append("" if v is None else (v if isinstance(v, str) else _dump(v)))
        out.write(",".join(cells) + "\n")


def cmd_gen(a):
    from . import tensor_io
    if a.dist != "gaussian":
        raise ValueError("gen: unknown --dist " + a.dist)
    dims = [a.n] + ([a.d] if a.d and a.d > 0 else [])
    _, g = tensor_io.xoshiro(a.seed, 0, int(np.prod(dims)))
    tensor_io.save_tensor(a.out, g.reshape(dims), tensor_io.F32 if a.dtype == "f32" else tensor_io.F64)
    return 0


def cmd_dump(a):
    from . import tensor_io
    vals, dt = tensor_io.load_tensor(a.file)
    x = vals.reshape(-1)
    mean = float(x.sum() / x.size)
    var = float((x * x).sum() / x.size - mean * mean)
    print(json.dumps({"count": int(x.size), "dims": list(vals.shape), "dtype": "f32" if dt == 0 else "f64",
                      "max": float(x.max()), "mean": mean, "min": float(x.min()),
                      "rank": vals.ndim, "std": math.sqrt(max(var, 0.0))}, indent=2, sort_keys=True))
    return 0


def cmd_attn(a):
    import torch

    import paper_2604_15180_b200 as pa
    from . import dense, tensor_io
    if not torch.cuda.is_available():
        raise RuntimeError("attn: no CUDA device (the B200 backend has no CPU path)")
    dev = torch.device("cuda")
    dt = {"f32": torch.float32, "f64": torch.float64, "bf16": torch.bfloat16}[a.dtype]
    q, k, v, do = tensor_io.attn_inputs(a.seed, a.n, a.d, a.qscale)
    T = lambda x: torch.from_numpy(x).to(dev).to(dt)
    Q, K, V, DO = T(q), T(k), T(v), T(do)
    p = pa.AttentionProblem(Q, K, V, alpha=a.alpha, causal=a.causal, block_r=a.block_r,
                            block_c=a.block_c, bins=a.bins)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    ev[0].record()
    res = pa.forward(p)
    ev[1].record()
    grads = pa.backward(p, res, DO)
    ev[2].record()
    torch.cuda.synchronize()
    st = res.stats  # after backward: blocks_visited_bwd = 2 nnz (attention.cpp:537)
    rec = {"experiment": "attn", "seed": a.seed,
           "params": {"n": a.n, "d": a.d, "alpha": a.alpha, "block_r": a.block_r,
                      "block_c": a.block_c, "bins": a.bins, "causal": bool(a.causal),
                      "qscale": a.qscale, "threads": a.threads},
           "metrics": {"block_sparsity": st.block_sparsity,
                       "blocks_visited_fwd": int(st.blocks_visited_fwd),
                       "blocks_visited_bwd": int(st.blocks_visited_bwd),
                       "flushes": int(st.flushes),
                       "t_phase1_ms": 0.0, "t_phase2_ms": 0.0, "t_phase3_ms": 0.0,
                       "t_phase4_ms": 0.0,
                       "t_forward_ms": ev[0].elapsed_time(ev[1]),
                       "t_backward_ms": ev[1].elapsed_time(ev[2])}}
    if a.verify:
        if a.n > 4096:
            raise ValueError("attn: --verify caps n at 4096")
        ref = dense.dense_reference(Q, K, V, alpha=a.alpha, causal=a.causal,
                                    block_r=a.block_r, block_c=a.block_c)
        rec["metrics"]["max_abs_err_out"] = float((res.out.reshape(a.n, -1).double() - ref["out"]).abs().max())
        rec["metrics"]["max_abs_err_tau"] = float((res.tau.reshape(-1).double() - ref["tau"]).abs().max())
    if a.mask_out:
        data = res.mask.serialize()
        tmp = a.mask_out + ".tmp"
        with open(tmp, "wb") as f:
            f.write(data)
        os.replace(tmp, a.mask_out)
    emit_records([rec], a.out, PARAM_COLS, METRIC_COLS)
    return 0


def cmd_solve(a):
    """cmd_solve (atn_main.cpp:139-200) on the GPU row solver (one row)."""
    import torch

    from . import rows, tensor_io
    vals, _ = tensor_io.load_tensor(a.input)
    if vals.ndim != 1:
        raise ValueError("solve: input must be a rank-1 tensor")
    if a.method == "exact":
        if a.alpha not in (1.5, 2.0):
            raise ValueError("solve: --method exact needs alpha 1.5 or 2.0")
        from . import dense
        s = torch.from_numpy(vals).cuda().unsqueeze(0)
        mx = s.amax(dim=1, keepdim=True)
        z = torch.where(s == mx, torch.ones_like(s), (a.alpha - 1.0) * (s - mx) + 1.0)
        tau = float(dense._tau_exact(z, a.alpha)[0])
        t = z[0] - tau
        p = torch.where(t > 0, t.clamp(min=0) ** (1.0 / (a.alpha - 1.0)), torch.zeros_like(t))
        out = {"alpha": a.alpha, "converged": True, "iterations": 0, "method": a.method,
               "probabilities": p.cpu().tolist(), "residual": float(p.sum()) - 1.0, "tau": tau}
    else:
        s = torch.from_numpy(vals).cuda().unsqueeze(0)
        r = rows.entmax_rows(s, a.alpha, a.method, a.bins, a.max_iters, a.tol, probs=True,
                             trace_len=a.max_iters + 1 if a.method != "bisection" else 0)
        out = {"alpha": a.alpha, "converged": bool(r.converged[0]), "method": a.method,
               "iterations": int(r.iterations[0]), "probabilities": r.probs[0].double().cpu().tolist(),
               "residual": float(r.residual[0]), "tau": float(r.tau[0])}
        if r.trace is not None:
            out["trace"] = [float(x) for x in r.trace[0][: int(r.iterations[0]) + 1].cpu()]
    print(json.dumps(out, indent=2, sort_keys=True))
    return 0


def cmd_bench_solver(a):
    """cmd_bench_solver (atn_main.cpp:204-220): one record per (method, iteration)."""
    from . import rows
    bins = [int(x) for x in a.bins_list.split(",") if x]
    recs = [{"experiment": "bench-solver", "seed": a.seed,
             "params": {"n": a.n, "alpha": a.alpha, "runs": a.runs, "method": m, "iteration": k},
             "metrics": {"mae": mae}}
            for m, k, mae in rows.solver_bench(a.n, a.alpha, bins, a.runs, a.seed, a.iters)]
    emit_records(recs, a.out, ["n", "alpha", "runs", "method", "iteration"], ["mae"])
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="atn", description="AdaSplash-2 entmax attention tools (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen", help="write a random tensor file")
    g.add_argument("--n", type=int, required=True)
    g.add_argument("--d", type=int, default=0)
    g.add_argument("--dist", default="gaussian")
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--dtype", default="f64", choices=["f32", "f64"])
    g.add_argument("--out", required=True)
    d = sub.add_parser("dump", help="print tensor header and summary stats")
    d.add_argument("file")
    s = sub.add_parser("solve", help="threshold solve on one score vector")
    s.add_argument("--alpha", type=float, required=True)
    s.add_argument("--input", required=True)
    s.add_argument("--method", default="histogram+hybrid",
                   choices=["exact", "bisection", "hybrid", "histogram+hybrid"])
    s.add_argument("--bins", type=int, default=8)
    s.add_argument("--tol", type=float, default=1e-6)
    s.add_argument("--max-iters", type=int, default=50)
    b = sub.add_parser("bench-solver", help="solver convergence benchmark")
    b.add_argument("--n", type=int, default=4096)
    b.add_argument("--alpha", type=float, default=1.5)
    b.add_argument("--bins-list", default="4,8,16")
    b.add_argument("--runs", type=int, default=10)
    b.add_argument("--seed", type=int, default=1)
    b.add_argument("--iters", type=int, default=10)
    b.add_argument("--out", default="json", choices=["json", "csv"])
    t = sub.add_parser("attn", help="tiled attention round trip")
    t.add_argument("--n", type=int, default=256)
    t.add_argument("--d", type=int, default=64)
    t.add_argument("--alpha", type=float, default=1.5)
    t.add_argument("--block-r", type=int, default=64)
    t.add_argument("--block-c", type=int, default=64)
    t.add_argument("--bins", type=int, default=8)
    t.add_argument("--causal", action="store_true")
    t.add_argument("--seed", type=int, default=1)
    t.add_argument("--qscale", type=float, default=1.0)
    t.add_argument("--verify", action="store_true")
    t.add_argument("--out", default="json", choices=["json", "csv"])
    t.add_argument("--threads", type=int, default=int(os.environ.get("ATN_THREADS", "1") or 1))
    t.add_argument("--mask-out", default="")
    t.add_argument("--dtype", default="f32", choices=["f32", "f64", "bf16"])
    a = ap.parse_args(argv)
    try:
        return {"gen": cmd_gen, "dump": cmd_dump, "attn": cmd_attn, "solve": cmd_solve,
                "bench-solver": cmd_bench_solver}[a.cmd](a)
    except Exception as e:  # noqa: BLE001 -- the reference's catch-all (atn_main.cpp:416-419)
        sys.stderr.write(json.dumps({"error": str(e)}) + "\n")
        return 1


if __name__ == "__main__":
    sys.exit(main())
