"""Generates tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref, compiled
from /root/reference sources).  Run here (the reference is absent on the GPU
box); the fixtures travel with the repo.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Oracle, Problem, gen_attn_inputs  # noqa: E402

# (name, seed, n, m, d, dv, alpha, causal, block_r, block_c, bins, refine_iters, refine_tol, qscale)
CASES = [
    ("ragged_causal_a15", 101, 130, 130, 16, 16, 1.5, True, 64, 64, 8, 2, 1e-6, 1.0),
    ("rect_a2_tiles16x8", 102, 96, 80, 8, 12, 2.0, False, 16, 8, 8, 2, 1e-6, 2.0),
    ("secant_a25_tiles8", 103, 64, 64, 4, 4, 2.5, True, 8, 8, 8, 24, 1e-12, 1.0),
    ("a125_causal_d32", 104, 128, 128, 32, 32, 1.25, True, 64, 64, 8, 2, 1e-6, 1.0),
    ("cfg1_like_n256_d64", 105, 256, 256, 64, 64, 1.5, True, 64, 64, 8, 2, 1e-6, 1.0),
    ("sparse_a15_q8_bins32", 106, 192, 192, 16, 16, 1.5, False, 64, 32, 32, 2, 1e-6, 8.0),
    ("bins4_a2_causal", 107, 160, 160, 8, 8, 2.0, True, 32, 32, 4, 3, 1e-9, 4.0),
    ("very_sparse_a2_q50_tiles4", 108, 48, 48, 4, 4, 2.0, False, 4, 4, 8, 2, 1e-6, 50.0),
    ("sparse_causal_a15_q40", 109, 320, 320, 8, 8, 1.5, True, 32, 32, 8, 2, 1e-6, 40.0),
]


def make(ref: Oracle):
    for (name, seed, n, m, d, dv, alpha, causal, br, bc, bins, iters, tol, qs) in CASES:
        g = ref.gaussian(seed, n * d + m * d + m * dv + n * dv)
        o = 0
        q = (qs * g[o:o + n * d]).reshape(n, d); o += n * d
        k = g[o:o + m * d].reshape(m, d); o += m * d
        v = g[o:o + m * dv].reshape(m, dv); o += m * dv
        do = g[o:o + n * dv].reshape(n, dv)
        # fp32-representable so the GPU's fp32/bf16 inputs carry identical values
        q, k, v, do = (x.astype(np.float32).astype(np.float64) for x in (q, k, v, do))
        pb = Problem(q, k, v, alpha=alpha, causal=causal, block_r=br, block_c=bc, bins=bins,
                     refine_iters=iters, refine_tol=tol)
        f = ref.forward(pb, threads=4)
        b = ref.backward(pb, f, do, threads=4)
        np.savez_compressed(
            os.path.join(HERE, name + ".npz"), q=q, k=k, v=v, dout=do,
            params=np.array([n, m, d, dv, alpha, int(causal), br, bc, bins, iters, tol]),
            out=f["out"], tau=f["tau"], row_max=f["row_max"], mask=f["mask"],
            block_sparsity=f["block_sparsity"], blocks_visited_fwd=f["blocks_visited_fwd"],
            flushes=f["flushes"], delta=b["delta"], dq=b["dq"], dk=b["dk"], dv=b["dv"],
            blocks_visited_bwd=b["blocks_visited_bwd"])
        print(name, "sparsity", f["block_sparsity"])


if __name__ == "__main__":
    make(Oracle("reference"))
