"""Synthetic inputs for the measurement harness (BASELINE.json configs).

* ``gaussian``  -- cmd_attn's distribution (atn_main.cpp:227-232): Q = qscale*N(0,1),
  K, V, dO ~ N(0,1), drawn on the GPU with torch (bf16).
* ``anchored``  -- SURVEY.md section 7 item 7: each 64-row query tile picks G=2 anchor
  key tiles (its diagonal tile and one random earlier tile); every row picks a
  random anchor key c <= r inside them and sets q_r = beta * k_c + N(0,1).
  beta is the temperature knob that sweeps 64x64 block sparsity from ~0 to the
  1 - G*T/A ceiling; the harness reports the sparsity it measures.
"""
from __future__ import annotations

import torch

# BASELINE.json "configs" (index -> shape); C3 is the headline (metric quoted at N=32K)
CONFIGS = {
    "c1": dict(B=1, H=4, N=1024, D=64, alpha=1.5, causal=True, dtype=torch.float32),
    "c2": dict(B=4, H=16, N=8192, D=128, alpha=1.5, causal=True, dtype=torch.bfloat16),
    "c3": dict(B=2, H=32, N=32768, D=128, alpha=1.5, causal=True, dtype=torch.bfloat16),
    "c4": dict(B=8, H=32, N=16384, D=64, alpha=1.5, causal=False, dtype=torch.bfloat16),
    "c5": dict(B=1, H=32, N=131072, D=128, alpha=1.5, causal=True, dtype=torch.bfloat16),
}


def gaussian(B, H, N, D, qscale=1.0, seed=0, device="cuda", dtype=torch.bfloat16):
    g = torch.Generator(device=device).manual_seed(seed)
    mk = lambda s: (s * torch.randn(B, H, N, D, generator=g, device=device)).to(dtype)
    q = mk(qscale)
    k, v, do = mk(1.0), mk(1.0), mk(1.0)
    return q, k, v, do


def anchored(B, H, N, D, beta, causal=True, seed=0, device="cuda", dtype=torch.bfloat16):
    g = torch.Generator(device=device).manual_seed(seed)
    k = torch.randn(B, H, N, D, generator=g, device=device)
    v = torch.randn(B, H, N, D, generator=g, device=device)
    do = torch.randn(B, H, N, D, generator=g, device=device)
    noise = torch.randn(B, H, N, D, generator=g, device=device)
    T = N // 64
    tiles = torch.arange(T, device=device)
    hi = tiles + 1 if causal else torch.full_like(tiles, T)
    other = (torch.rand(B, H, T, generator=g, device=device) * hi).long()  # random tile
    other = torch.minimum(other, hi - 1)
    r = torch.arange(N, device=device)
    rt = r // 64
    pick = torch.rand(B, H, N, generator=g, device=device) < 0.5
    tile = torch.where(pick, other[:, :, rt], rt.expand(B, H, N))
    # key inside the tile; in the diagonal tile stay at or below the row (causal)
    width = torch.where((tile == rt) & causal, (r % 64) + 1, torch.full_like(r, 64))
    off = (torch.rand(B, H, N, generator=g, device=device) * width).long()
    c = tile * 64 + torch.minimum(off, width - 1)
    kc = torch.gather(k, 2, c.unsqueeze(-1).expand(B, H, N, D))
    q = beta * kc + noise
    return q.to(dtype), k.to(dtype), v.to(dtype), do.to(dtype)


def gaussian_heads(heads, N, D, qscale=1.0, seed=0, device="cuda", dtype=torch.bfloat16):
    """``[1, len(heads), N, D]`` q, k, v, dO where head h is drawn from its own
    generator (seed + h): a head's values do not depend on how the B x H heads are
    sharded over ranks, so a sharded run is comparable head by head with a
    single-GPU run of the same heads (bench.py validation)."""
    heads = list(heads)
    out = [torch.empty(1, len(heads), N, D, dtype=dtype, device=device) for _ in range(4)]
    for i, h in enumerate(heads):
        g = torch.Generator(device=device).manual_seed(seed + h)
        for j, s in enumerate((qscale, 1.0, 1.0, 1.0)):
            out[j][0, i] = (s * torch.randn(N, D, generator=g, device=device)).to(dtype)
    return tuple(out)


def anchored_heads(heads, N, D, beta, causal=True, seed=0, device="cuda",
                   dtype=torch.bfloat16):
    """Per-head-seeded ``anchored`` inputs, ``[1, len(heads), N, D]`` (see gaussian_heads)."""
    heads = list(heads)
    out = [torch.empty(1, len(heads), N, D, dtype=dtype, device=device) for _ in range(4)]
    for i, h in enumerate(heads):
        parts = anchored(1, 1, N, D, beta, causal, seed=seed + h, device=device, dtype=dtype)
        for j in range(4):
            out[j][0, i] = parts[j][0, 0]
    return tuple(out)


def flops(D: int, nnz: int, addressable: int, ref_passes: int = 3) -> dict:
    """F_eff = 14 d 4096 nnz (fwd QK^T+PV, bwd S, dP, dV, dK, dQ
    over active 64x64 blocks); F_alg = F_eff + 2 d 4096 (2 + R) A (max, histogram and
    R refinement QK^T passes over every addressable block)."""
    f_eff = 14.0 * D * 4096 * nnz
    f_alg = f_eff + 2.0 * D * 4096 * (2 + ref_passes) * addressable
    f_fwd = 4.0 * D * 4096 * nnz + 2.0 * D * 4096 * (2 + ref_passes) * addressable
    return dict(f_eff=f_eff, f_alg=f_alg, f_fwd=f_fwd)


def executed_flops(mask_words, n: int, d: int, causal: bool, dv_f16=None, alpha: float = 1.5,
                   row_steps=None) -> dict:
    """Tensor-core flops each kernel actually issues for one problem (all heads),
    from the 64x64 block mask ([B][H][t_r][wpr] u32) -- the numerator of the
    per-kernel roofline.  Counts every tcgen05 MMA the
    kernels issue, including the hi/lo split halves; the forward's threshold
    sweeps are counted without tile skipping (exact for inputs where no tile
    is skippable, an upper bound otherwise).

    tc_fwd   list mode (alpha >= 1.4, the default): 2 sweeps (MAX, CAND) of S over
             the causal 128x128 tiles of each 128-row group; sweep mode (alpha < 1.4):
             MAX + HIST + one REF sweep per refinement pass (the most steps of any
             row of the 256-row CTA + 1, from row_steps; 3 if not given) -- plus OUT
             (S and P V) over active tiles
             + with the delta fold (alpha = 2 without support lists; ADATTN_DELTA_FOLD=1/0;
             single-CTA forward, n % 256 == 0, m % 128 == 0) U V over active tiles
    tc_delta S, dP over active (128 rows x 128 keys) tiles; 0 with the support lists
             (list mode: delta = sum u (dO . v) / sum u over each row's support, a
             SIMT gather kernel) or the delta fold (delta = dO . Ubar / sum u)
    tc_dq    S, dP, dQ (fp16 sigma dS and K: one product -- default for alpha <= 1.5;
             bf16 hi/lo otherwise)
             over active (128 x 128) tiles
    (support lists, the default in list mode: tc_delta, tc_dq and tc_dkdv are 0 -- delta
    and dQ come from sparse_rows_kernel, dK and dV from sparse_keys_kernel, gathers over
    each row's / key's support entries)
    tc_dkdv  S^T, dP^T, dV (fp16 P and dO: one product; bf16 hi/lo with
             ADATTN_DV_F16=0 or for d != 128), dK (fp16 sigma dS: one product, as
             for dQ; else hi/lo) over active (128 keys x 64 queries) units
    (A CTA whose candidate list overflows re-runs HIST + REF sweeps; not counted.)
    """
    import os
    import torch
    w = mask_words.view(torch.int32)
    Bh = w.shape[0] * w.shape[1]
    t_r = w.shape[2]
    t_c = n // 64
    bits = ((w.reshape(Bh, t_r, -1, 1) >> torch.arange(32, device=w.device)) & 1).reshape(Bh, t_r, -1)
    bits = bits[:, :, :t_c].bool()
    g = bits.reshape(Bh, t_r // 2, 2, t_c // 2, 2).any(dim=4).any(dim=2)  # 128 x 128 tiles
    u = bits.reshape(Bh, t_r, t_c // 2, 2).any(dim=3)                    # 64 q x 128 keys
    tile = 2.0 * 128 * 128 * d
    nr = t_r // 2
    if causal:
        J = torch.arange(t_c // 2)
        rg = torch.arange(nr)
        sweep_tiles = int(((J[None, :] <= rg[:, None]).sum())) * Bh
    else:
        sweep_tiles = nr * (t_c // 2) * Bh
    act = int(g.sum())
    units = int(u.sum())
    list_mode = alpha >= 1.4 and int(os.environ.get("ADATTN_CAND_CAP", "512")) >= 64
    if list_mode:
        sweeps_fwd = 2.0 * sweep_tiles
    else:  # per 256-row CTA: MAX, HIST, then (max steps + 1) REF sweeps over its tiles
        if causal:
            per_rg = (J[None, :] <= rg[:, None]).sum(dim=1).double()  # tiles of each 128-row group
        else:
            per_rg = torch.full((nr,), float(t_c // 2), dtype=torch.float64)
        if row_steps is not None:
            st = row_steps.reshape(Bh, -1).to(torch.int64).cpu()
            passes = st.reshape(Bh, -1, 256).amax(dim=2).double() + 1.0  # [Bh, n/256]
        else:
            passes = torch.full((Bh, max(1, nr // 2)), 3.0, dtype=torch.float64)
        rg_pass = passes.repeat_interleave(2, dim=1)[:, :nr]             # [Bh, nr]
        sweeps_fwd = float(((2.0 + rg_pass) * per_rg[None, :]).sum())
    if dv_f16 is None:  # the library's default (csrc/tc_bwd.cu dv_f16_enabled, pair kernel)
        dv_f16 = (d == 128 and os.environ.get("ADATTN_DV_F16", "1") != "0"
                  and os.environ.get("ADATTN_KV_PAIRS", "1") != "0")
    ds_env = os.environ.get("ADATTN_DS_F16", "auto")  # the library's rule (tc_bwd.cu ds_f16_enabled)
    ds_f16 = d == 128 and (ds_env == "1" or (ds_env not in ("0", "1") and alpha <= 1.5))
    kv_pairs = os.environ.get("ADATTN_KV_PAIRS", "1") != "0"
    dq_pairs = os.environ.get("ADATTN_DQ_PAIRS", "1") != "0"
    # delta source (tc.cu delta_supp_possible / tc_fwd.cu fwd_delta_fold): the forward's
    # support lists in list mode (a SIMT gather kernel, no MMA), else the fold (alpha = 2,
    # or ADATTN_DELTA_FOLD=1), else the S, dP pre-pass
    supp = list_mode and os.environ.get("ADATTN_DELTA_SUPP", "1") != "0"
    fold_env = os.environ.get("ADATTN_DELTA_FOLD", "")
    fold = ((fold_env == "1" or (fold_env in ("", "auto") and alpha == 2.0 and not supp))
            and n % 256 == 0
            and (d != 128 or os.environ.get("ADATTN_FWD_PAIRS", "0") in ("", "0")))
    # with the support lists the gradients come from gather kernels too (no MMA):
    # sparse_rows_kernel (delta, dQ; reported as tc_delta) and sparse_keys_kernel (dK, dV;
    # reported as tc_dkdv) unless ADATTN_SPARSE_DQ / ADATTN_SPARSE_KV = 0
    sp_dq = supp and os.environ.get("ADATTN_SPARSE_DQ", "1") != "0"
    sp_kv = sp_dq and os.environ.get("ADATTN_SPARSE_KV", "1") != "0"
    # O from the support lists (sparse_out_kernel) replaces the output pass (S, P V) in
    # list mode with the support lists (single-CTA forward)
    sp_out = (supp and os.environ.get("ADATTN_SPARSE_OUT", "1") != "0"
              and not (d == 128 and os.environ.get("ADATTN_FWD_PAIRS", "0") not in ("", "0")))
    return {"tc_fwd": (sweeps_fwd + (0 if sp_out else (3 if fold else 2) * act)) * tile,
            "tc_delta": (0 if (fold or supp) else 2) * act * tile,
            "tc_dq": 0 if sp_dq else (3 if ds_f16 and dq_pairs else 4) * act * tile,
            "tc_dkdv": 0 if sp_kv else (4 + (0 if dv_f16 else 1) + (0 if ds_f16 and kv_pairs else 1))
            * units * (2.0 * 128 * 64 * d)}
