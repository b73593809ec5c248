"""Dense (materialized-scores) alpha-entmax attention on the GPU in fp64 -- the
`--verify` comparison of the `atn attn` record path.

Restates dense_reference (/root/reference/proj/src/attention.cpp:363-409):
scores s = scale q.k, causal masking, centring z = 1 at the row max else
(alpha-1)(s-m)+1 (entmax.cpp:22-57), the exact threshold by the sorted
top-k closed forms for alpha in {1.5, 2} (entmax.cpp:80-126) or bisection
(tol 1e-14, 200 iterations; entmax.cpp:128-164), p = [z - tau]_+^(1/(alpha-1))
(entmax.cpp:166-180), O = P V.  Vectorized over rows with torch (fp64); capped
at 4096 rows like the reference.
"""
from __future__ import annotations

import math

import torch


def _center(q, k, alpha, scale, causal):
    s = (q @ k.transpose(-1, -2)) * scale
    n, m = s.shape[-2], s.shape[-1]
    if causal:
        vis = torch.ones(n, m, dtype=torch.bool, device=s.device).tril()
        s = s.masked_fill(~vis, float("-inf"))
    mx = s.amax(dim=-1, keepdim=True)
    z = (alpha - 1.0) * (s - mx) + 1.0
    z = torch.where(s == mx, torch.ones_like(z), z)
    z = z.masked_fill(torch.isinf(s), float("-inf"))
    return z, mx.squeeze(-1)


def _tau_exact(z, alpha):
    zs, _ = torch.sort(z, dim=-1, descending=True)
    vis = torch.isfinite(zs)
    zs0 = torch.where(vis, zs, torch.zeros_like(zs))
    k = torch.arange(1, z.shape[-1] + 1, device=z.device, dtype=z.dtype)
    c1 = torch.cumsum(zs0, dim=-1)
    if alpha == 2.0:
        cand = (c1 - 1.0) / k
    else:
        c2 = torch.cumsum(zs0 * zs0, dim=-1)
        mean = c1 / k
        disc = torch.clamp(1.0 / k - (c2 / k - mean * mean), min=0.0)
        cand = mean - torch.sqrt(disc)
    nxt = torch.cat([zs[..., 1:], torch.full_like(zs[..., :1], float("-inf"))], dim=-1)
    stop = (nxt <= cand) | ~torch.isfinite(nxt)
    stop = stop & vis
    first = torch.argmax(stop.to(torch.int8), dim=-1, keepdim=True)  # first k meeting the test
    return torch.gather(cand, -1, first).squeeze(-1)


def _tau_bisection(z, alpha, tol=1e-14, iters=200):
    e0 = 1.0 / (alpha - 1.0)
    nvis = torch.isfinite(z).sum(dim=-1).to(z.dtype)
    lo = torch.zeros_like(nvis)
    hi = 1.0 - torch.pow(nvis, 1.0 - alpha)
    tau = lo.clone()
    done = hi <= lo
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        t = torch.clamp(z - mid.unsqueeze(-1), min=0.0)
        f = torch.where(t > 0, t ** e0, torch.zeros_like(t)).sum(dim=-1) - 1.0
        tau = torch.where(done, tau, mid)
        conv = f.abs() <= tol
        lo = torch.where(~done & ~conv & (f > 0), mid, lo)
        hi = torch.where(~done & ~conv & (f <= 0), mid, hi)
        done = done | conv
        if bool(done.all()):
            break
    return torch.where(hi <= 0.0, torch.zeros_like(tau), tau)


def dense_reference(q, k, v, alpha=1.5, causal=False, scale=0.0, block_r=64, block_c=64):
    """q [n, d], k [m, d], v [m, dv] (any float dtype; computed in fp64 on q's device).
    Returns dict(out, tau, row_max, mask_bits [t_r, t_c] bool)."""
    q, k, v = (x.to(torch.float64) for x in (q, k, v))
    n, d = q.shape
    m = k.shape[0]
    if n > 4096 or m > 4096:
        raise ValueError("dense_reference: capped at 4096 rows")
    sc = scale if scale > 0 else 1.0 / math.sqrt(d)
    z, mx = _center(q, k, alpha, sc, causal)
    tau = _tau_exact(z, alpha) if alpha in (1.5, 2.0) else _tau_bisection(z, alpha)
    t = z - tau.unsqueeze(-1)
    e0 = 1.0 / (alpha - 1.0)
    p = torch.where(t > 0, torch.clamp(t, min=0.0) ** e0, torch.zeros_like(t))
    out = p @ v
    t_r, t_c = -(-n // block_r), -(-m // block_c)
    pad = torch.zeros(t_r * block_r, t_c * block_c, dtype=torch.bool, device=q.device)
    pad[:n, :m] = p > 0
    bits = pad.reshape(t_r, block_r, t_c, block_c).any(dim=3).any(dim=1)
    return {"out": out, "tau": tau, "row_max": mx, "mask_bits": bits}
