"""GPU parity of the EXACT (fp64 SIMT) path against the reference, through the
Python mirror of the reference interface and the C-ABI.

Bar: bit-identical tau / row_max / mask / out / delta / dq / dk / dv to the
reference for alpha in {1.5, 2} (the pow_e fast paths, internal.hpp:13-19); for
other alpha the reference calls std::pow, whose last-bit rounding differs from
CUDA's pow, so those compare within 1e-12 relative.  The fixtures in
tests/golden/ were produced by the compiled reference itself.
"""
import glob
import os

import numpy as np
import pytest
import torch

import paper_2604_15180_b200 as pa
from oracle.oracle import Oracle, Problem, gen_attn_inputs

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))
DEV = "cuda:0"


def np_(t):
    t = t.detach().cpu()
    if t.dtype == torch.int32:
        return t.numpy().view(np.uint32)
    return t.numpy()


def same(a, b, alpha, what):
    if alpha in (1.5, 2.0):
        assert np.array_equal(a, b), f"{what}: max|diff| {np.abs(a - b).max()}"
    else:
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-13, err_msg=what)


def run_gpu(q, k, v, do, dtype, **kw):
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV, dtype)
    prob = pa.AttentionProblem(T(q), T(k), T(v), path="exact", **kw)
    res = pa.forward(prob)
    grads = pa.backward(prob, res, T(do)) if do is not None else None
    torch.cuda.synchronize()
    return prob, res, grads


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_golden_bitwise(path, dtype):
    z = np.load(path)
    n, m, d, dv, alpha, causal, br, bc, bins, iters, tol = z["params"]
    alpha = float(alpha)
    kw = dict(alpha=alpha, causal=bool(causal), block_r=int(br), block_c=int(bc),
              bins=int(bins), refine_iters=int(iters), refine_tol=float(tol))
    prob, res, g = run_gpu(z["q"], z["k"], z["v"], z["dout"], dtype, **kw)
    assert np.array_equal(np_(res.mask.words), z["mask"])
    same(np_(res.row_max), z["row_max"], alpha, "row_max")
    same(np_(res.tau), z["tau"], alpha, "tau")
    same(np_(res.out), z["out"], alpha, "out")
    same(np_(g.delta), z["delta"], alpha, "delta")
    same(np_(g.dq), z["dq"], alpha, "dq")
    same(np_(g.dk), z["dk"], alpha, "dk")
    same(np_(g.dv), z["dv"], alpha, "dv")
    st = res.stats
    assert st.block_sparsity == float(z["block_sparsity"])
    assert st.blocks_visited_fwd == int(z["blocks_visited_fwd"])
    assert st.flushes == int(z["flushes"])
    assert 2 * st.blocks_visited_fwd == int(z["blocks_visited_bwd"])
    # compute_delta on its own equals the backward's delta pre-pass
    dl = pa.compute_delta(prob, res, torch.from_numpy(z["dout"]).to(DEV, dtype))
    assert torch.equal(dl, g.delta)


def test_kat_point_mass():
    # test_attention.cpp:107-131
    prob, res, g = run_gpu(np.array([[2.0]]), np.array([[1.0]]), np.array([[5.0]]),
                           np.array([[1.0]]), torch.float64, alpha=2.0, scale=1.0)
    assert res.out.item() == 5.0 and res.tau.item() == 0.0 and res.row_max.item() == 2.0
    assert res.mask.test(0, 0) and res.stats.blocks_visited_fwd == 1
    assert res.stats.block_sparsity == 0.0
    assert g.delta.item() == 5.0 and g.dv.item() == 1.0
    assert g.dk.item() == 0.0 and g.dq.item() == 0.0
    assert res.stats.blocks_visited_bwd == 2


def test_kat_two_key_sparsemax():
    # test_attention.cpp:133-163
    prob, res, g = run_gpu(np.array([[1.0], [1.0]]), np.array([[1.0], [0.5]]),
                           np.array([[2.0, 0.0], [0.0, 4.0]]), np.eye(2), torch.float64,
                           alpha=2.0, scale=1.0)
    assert np_(res.tau).tolist() == [0.25, 0.25]
    assert np_(res.out).tolist() == [[1.5, 1.0], [1.5, 1.0]]
    assert np_(g.delta).tolist() == [1.0, 2.0]
    np.testing.assert_allclose(np_(g.dq)[:, 0], [0.5, -1.0], rtol=1e-12)
    np.testing.assert_allclose(np_(g.dk)[:, 0], [-1.0, 1.0], rtol=1e-12)
    np.testing.assert_allclose(np_(g.dv), [[0.75, 0.75], [0.25, 0.25]], rtol=1e-12)


def test_config1_fp32_four_heads():
    """BASELINE config 1: alpha 1.5, causal, B=1 H=4 N=1024 d=64, fp32 inputs
    (cmd_attn's generator, one seed per head).  North-star bar: tau 1e-5 rel,
    out/grads 1e-5 abs; the exact path is bit-identical."""
    orc = Oracle("port")
    H, N, D = 4, 1024, 64
    qs, ks, vs, dos = [], [], [], []
    for h in range(H):
        q, k, v, do = gen_attn_inputs(1 + h, N, D, 1.0, orc)
        qs.append(q), ks.append(k), vs.append(v), dos.append(do)
    f32 = lambda xs: np.stack(xs)[None].astype(np.float32)
    Q, K, V, DO = f32(qs), f32(ks), f32(vs), f32(dos)
    prob, res, g = run_gpu(Q, K, V, DO, torch.float32, alpha=1.5, causal=True)
    steps = np_(res.row_steps)
    for h in range(H):
        pb = Problem(*(x[0, h].astype(np.float64) for x in (Q, K, V)), alpha=1.5, causal=True)
        f = orc.forward(pb, threads=8)
        b = orc.backward(pb, f, DO[0, h].astype(np.float64), threads=8)
        assert np.array_equal(np_(res.mask.words)[0, h], f["mask"])
        for key, gv in (("tau", res.tau), ("row_max", res.row_max), ("out", res.out)):
            assert np.array_equal(np_(gv)[0, h], f[key]), key
        for key, gv in (("dq", g.dq), ("dk", g.dk), ("dv", g.dv), ("delta", g.delta)):
            assert np.array_equal(np_(gv)[0, h], b[key]), key
        assert np.array_equal(steps[0, h], f["row_steps"])
    assert steps.mean() <= 2.0


def test_exact_tau_h_matches_restatement():
    """The histogram solution tau_h (private in the reference, attention.cpp:223)
    of the EXACT path equals the C restatement's bit for bit."""
    orc = Oracle("port")
    q, k, v, do = gen_attn_inputs(21, 512, 64, 1.0, orc)
    prob, res, _ = run_gpu(q, k, v, None, torch.float64, alpha=1.5, causal=True)
    th = torch.empty(512, dtype=torch.float64, device=DEV)
    pa.forward(prob, tau_h=th)
    fp = orc.forward_hist(Problem(q, k, v, alpha=1.5, causal=True), threads=4)
    assert np.array_equal(np_(th), fp["tau_h"])


def test_bf16_inputs_exact_path():
    orc = Oracle("port")
    q, k, v, do = gen_attn_inputs(77, 320, 64, 1.0, orc)
    bf = lambda a: torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16)
    Qb, Kb, Vb, Db = (bf(x) for x in (q, k, v, do))
    vals = [x.float().numpy().astype(np.float64) for x in (Qb, Kb, Vb, Db)]
    prob = pa.AttentionProblem(Qb.to(DEV), Kb.to(DEV), Vb.to(DEV), alpha=1.5, causal=True,
                               path="exact")
    res = pa.forward(prob)
    g = pa.backward(prob, res, Db.to(DEV))
    pb = Problem(vals[0], vals[1], vals[2], alpha=1.5, causal=True)
    f = orc.forward(pb)
    b = orc.backward(pb, f, vals[3])
    assert np.array_equal(np_(res.tau), f["tau"]) and np.array_equal(np_(res.out), f["out"])
    assert np.array_equal(np_(g.dq), b["dq"]) and np.array_equal(np_(g.dk), b["dk"])
    assert np.array_equal(np_(g.dv), b["dv"])


def test_batched_heads_match_single_head():
    orc = Oracle("port")
    rng = np.random.default_rng(5)
    B, H, N, D = 2, 3, 200, 32
    Q, K, V, DO = (rng.standard_normal((B, H, N, D)).astype(np.float32) for _ in range(4))
    prob, res, g = run_gpu(Q, K, V, DO, torch.float32, alpha=2.0, causal=False, block_c=32)
    for b_ in range(B):
        for h in range(H):
            pb = Problem(*(x[b_, h].astype(np.float64) for x in (Q, K, V)), alpha=2.0,
                         block_c=32)
            f = orc.forward(pb, threads=4)
            gb = orc.backward(pb, f, DO[b_, h].astype(np.float64), threads=4)
            assert np.array_equal(np_(res.out)[b_, h], f["out"])
            assert np.array_equal(np_(g.dk)[b_, h], gb["dk"])


def test_validation_raises_reference_messages():
    x = torch.zeros(8, 4, device=DEV)
    with pytest.raises(ValueError, match="alpha must exceed 1"):
        pa.forward(pa.AttentionProblem(x, x, x, alpha=1.0))
    with pytest.raises(ValueError, match="causal needs square"):
        y = torch.zeros(6, 4, device=DEV)
        pa.forward(pa.AttentionProblem(x, y, y, causal=True))
    with pytest.raises(ValueError, match="bins must divide"):
        pa.forward(pa.AttentionProblem(x, x, x, bins=5))
    with pytest.raises(ValueError, match="q/k width mismatch"):
        pa.forward(pa.AttentionProblem(x, torch.zeros(8, 3, device=DEV), x))


def test_mask_serialize_layout():
    prob, res, _ = run_gpu(*(np.random.default_rng(2).standard_normal((100, 8)) for _ in range(3)),
                           None, torch.float32, block_r=16, block_c=16)
    raw = res.mask.serialize()
    assert raw[:8] == (7).to_bytes(4, "little") + (7).to_bytes(4, "little")
    assert len(raw) == 8 + 7 * 4
    assert pa.block_sparsity(res.mask, False) == res.stats.block_sparsity


GENERIC = [
    # (n, m, d, dv, alpha, causal, block_r, block_c, bins)
    (200, 200, 200, 150, 1.5, True, 128, 96, 8),
    (150, 170, 40, 260, 2.0, False, 80, 70, 8),
    (130, 130, 130, 64, 2.5, True, 100, 128, 4),
    (190, 190, 16, 16, 1.25, True, 65, 200, 32),
    (97, 61, 300, 129, 1.5, False, 256, 32, 16),
]


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("case", GENERIC, ids=[str(c) for c in GENERIC])
def test_generic_blocks_and_widths_bitwise(case, dtype):
    """Blocks larger than 64 and widths above 128 (which the reference's validate
    accepts, attention.cpp:42-63) run on the one-thread-per-row EXACT kernels
    (exact_generic.cu) and stay bit-identical to the compiled reference."""
    n, m, d, dv, alpha, causal, br, bc, bins = case
    rng = np.random.default_rng(n * 3 + d)
    cast = (lambda a: a.astype(np.float32).astype(np.float64)) if dtype == torch.float32 else (lambda a: a)
    q = cast(rng.standard_normal((n, d)) * 1.5)
    k = cast(rng.standard_normal((m, d)))
    v = cast(rng.standard_normal((m, dv)))
    do = cast(rng.standard_normal((n, dv)))
    kw = dict(alpha=alpha, causal=causal, block_r=br, block_c=bc, bins=bins)
    prob, res, g = run_gpu(q, k, v, do, dtype, **kw)
    ref = Oracle("reference")
    pb = Problem(q, k, v, **kw)
    f = ref.forward(pb, threads=8)
    b = ref.backward(pb, f, do, threads=8)
    assert np.array_equal(np_(res.mask.words), f["mask"])
    same(np_(res.row_max), f["row_max"], alpha, "row_max")
    same(np_(res.tau), f["tau"], alpha, "tau")
    same(np_(res.out), f["out"], alpha, "out")
    for key in ("delta", "dq", "dk", "dv"):
        same(np_(getattr(g, key)), b[key], alpha, key)
    st = res.stats
    assert st.block_sparsity == f["block_sparsity"]
    assert st.blocks_visited_fwd == f["blocks_visited_fwd"]
    assert st.flushes == f["flushes"]
    assert res.stats.blocks_visited_bwd == b["blocks_visited_bwd"]
