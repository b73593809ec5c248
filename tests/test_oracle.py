"""Pins the CPU oracle (test infrastructure) before anything trusts it.

* the plain-C restatement (oracle/liboracle.so, "port") is checked bit-for-bit
  against the reference itself compiled from /root/reference sources
  (oracle/_ref/libadattn_ref.so, "reference") on randomized configs modelled on
  test_attention.cpp:165-215 and on the committed golden fixtures;
* both are checked against the reference test-suite's known-answer values
  (test_attention.cpp:107-163, test_histogram.cpp:76-113, test_entmax.cpp:90-110,
  test_hybrid.cpp:48-80) and the RNG vectors SURVEY.md §8c pins.
"""
import glob
import math
import os
import subprocess

import numpy as np
import pytest

from oracle.oracle import Oracle, OracleError, Problem, REF_LIB, gen_attn_inputs

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))

have_ref = os.path.exists(REF_LIB)
KINDS = ["port"] + (["reference"] if have_ref else [])


@pytest.fixture(scope="module")
def port():
    return Oracle("port")


@pytest.fixture(scope="module")
def ref():
    if not have_ref:
        pytest.skip("oracle/_ref not built")
    return Oracle("reference")


def golden_problem(z):
    n, m, d, dv, alpha, causal, br, bc, bins, iters, tol = z["params"]
    return Problem(z["q"], z["k"], z["v"], alpha=float(alpha), causal=bool(causal),
                   block_r=int(br), block_c=int(bc), bins=int(bins), refine_iters=int(iters),
                   refine_tol=float(tol))


@pytest.mark.parametrize("kind", KINDS)
def test_rng_vectors(kind):
    o = Oracle(kind)
    assert [int(x) for x in o.xoshiro_next(1, 3)] == [
        0xCFC5D07F6F03C29B, 0xBF424132963FE08D, 0x19A37D5757AAF520]
    g = o.gaussian(1, 4)
    assert g.tolist() == [0.74977656920000146, 0.59456385456536842, -0.42669737721760126,
                          0.26274935681340256]


@pytest.mark.parametrize("kind", KINDS)
def test_kat_point_mass(kind):
    # test_attention.cpp:107-131
    o = Oracle(kind)
    pb = Problem(np.array([[2.0]]), np.array([[1.0]]), np.array([[5.0]]), alpha=2.0, scale=1.0)
    r = o.forward(pb)
    assert r["out"][0, 0] == 5.0 and r["tau"][0] == 0.0 and r["row_max"][0] == 2.0
    assert r["mask"][0, 0] == 1 and r["blocks_visited_fwd"] == 1 and r["block_sparsity"] == 0.0
    g = o.backward(pb, r, np.array([[1.0]]))
    assert g["delta"][0] == 5.0 and g["dv"][0, 0] == 1.0
    assert g["dk"][0, 0] == 0.0 and g["dq"][0, 0] == 0.0 and g["blocks_visited_bwd"] == 2


@pytest.mark.parametrize("kind", KINDS)
def test_kat_two_key_sparsemax(kind):
    # test_attention.cpp:133-163
    o = Oracle(kind)
    pb = Problem(np.array([[1.0], [1.0]]), np.array([[1.0], [0.5]]),
                 np.array([[2.0, 0.0], [0.0, 4.0]]), alpha=2.0, scale=1.0)
    r = o.forward(pb)
    assert r["tau"].tolist() == [0.25, 0.25]
    assert r["out"].tolist() == [[1.5, 1.0], [1.5, 1.0]]
    g = o.backward(pb, r, np.eye(2))
    assert g["delta"].tolist() == [1.0, 2.0]
    np.testing.assert_allclose(g["dq"][:, 0], [0.5, -1.0], rtol=1e-12)
    np.testing.assert_allclose(g["dk"][:, 0], [-1.0, 1.0], rtol=1e-12)
    np.testing.assert_allclose(g["dv"], [[0.75, 0.75], [0.25, 0.25]], rtol=1e-12)


@pytest.mark.parametrize("kind", KINDS)
def test_kat_histogram(kind):
    # test_histogram.cpp:76-113
    o = Oracle(kind)
    th, fl, lo, hi = o.solve_histogram([1, 0, 1, 1], 2.0)
    assert fl == 0 and th == pytest.approx(0.125) and (lo, hi) == pytest.approx((0.125, 0.375))
    th, fl, _, _ = o.solve_histogram([0, 0, 0, 0, 0, 0, 0, 2], 2.0)
    assert fl == 3 and th == pytest.approx(0.375)
    th, fl, _, _ = o.solve_histogram([0, 0, 0, 0, 0, 0, 0, 2], 1.5)
    assert fl == 1 and th == pytest.approx((1.75 - math.sqrt(2.0)) / 2.0)
    assert th == 0.16789321881345243  # SURVEY.md App. A, measured on the reference
    th, fl, _, _ = o.solve_histogram([0, 0, 0, 1], 2.0)
    assert th == 0.0 and fl == 0
    with pytest.raises(OracleError, match="empty histogram"):
        o.solve_histogram([0, 0, 0, 0], 1.5)
    with pytest.raises(OracleError, match="alpha must exceed 1"):
        o.solve_histogram([1, 1, 1, 1], 1.0)


@pytest.mark.parametrize("kind", KINDS)
def test_kat_f_eval(kind):
    # test_entmax.cpp:90-110: z=[1,1], alpha 1.5, tau .5 -> (-.5, -2, 4)
    o = Oracle(kind)
    assert o.f_eval([1.0, 1.0], 1.5, 0.5) == (-0.5, -2.0, 4.0)


def test_kat_newton_from_histogram(port):
    # test_hybrid.cpp:48-64: z=[1,1], alpha 2, B=8 -> tau_h=.375, f=.25, Newton -> .5, f=0
    th, _, lo, hi = port.solve_histogram([0, 0, 0, 0, 0, 0, 0, 2], 2.0)
    assert th == 0.375
    f, f1, f2 = port.f_eval([1.0, 1.0], 2.0, th)
    assert f == 0.25
    tau, kind = port.propose_step(2.0, th, f, f1, f2, 0.0, 0.0, lo, hi)
    assert kind == 2 and tau == 0.5 and port.f_eval([1.0, 1.0], 2.0, tau)[0] == 0.0


def test_kat_halley_two_steps(port):
    # test_hybrid.cpp:66-80 / SURVEY App. A: tau_h=0.1830582618 -> 0.2394408642
    s = np.array([1.0, 0.5, 0.25, -0.3])
    z = np.where(s == s.max(), 1.0, 0.5 * (s - s.max()) + 1.0)
    counts = np.zeros(8, dtype=np.uint32)
    for zi in z:
        if zi >= 0:
            counts[min(int(8 * zi), 7)] += 1
    th, _, lo, hi = port.solve_histogram(counts, 1.5)
    assert th == pytest.approx(0.18305826, rel=1e-6)
    tau = th
    for _ in range(2):
        f, f1, f2 = port.f_eval(z, 1.5, tau)
        if f > 0:
            lo = tau
        else:
            hi = tau
        tau, kind = port.propose_step(1.5, tau, f, f1, f2, 0.0, 0.0, lo, hi)
        assert kind == 1
    assert tau == pytest.approx(0.2394408642, rel=1e-9)
    assert abs(port.f_eval(z, 1.5, tau)[0]) <= 1e-6


@pytest.mark.skipif(not have_ref, reason="oracle/_ref not built")
def test_port_equals_reference_random(port, ref):
    """Bit-identical forward/backward on configs like test_attention.cpp:165-215,
    plus threads invariance (test_attention.cpp:287-307)."""
    rng = np.random.default_rng(424242)
    for rep in range(30):
        n = int(rng.integers(5, 97))
        causal = bool(rng.integers(0, 2))
        m = n if causal else int(rng.integers(5, 97))
        d = int(rng.integers(1, 9))
        dv = int(rng.integers(1, 9))
        alpha = [1.5, 2.0, 2.5, 1.25, 1.75][rep % 5]
        br = int(rng.choice([4, 8, 16, 64]))
        bc = int(rng.choice([4, 8, 16, 64]))
        bins = int(rng.choice([2, 4, 8, 16, 32]))
        iters = int(rng.choice([0, 1, 2, 3, 6]))
        qs = float(rng.choice([0.5, 1.0, 4.0, 30.0]))
        q = qs * rng.standard_normal((n, d))
        k = rng.standard_normal((m, d))
        v = rng.standard_normal((m, dv))
        do = rng.standard_normal((n, dv))
        pb = Problem(q, k, v, alpha=alpha, causal=causal, block_r=br, block_c=bc, bins=bins,
                     refine_iters=iters, refine_tol=1e-6)
        a = port.forward(pb, threads=1 + rep % 3)
        b = ref.forward(pb, threads=1 + (rep + 1) % 4)
        for key in ("out", "tau", "row_max", "mask"):
            assert np.array_equal(a[key], b[key]), (rep, key)
        for key in ("block_sparsity", "blocks_visited_fwd", "flushes"):
            assert a[key] == b[key], (rep, key)
        ga = port.backward(pb, a, do, threads=2)
        gb = ref.backward(pb, b, do, threads=3)
        for key in ("dq", "dk", "dv", "delta", "blocks_visited_bwd"):
            assert np.array_equal(ga[key], gb[key]), (rep, key)


@pytest.mark.skipif(not have_ref, reason="oracle/_ref not built")
def test_port_equals_reference_dense(port, ref):
    rng = np.random.default_rng(7)
    for alpha in (1.5, 2.0, 1.25):
        for causal in (False, True):
            n = 70
            q, k, v = (rng.standard_normal((n, 6)) for _ in range(3))
            pb = Problem(q, k, v, alpha=alpha, causal=causal, block_r=16, block_c=16)
            a, b = port.dense_reference(pb), ref.dense_reference(pb)
            for key in ("out", "tau", "row_max", "mask"):
                assert np.array_equal(a[key], b[key]), (alpha, causal, key)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_port_reproduces_golden(port, path):
    z = np.load(path)
    pb = golden_problem(z)
    f = port.forward(pb, threads=2)
    for key in ("out", "tau", "row_max", "mask"):
        assert np.array_equal(f[key], z[key]), key
    assert f["block_sparsity"] == float(z["block_sparsity"])
    assert f["flushes"] == int(z["flushes"])
    assert f["blocks_visited_fwd"] == int(z["blocks_visited_fwd"])
    g = port.backward(pb, f, z["dout"], threads=2)
    for key in ("dq", "dk", "dv", "delta"):
        assert np.array_equal(g[key], z[key]), key


@pytest.mark.parametrize("kind", KINDS)
def test_validation_messages(kind):
    o = Oracle(kind)
    rng = np.random.default_rng(1)
    q = rng.standard_normal((8, 4))
    cases = [
        (dict(causal=True, k=rng.standard_normal((6, 4)), v=rng.standard_normal((6, 4))),
         "causal needs square"),
        (dict(alpha=1.0), "alpha must exceed 1"),
        (dict(block_r=0), "bad tile size"),
        (dict(refine_tol=0.0), "bad refinement config"),
        (dict(bins=5), "bins must divide word_bits"),
    ]
    for kw, msg in cases:
        args = dict(q=q, k=q.copy(), v=q.copy(), block_r=4, block_c=4)
        args.update(kw)
        with pytest.raises(OracleError, match=msg):
            o.forward(Problem(**args))
    o.forward(Problem(q, q.copy(), q.copy(), bins=32, block_r=4, block_c=4))  # 128-bit words


def test_flush_count_512_tiles(port):
    # acceptance #9 analogue: 512 key tiles at 8 bits per bin -> 3 flushes per query tile
    n = 512 * 4
    rng = np.random.default_rng(3)
    q = rng.standard_normal((4, 2))
    k = rng.standard_normal((n, 2))
    f = port.forward(Problem(q, k, k.copy(), block_r=4, block_c=4))
    assert f["flushes"] == 3


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(REF_LIB), "acceptance")),
                    reason="reference acceptance binary not built")
def test_reference_acceptance_battery():
    """The reference's own acceptance battery (tests/acceptance_main.cpp): 8/10
    PASS + 2 known limits, 0 unexpected failures (README.md:56-59)."""
    exe = os.path.join(os.path.dirname(REF_LIB), "acceptance")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:]
    assert "8/10 criteria passed, 2 known limit(s), 0 unexpected failure(s)" in r.stdout


def test_gen_attn_inputs_order(port):
    q, k, v, do = gen_attn_inputs(5, 3, 2, 2.0, port)
    g = port.gaussian(5, 24)
    assert np.array_equal(q.ravel(), 2.0 * g[:6]) and np.array_equal(do.ravel(), g[18:])


def test_port_histogram_state_consistent_with_reference_solver():
    """orc_forward_ex's private histogram state: solving its counts with the
    reference's own solve_histogram (oracle/_ref) reproduces its tau_h, and the
    forward outputs equal the reference's forward bit for bit."""
    port, ref = Oracle("port"), Oracle("reference")
    q, k, v, _ = gen_attn_inputs(31, 300, 32, 2.0, port)
    for alpha, bins in ((1.5, 8), (2.0, 4), (1.25, 16)):
        pb = Problem(q, k, v, alpha=alpha, causal=True, bins=bins)
        fh = port.forward_hist(pb, threads=4)
        fr = ref.forward(pb, threads=4)
        assert np.array_equal(fh["tau"], fr["tau"]) and np.array_equal(fh["out"], fr["out"])
        for r in range(0, 300, 7):
            th, _, _, _ = ref.solve_histogram(fh["counts"][r], alpha)
            assert th == fh["tau_h"][r]
