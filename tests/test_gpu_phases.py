"""PhaseTimings (attention.hpp:62-66, filled at attention.cpp:196-199, 229-232,
329-332, 352): the GPU forward reports the time of its four reference phases
(row max, histogram, refinement, output) on both paths and both TC modes
(candidate lists / refinement sweeps), and the timed entry computes exactly
what the untimed one does."""
import pytest
import torch

import paper_2604_15180_b200 as pa

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.mark.parametrize("path,dtype,alpha", [("tc", torch.bfloat16, 1.5),
                                              ("tc", torch.bfloat16, 1.25),
                                              ("exact", torch.float32, 1.5)])
def test_phase_timings(path, dtype, alpha):
    g = torch.Generator(device="cpu").manual_seed(3)
    q, k, v = (torch.randn(1, 2, 2048, 128, generator=g).to(dtype).to(DEV) for _ in range(3))
    prob = pa.AttentionProblem(q, k, v, alpha=alpha, causal=True, path=path)
    pa.forward(prob)  # warm
    t = pa.PhaseTimings()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r1 = pa.forward(prob, 1, t)
    e1.record()
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1)
    print(path, alpha, [round(x, 3) for x in t.ms], round(total, 3))
    assert all(x > 0.0 for x in t.ms)
    assert sum(t.ms) <= 1.05 * total + 0.05
    r2 = pa.forward(prob)
    assert torch.equal(r1.tau, r2.tau) and torch.equal(r1.out, r2.out)
    assert torch.equal(r1.mask.words, r2.mask.words)
    # threads > 1: the reference leaves the timings untouched (attention.cpp:170)
    u = pa.PhaseTimings()
    pa.forward(prob, 4, u)
    assert u.ms == [0.0, 0.0, 0.0, 0.0]
