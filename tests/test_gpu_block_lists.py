"""The nonzero-block lists (north_star item 3): emitted by the forward kernels
(tc_fwd.cu, per row block its active key blocks ascending; EXACT path: built
from its mask), walked by the output pass and -- with their transpose -- by the
backward kernels.  They must equal the reference's PackedBlockMask::for_each_set
order (bitpack.hpp:85-92) of the mask the forward returns, and the backward must
give identical results whether it walks the forward's lists or lists rebuilt
from the mask."""
import numpy as np
import pytest
import torch

import paper_2604_15180_b200 as pa

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def rows_from_mask(words, t_c):
    w = words.cpu().numpy().view(np.uint32)
    bits = np.unpackbits(w.view(np.uint8), bitorder="little").reshape(*w.shape[:-1], -1)[..., :t_c]
    return bits.astype(bool)


@pytest.mark.parametrize("path,dtype,n,m,causal,beta", [
    ("tc", torch.bfloat16, 2048, 2048, True, None),
    ("tc", torch.bfloat16, 4096, 4096, True, 0.8),
    ("tc", torch.bfloat16, 1000, 1000, True, None),     # ragged (padded execution)
    ("tc", torch.bfloat16, 700, 1300, False, None),
    ("exact", torch.float32, 300, 300, True, None),
])
def test_forward_emits_lists_and_backward_walks_them(path, dtype, n, m, causal, beta):
    from paper_2604_15180_b200 import workloads
    if beta is None:
        g = torch.Generator(device="cpu").manual_seed(n + m)
        q = torch.randn(1, 2, n, 128, generator=g).to(dtype).to(DEV)
        k, v = (torch.randn(1, 2, m, 128, generator=g).to(dtype).to(DEV) for _ in range(2))
        do = torch.randn(1, 2, n, 128, generator=g).to(dtype).to(DEV)
    else:
        q, k, v, do = workloads.anchored(1, 2, n, 128, beta, causal, seed=3, device=DEV,
                                         dtype=dtype)
    prob = pa.AttentionProblem(q, k, v, alpha=1.5, causal=causal, path=path)
    res = pa.forward(prob)
    torch.cuda.synchronize()
    t_r, t_c = res.mask.t_r, res.mask.t_c
    bits = rows_from_mask(res.mask.words, t_c)          # [1, 2, t_r, t_c]
    cnt = res.lists.cnt.cpu().numpy()
    cols = res.lists.cols.cpu().numpy().view(np.uint16)
    for h in range(2):
        for i in range(t_r):
            want = np.nonzero(bits[0, h, i])[0]
            assert cnt[0, h, i] == want.size
            assert np.array_equal(cols[0, h, i, :want.size], want)
    print(path, n, m, causal, beta, "nnz", int(cnt.sum()), "of", bits.size)
    g1 = pa.backward(prob, res, do)                      # walks the forward's lists
    res.lists = None
    g2 = pa.backward(prob, res, do)                      # lists rebuilt from the mask
    torch.cuda.synchronize()
    for name in ("dq", "dk", "dv", "delta"):
        assert torch.equal(getattr(g1, name), getattr(g2, name)), name
