"""Nonzero-block lists (adattn_b200_block_lists): the per-row-block lists of
active key blocks in PackedBlockMask::for_each_set order (bitpack.hpp:85-92)
and the transposed lists (PackedBlockMask::transposed, bitpack.cpp:138-143),
checked against a direct restatement over the mask words."""
import numpy as np
import pytest
import torch

import paper_2604_15180_b200 as pa
from paper_2604_15180_b200 import workloads

pytestmark = pytest.mark.gpu


def expected_lists(words, t_r, t_c):
    w = words.cpu().view(torch.int32).numpy().view(np.uint32).reshape(-1, t_r, (t_c + 31) // 32)
    rowptr, cols, colptr, rows = [0], [], [0], []
    for h in range(w.shape[0]):
        for i in range(t_r):
            for m, word in enumerate(w[h, i]):  # for_each_set: words in order, bits LSB-first
                word = int(word)
                while word:
                    b = (word & -word).bit_length() - 1
                    word &= word - 1
                    cols.append(32 * m + b)
            rowptr.append(len(cols))
        for j in range(t_c):
            for i in range(t_r):
                if (int(w[h, i, j // 32]) >> (j % 32)) & 1:
                    rows.append(i)
            colptr.append(len(rows))
    return rowptr, cols, colptr, rows


@pytest.mark.parametrize("causal,beta,heads", [(True, None, 2), (True, 0.8, 3), (False, 0.7, 2)])
def test_block_lists_match_mask(causal, beta, heads):
    N, D = 2048, 128
    if beta is None:
        q, k, v, _ = workloads.gaussian(1, heads, N, D, 1.0, seed=5)
    else:
        q, k, v, _ = workloads.anchored(1, heads, N, D, beta, causal, seed=5)
    prob = pa.AttentionProblem(q, k, v, path="tc", alpha=1.5, causal=causal)
    res = pa.forward(prob)
    bl = pa.block_lists(prob, res)
    torch.cuda.synchronize()
    rp, cl, cp, rw = expected_lists(res.mask.words, res.mask.t_r, res.mask.t_c)
    assert bl.rowptr.cpu().tolist() == rp
    assert bl.cols.cpu().tolist() == cl
    assert bl.colptr.cpu().tolist() == cp
    assert bl.rows.cpu().tolist() == rw
    assert rp[-1] == res.stats.blocks_visited_fwd
