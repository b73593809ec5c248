"""B200-native AdaSplash-2 alpha-entmax attention (forward + backward).

Drop-in for the reference's tiled attention path
(/root/reference/proj/include/adattn/attention.hpp): hand-written sm_100a CUDA
kernels behind a C-ABI (include/adattn_b200.h, libadattn_b200.so), with a
Python mirror of the reference interface in :mod:`.attention`.
"""
from .attention import (AttentionGradients, AttentionProblem, AttentionResult, AttentionStats,
                        BlockLists, NonzeroBlockLists, PackedBlockMask, PhaseTimings, backward,
                        block_lists,
                        block_sparsity, compute_delta, forward)

__all__ = [
    "AttentionProblem", "AttentionResult", "AttentionGradients", "AttentionStats",
    "PackedBlockMask", "PhaseTimings", "forward", "compute_delta", "backward", "block_sparsity",
    "BlockLists", "block_lists", "NonzeroBlockLists",
]
