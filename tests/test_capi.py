"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/adattn_b200.h declares, and host-side validation mirrors the
reference's validate() messages (attention.cpp:42-63, bitpack.cpp:55-65)."""
import ctypes as C
import os
import re

import pytest

from paper_2604_15180_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "adattn_b200.h")).read()
    return sorted(set(re.findall(r"\b(adattn_b200_\w+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.EXPORTS) == syms
    assert lib.adattn_b200_abi_version() == 2


def prob(**kw):
    base = dict(batch=1, heads=1, n=8, m=8, d=4, dv=4, alpha=1.5, scale=0.0, causal=0,
                block_r=4, block_c=4, bins=8, refine_iters=2, refine_tol=1e-6,
                in_dtype=_lib.F32, out_dtype=_lib.F64, path=_lib.PATH_AUTO, reserved=0)
    base.update(kw)
    return _lib.Problem(**base)


@pytest.mark.parametrize("kw,msg", [
    (dict(n=0), "attention: empty operand"),
    (dict(causal=1, m=6), "attention: causal needs square score matrix"),
    (dict(alpha=1.0), "attention: alpha must exceed 1"),
    (dict(block_r=0), "attention: bad tile size"),
    (dict(refine_iters=-1), "attention: bad refinement config"),
    (dict(refine_tol=0.0), "attention: bad refinement config"),
    (dict(bins=5), "PackedHistogramAcc: bins must divide word_bits"),
    (dict(bins=64), "PackedHistogramAcc: needs at least 4 bits per bin"),
])
def test_validate_messages(kw, msg):
    lib = _lib.load()
    p = prob(**kw)
    assert lib.adattn_b200_validate(C.byref(p)) == _lib.ADATTN_ERR_INVALID
    assert lib.adattn_b200_last_error().decode() == msg
    with pytest.raises(ValueError, match=re.escape(msg)):
        _lib.check(_lib.ADATTN_ERR_INVALID)


def test_valid_and_envelope():
    lib = _lib.load()
    assert lib.adattn_b200_validate(C.byref(prob(bins=32))) == 0  # 128-bit words
    assert lib.adattn_b200_validate(C.byref(prob(bins=2))) == 0
    assert lib.adattn_b200_resolved_path(C.byref(prob())) == _lib.PATH_EXACT
    # every problem the reference accepts has a GPU path: wide and large-tile
    # problems resolve to the exact kernels (exact_generic.cu)
    assert lib.adattn_b200_validate(C.byref(prob(d=256))) == 0
    assert lib.adattn_b200_validate(C.byref(prob(block_r=128))) == 0
    assert lib.adattn_b200_resolved_path(C.byref(prob(d=256, in_dtype=_lib.BF16))) == _lib.PATH_EXACT
    # the tensor-core path takes bf16 at d = dv in {64, 128} for any n, m
    assert lib.adattn_b200_resolved_path(C.byref(prob(d=128, dv=128, n=100, m=100,
                                                      block_r=64, block_c=64,
                                                      in_dtype=_lib.BF16))) == _lib.PATH_TC
    # fp32 inputs never take the tensor-core path
    assert lib.adattn_b200_validate(C.byref(prob(path=_lib.PATH_TC))) == _lib.ADATTN_ERR_UNSUPPORTED


def test_delta_aux_size_query():
    """adattn_b200_delta_aux_bytes (a pure host query, no GPU): the forward folds the
    delta accumulation (sum u V and sum u per row, [B][H][n][dv] then [B][H][n] float)
    only on the tensor-core path of unpadded problems, by default for alpha = 2."""
    lib = _lib.load()
    tc = dict(batch=2, heads=3, n=512, m=512, d=128, dv=128, causal=1, block_r=64, block_c=64,
              in_dtype=_lib.BF16, out_dtype=_lib.F32)
    old = os.environ.pop("ADATTN_DELTA_FOLD", None)
    try:
        assert lib.adattn_b200_delta_aux_bytes(C.byref(prob(alpha=2.0, **tc))) == 2 * 3 * 512 * 129 * 4
        assert lib.adattn_b200_delta_aux_bytes(C.byref(prob(alpha=1.5, **tc))) == 0
        assert lib.adattn_b200_delta_aux_bytes(C.byref(prob(alpha=2.0, **dict(tc, n=500, m=500)))) == 0
        assert lib.adattn_b200_delta_aux_bytes(C.byref(prob(alpha=2.0, **dict(tc, in_dtype=_lib.F32)))) == 0
        os.environ["ADATTN_DELTA_FOLD"] = "1"
        assert lib.adattn_b200_delta_aux_bytes(C.byref(prob(alpha=1.5, **tc))) == 2 * 3 * 512 * 129 * 4
        os.environ["ADATTN_DELTA_FOLD"] = "0"
        assert lib.adattn_b200_delta_aux_bytes(C.byref(prob(alpha=2.0, **tc))) == 0
    finally:
        os.environ.pop("ADATTN_DELTA_FOLD", None)
        if old is not None:
            os.environ["ADATTN_DELTA_FOLD"] = old
