"""`atn attn` with the B200 backend: the record path
reproduces cmd_attn's inputs, keys and mask bytes (atn_main.cpp:224-328)."""
import io
import json
import os
from contextlib import redirect_stdout

import numpy as np
import pytest

from oracle.oracle import Oracle, Problem, gen_attn_inputs
from paper_2604_15180_b200 import atn

pytestmark = pytest.mark.gpu


def run(args):
    buf = io.StringIO()
    with redirect_stdout(buf):
        rc = atn.main(args)
    assert rc == 0
    return buf.getvalue()


@pytest.mark.parametrize("n,d,alpha,causal", [(256, 64, 1.5, True), (200, 32, 2.0, False)])
def test_attn_record_and_mask_bytes(tmp_path, n, d, alpha, causal):
    mask_path = str(tmp_path / "mask.bin")
    args = ["attn", "--n", str(n), "--d", str(d), "--alpha", str(alpha), "--seed", "5",
            "--verify", "--mask-out", mask_path] + (["--causal"] if causal else [])
    rec = json.loads(run(args))
    assert rec["experiment"] == "attn" and rec["seed"] == 5
    assert set(rec["params"]) == set(atn.PARAM_COLS)
    assert set(atn.METRIC_COLS[:10]) <= set(rec["metrics"])
    # the reference's own numbers for the same seed: stats and mask bytes identical
    # (f32 inputs run the exact path)
    orc = Oracle("reference")
    q, k, v, do = gen_attn_inputs(5, n, d, 1.0, orc)
    q, k, v, do = (x.astype(np.float32).astype(np.float64) for x in (q, k, v, do))
    ref = orc.forward(Problem(q, k, v, alpha=alpha, causal=causal))
    assert rec["metrics"]["blocks_visited_fwd"] == ref["blocks_visited_fwd"]
    assert rec["metrics"]["blocks_visited_bwd"] == 2 * ref["blocks_visited_fwd"]
    assert abs(rec["metrics"]["block_sparsity"] - ref["block_sparsity"]) < 1e-15
    t_r, t_c = -(-n // 64), -(-n // 64)
    expect = np.array([t_r, t_c], "<u4").tobytes() + ref["mask"].astype("<u4").tobytes()
    assert open(mask_path, "rb").read() == expect
    # against the dense fp64 reference: the 2-step forward's own tau error
    # (up to ~1e-2 at alpha=2, where Newton is unconverged after 2 steps)
    assert rec["metrics"]["max_abs_err_tau"] < 5e-2 and rec["metrics"]["max_abs_err_out"] < 1e-1
    csv = run([a for a in args if a not in ("--mask-out", mask_path)] + ["--out", "csv"]).splitlines()
    assert csv[0].split(",")[:4] == ["experiment", "seed", "n", "d"]
    assert len(csv) == 2
