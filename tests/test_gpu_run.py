"""GPU whole-path call sidwt_run (analysis of row chunk k+1 overlapping the correlation of
chunk k on a second stream): bit-identical bands, corr and peaks to the two-call path
(analyze + correlate_peaks) for every chunk count, including chunk counts that do not
divide the rows, the tensor-core bank path and the peaks-only mode; and oracle parity."""
import os

import numpy as np
import pytest

import workloads as W

from parity import compare, oracle_for, run_gpu

pytestmark = pytest.mark.gpu


def _run(plan, rows, chunks, want_corr=True):
    import torch
    os.environ["SIDWT_RUN_CHUNKS"] = str(chunks)
    try:
        d = plan.rows_to_device(rows)
        bands = plan.empty_bands(rows.shape[0])
        corr, lag, val = plan.run(d, rows.shape[0], bands, want_corr=want_corr)
        torch.cuda.synchronize()
        launches = plan.last_launches()
    finally:
        del os.environ["SIDWT_RUN_CHUNKS"]
    return (bands.cpu().numpy(), corr.cpu().numpy() if corr is not None else None, lag.cpu().numpy(),
            val.cpu().numpy(), launches)


@pytest.mark.parametrize("cid,nrows", [(1, 1), (2, 7), (3, 3), (5, 5)])
@pytest.mark.parametrize("chunks", [1, 2, 3, 16])
def test_run_equals_two_call_path(cid, nrows, chunks):
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    cfg = W.CONFIGS[cid]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, nrows, tm)
    plan = Plan(cfg.family, cfg.levels, cfg.N, nrows, cfg.ext).load_templates(tm)
    g = run_gpu(plan, rows, fused=True)
    b, c, l, v, launches = _run(plan, rows, chunks)
    assert np.array_equal(b, g["bands"]), "run: bands differ from sidwt_analyze"
    assert np.array_equal(c, g["corr"]), "run: corr differs from the two-call path"
    assert np.array_equal(l, g["lag"]) and np.array_equal(v, g["val"])
    per_chunk = 2 if plan.tensor_core_path() in (2, 3) else 3        # analyze + correlate (+ peak finalize)
    assert launches == per_chunk * min(chunks, nrows)
    _, _, pl, pv, _ = _run(plan, rows, chunks, want_corr=False)         # peaks only
    assert np.array_equal(pl, g["lag"]) and np.array_equal(pv, g["val"])
    if chunks == 3:
        compare(plan, dict(bands=b, corr=c, lag=l, val=v), oracle_for(plan, rows, tm))


def test_run_tensor_core_bank():
    """C4-shaped bank (64 templates) on a few rows: the tcgen05 path under sidwt_run."""
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    cfg = W.CONFIGS[4]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, 5, tm)
    plan = Plan(cfg.family, cfg.levels, cfg.N, 5, cfg.ext).load_templates(tm)
    assert plan.uses_tensor_cores()
    g = run_gpu(plan, rows, fused=True)
    b, c, l, v, _ = _run(plan, rows, 2)
    assert np.array_equal(c, g["corr"]) and np.array_equal(l, g["lag"]) and np.array_equal(v, g["val"])
