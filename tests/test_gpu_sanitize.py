"""Every kernel of libsidwt on small inputs, compared with the oracle: the workload that
tools/gpu_round.sh runs under compute-sanitizer (memcheck, racecheck, synccheck, initcheck),
one tool per GPU call.  C1 at full size and C2-C5 on reduced batches, plus the variants that
take different kernels: fused analyze->correlate, peaks-only, standalone peaks, synthesis,
the paper's orientation, taps in shared memory, the template-bank and single-template
tensor-core kernels."""
import os

import numpy as np
import pytest

import oracle as O
import workloads as W

from parity import compare, oracle_for, run_gpu

pytestmark = pytest.mark.gpu


def _plan(cfg, batch, tm, **kw):
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    return Plan(cfg.family, cfg.levels, cfg.N, batch, cfg.ext, **kw).load_templates(tm)


@pytest.mark.parametrize("cid,nrows,nt", [(1, 1, 1), (2, 4, 1), (3, 2, 1), (4, 2, 16), (5, 4, 1)])
def test_kernels_small(cid, nrows, nt):
    import torch
    cfg = W.CONFIGS[cid]
    tm = W.templates(cfg)[:nt * (4 if cid == 4 else 1):(4 if cid == 4 else 1)].copy()
    rows = W.make_rows(cfg, 0, nrows, W.templates(cfg))
    plan = _plan(cfg, nrows, tm)
    r = oracle_for(plan, rows, tm)
    compare(plan, run_gpu(plan, rows, fused=False), r)      # analyze, correlate, peaks
    g = run_gpu(plan, rows, fused=True)                      # correlate_peaks
    compare(plan, g, r)
    d_rows = plan.rows_to_device(rows)
    _, lag, _ = plan.correlate_peaks(plan.analyze(d_rows, nrows), nrows, want_corr=False)   # peaks only
    if plan.fused_available():
        corr, flag, fval = plan.analyze_correlate(d_rows, nrows)                             # k_fused
        torch.cuda.synchronize()
        gf = dict(bands=g["bands"], corr=corr.cpu().numpy(), lag=flag.cpu().numpy(), val=fval.cpu().numpy())
        if plan.tensor_core_path() == 0:          # same SIMT arithmetic: bit-identical
            assert np.array_equal(gf["lag"], g["lag"]) and np.array_equal(gf["corr"], g["corr"])
        compare(plan, gf, r)
    out = plan.synthesize(plan.analyze(d_rows, nrows), nrows, 0)                             # k_synthesize
    torch.cuda.synchronize()
    assert np.array_equal(lag.cpu().numpy(), g["lag"])
    o = out.cpu().numpy()
    if plan.is_int:
        assert np.array_equal(o, rows.astype(np.int32))
    else:
        rec = o[..., 0] + 1j * o[..., 1]
        assert np.abs(rec - rows).max() <= 1e-4 * max(np.abs(rows).max(), 1.0)


def test_variants_small():
    """Paper orientation (template tree) and shared-memory taps on a C1-sized plan."""
    cfg = W.CONFIGS[1]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, 1, tm)
    p = _plan(cfg, 1, tm, orientation=1)
    g = run_gpu(p, rows, fused=True)
    r = O.run_paper(cfg.family, cfg.levels, cfg.ext, cfg.N, rows, tm)
    c = g["corr"][..., 0] + 1j * g["corr"][..., 1]
    assert (np.abs(c - r["corr"]).max(-1) / np.abs(r["corr"]).max(-1)).max() <= 1e-4
    os.environ["SIDWT_CTAPS"] = "0"
    try:
        p2 = _plan(cfg, 1, tm)
    finally:
        os.environ.pop("SIDWT_CTAPS", None)
    compare(p2, run_gpu(p2, rows, fused=True), oracle_for(p2, rows, tm))
