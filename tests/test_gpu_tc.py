"""GPU parity of the tensor-core template-bank correlation (csrc/corr_tc.cuh).

The bank path (tcgen05.mma, bf16x3 split, fp32 accumulation in TMEM) is taken
for float families when n_templates >= 16 and N is a multiple of 512; SIDWT_TC=1
forces it for smaller banks, SIDWT_TC=0 disables it.  Every case is compared
element by element with the CPU oracle (fp64), same tolerances as the SIMT path.
"""
import os

import numpy as np
import pytest

import oracle as O
import workloads as W

from parity import compare, oracle_for, run_gpu

pytestmark = pytest.mark.gpu


def _plan(fam, J, N, rows, ext, tm, force=None):
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    old = os.environ.get("SIDWT_TC")
    if force is not None:
        os.environ["SIDWT_TC"] = force
    try:
        return Plan(fam, J, N, rows, ext).load_templates(tm)
    finally:
        if old is None:
            os.environ.pop("SIDWT_TC", None)
        else:
            os.environ["SIDWT_TC"] = old


def test_tc_c4_bank_reduced_n():
    """C4 bank (64 Doppler-shifted LFM templates, 9/7, J=4, symmetric) on rows cut to N=4096."""
    cfg = W.CONFIGS[4]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, 2, tm)[:, 4096:8192].copy()
    plan = _plan(cfg.family, cfg.levels, 4096, 2, cfg.ext, tm)
    assert plan.uses_tensor_cores()
    g = run_gpu(plan, rows, fused=True)
    r = oracle_for(plan, rows, tm)
    st = compare(plan, g, r)
    print("tc C4 N=4096", st)


def test_tc_matches_simt_path():
    """Same inputs through the tensor-core and the SIMT correlation: both within tolerance of
    the oracle, and of each other."""
    cfg = W.CONFIGS[4]
    tm = W.templates(cfg)[:16].copy()
    rows = W.make_rows(cfg, 0, 2, W.templates(cfg))[:, :2048].copy()
    p_tc = _plan(cfg.family, cfg.levels, 2048, 2, cfg.ext, tm, force="1")
    p_si = _plan(cfg.family, cfg.levels, 2048, 2, cfg.ext, tm, force="0")
    assert p_tc.uses_tensor_cores() and not p_si.uses_tensor_cores()
    g1 = run_gpu(p_tc, rows, fused=True)
    g2 = run_gpu(p_si, rows, fused=True)
    r = oracle_for(p_tc, rows, tm)
    compare(p_tc, g1, r)
    compare(p_si, g2, r)
    assert np.array_equal(g1["bands"], g2["bands"])


TC_EDGE = [
    # family, J, ext, N, T, n_templates
    (0, 3, 0, 1024, 64, 16),       # LeGall 5/3, periodic (wrapped band reads)
    (2, 5, 1, 2048, 130, 20),      # causal D4, symmetric, ragged last template tile
    (1, 6, 1, 2048, 200, 70),      # 9/7, g = 64 (zero-stuffed taps, f = 8), two template tiles
    (1, 1, 1, 512, 40, 64),        # one level, smallest N the path takes
    (0, 2, 1, 1024, 1, 32),        # T = 1
]


@pytest.mark.parametrize("fam,J,ext,N,T,nt", TC_EDGE)
def test_tc_edge(fam, J, ext, N, T, nt):
    rng = np.random.default_rng(4242 + fam * 10 + J + nt)
    tm = (rng.normal(size=(nt, T)) + 1j * rng.normal(size=(nt, T))).astype(np.complex64)
    rows = (rng.normal(size=(2, N)) + 1j * rng.normal(size=(2, N))).astype(np.complex64)
    rows[1, 100:100 + T] += 3 * tm[nt // 2]                          # a clear peak for one template
    plan = _plan(fam, J, N, 2, ext, tm, force="1")
    assert plan.uses_tensor_cores()
    g = run_gpu(plan, rows, fused=True)
    g2 = run_gpu(plan, rows, fused=False)
    assert np.array_equal(g["corr"], g2["corr"])
    r = oracle_for(plan, rows, tm)
    compare(plan, g, r)


def test_tc_full_size_c4_sampled():
    """BASELINE C4 at full size (2048 x 16384, 64 templates) in bench.py's launch
    configuration (corr written + fused peaks); sampled rows against the oracle."""
    import torch
    cfg = W.CONFIGS[4]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, cfg.rows, tm)
    plan = _plan(cfg.family, cfg.levels, cfg.N, cfg.rows, cfg.ext, tm)
    assert plan.uses_tensor_cores()
    d_rows = plan.rows_to_device(rows)
    bands = plan.analyze(d_rows, cfg.rows)
    corr, lag, val = plan.correlate_peaks(bands, cfg.rows)
    torch.cuda.synchronize()
    ids = [0, 777, cfg.rows - 1]
    g = dict(bands=bands[ids].cpu().numpy(), corr=corr[ids].cpu().numpy(),
             lag=lag[ids].cpu().numpy(), val=val[ids].cpu().numpy())
    del corr
    r = oracle_for(plan, rows[ids], tm)
    st = compare(plan, g, r)
    lg = lag.cpu().numpy()
    assert lg.min() >= 0 and lg.max() < cfg.N
    print("tc C4 full-size sampled", st)
