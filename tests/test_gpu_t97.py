"""GPU parity for the paper's free-variable CDF 9/7 family (
sidwt_plan_set_lifting_t), including the irrational CDF 9/7 (t = SIDWT_CDF97_T_EXACT):
template taps, bands, correlation and peaks against the oracle run at the same t
(oracle.t97), through the SIMT path, the fused path, the tensor-core bank path and the
synthesis (perfect reconstruction)."""
import os

import numpy as np
import pytest

import oracle as O
import workloads as W

from parity import compare, oracle_for, run_gpu

pytestmark = pytest.mark.gpu

T_EXACT = 1.2301741049140007


def _plan(fam, J, N, batch, ext, tm, t, tc=None):
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    old = os.environ.get("SIDWT_TC")
    if tc is not None:
        os.environ["SIDWT_TC"] = tc
    try:
        return Plan(fam, J, N, batch, ext, lifting_t=t).load_templates(tm)
    finally:
        if old is None:
            os.environ.pop("SIDWT_TC", None)
        else:
            os.environ["SIDWT_TC"] = old


def _taps_match(plan, tm, t):
    got = plan.template_taps()
    with O.t97(t):
        for i in range(tm.shape[0]):
            ref = O.template_pyramid(O.CDF97, plan.levels, tm[i])
            for (k0, c), (k1, d) in zip(got[i], ref):
                assert k0 == k1 and len(c) == len(d)
                assert np.abs(c - d).max() <= 2e-7 * max(np.abs(d).max(), 1e-30)


@pytest.mark.parametrize("t", [T_EXACT, 0.8, 1.6])
@pytest.mark.parametrize("fused", [False, True])
def test_t97_config3_small(t, fused):
    """C3 shape (N = 8192, J = 6, symmetric, LFM 512) at other t."""
    cfg = W.CONFIGS[3]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, 2, tm)
    plan = _plan(cfg.family, cfg.levels, cfg.N, 2, cfg.ext, tm, t)
    _taps_match(plan, tm, t)
    g = run_gpu(plan, rows, fused=fused)
    with O.t97(t):
        r = oracle_for(plan, rows, tm)
    print(t, compare(plan, g, r))


@pytest.mark.parametrize("t", [T_EXACT, 1.85])
def test_t97_periodic_and_fused_kernel(t):
    from paper_cs_0607001_b200 import _native
    rng = np.random.default_rng(4242)
    N, J = 2048, 5
    tm = (rng.normal(size=(1, 100)) + 1j * rng.normal(size=(1, 100))).astype(np.complex64)
    rows = (rng.normal(size=(3, N)) + 1j * rng.normal(size=(3, N))).astype(np.complex64)
    plan = _plan(O.CDF97, J, N, 3, O.PERIODIC, tm, t)
    g = run_gpu(plan, rows, fused=True)
    with O.t97(t):
        r = oracle_for(plan, rows, tm)
    compare(plan, g, r)
    if plan.fused_available():
        import torch
        corr, lag, val = plan.analyze_correlate(plan.rows_to_device(rows), 3)
        torch.cuda.synchronize()
        assert np.array_equal(corr.cpu().numpy(), g["corr"]) and np.array_equal(lag.cpu().numpy(), g["lag"])
    assert _native.CDF97_T_EXACT == T_EXACT


def test_t97_tensor_core_bank():
    """C4 bank on rows cut to N = 4096 with the exact CDF 9/7 (tcgen05 path)."""
    cfg = W.CONFIGS[4]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, 2, tm)[:, 4096:8192].copy()
    plan = _plan(cfg.family, cfg.levels, 4096, 2, cfg.ext, tm, T_EXACT)
    assert plan.uses_tensor_cores()
    g = run_gpu(plan, rows, fused=True)
    with O.t97(T_EXACT):
        r = oracle_for(plan, rows, tm)
    compare(plan, g, r)


@pytest.mark.parametrize("ext", [0, 1])
def test_t97_synthesis_perfect_reconstruction(ext):
    import torch
    rng = np.random.default_rng(99 + ext)
    N, J = 4096, 5
    y = (rng.normal(size=(2, N)) + 1j * rng.normal(size=(2, N))).astype(np.complex64)
    tm = (rng.normal(size=(1, 40)) + 1j * rng.normal(size=(1, 40))).astype(np.complex64)
    plan = _plan(O.CDF97, J, N, 2, ext, tm, T_EXACT)
    bands = plan.analyze(plan.rows_to_device(y), 2)
    for level in (0, 2, J - 1):
        g = plan.synthesize(bands, 2, level).cpu().numpy()
        torch.cuda.synchronize()
        gc = g[..., 0].astype(np.float64) + 1j * g[..., 1]
        with O.t97(T_EXACT):
            ref = O.approx(O.CDF97, ext, N, y, level)
        for r in range(2):
            rel = np.sqrt((np.abs(gc[r] - ref[r]) ** 2).sum() / (np.abs(ref[r]) ** 2).sum())
            assert rel <= 1e-5, (level, r, rel)


def test_t97_status():
    from paper_cs_0607001_b200 import Plan, SidwtError, _native
    _native.build()
    with pytest.raises(SidwtError):
        Plan(O.LEGALL53, 3, 1024, 1, 0, lifting_t=1.3)          # not a 9/7 plan
    for bad in (0.5, 1.0, 2.0):
        with pytest.raises(SidwtError):
            Plan(O.CDF97, 3, 1024, 1, 0, lifting_t=bad)
    p = Plan(O.CDF97, 3, 1024, 1, 0).load_templates(np.ones((1, 16), np.complex64))
    with pytest.raises(SidwtError):
        _native.sidwt_plan_set_lifting_t(p.handle, 1.3)          # after template_load: STATE
