"""GPU fused analyze -> correlate -> peaks: bit-identical corr and
peaks to the two-call path (same lifting and correlation code, same summation order), and
element-by-element parity with the oracle."""
import numpy as np
import pytest

import oracle as O
import workloads as W

from parity import compare, oracle_for, run_gpu

pytestmark = pytest.mark.gpu


def _fused(plan, rows, want_corr=True):
    import torch
    d = plan.rows_to_device(rows)
    corr, lag, val = plan.analyze_correlate(d, rows.shape[0], want_corr=want_corr)
    torch.cuda.synchronize()
    return (corr.cpu().numpy() if corr is not None else None), lag.cpu().numpy(), val.cpu().numpy()


@pytest.mark.parametrize("cid,nrows", [(1, 1), (2, 6), (3, 2), (5, 4)])
def test_fused_equals_two_call_path(cid, nrows, monkeypatch):
    """Bit-identical to the two-call path through the SIMT correlation (whose item code the
    fused kernel shares; SIDWT_TCS=0 keeps C3 off the tensor-core kernel for the comparison)."""
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    monkeypatch.setenv("SIDWT_TCS", "0")
    cfg = W.CONFIGS[cid]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, nrows, tm)
    plan = Plan(cfg.family, cfg.levels, cfg.N, nrows, cfg.ext).load_templates(tm)
    if not plan.fused_available():
        pytest.skip(f"{cfg.name}: no fused tiling")
    g = run_gpu(plan, rows, fused=True)
    fc, fl, fv = _fused(plan, rows)
    assert np.array_equal(fc, g["corr"]), "fused corr differs from the two-call path"
    assert np.array_equal(fl, g["lag"]) and np.array_equal(fv, g["val"])
    _, pl, pv = _fused(plan, rows, want_corr=False)             # peaks-only mode
    assert np.array_equal(pl, g["lag"]) and np.array_equal(pv, g["val"])
    r = oracle_for(plan, rows, tm)
    g2 = dict(g)
    g2.update(corr=fc, lag=fl, val=fv)
    compare(plan, g2, r)


FUSED_EDGE = [
    (0, 1, 0, 512, 1),
    (1, 3, 1, 1024, 64),
    (2, 4, 0, 2048, 130),
    (3, 6, 1, 4096, 50),
    (1, 2, 1, 16384, 300),
]


@pytest.mark.parametrize("fam,J,ext,N,T", FUSED_EDGE)
def test_fused_edge(fam, J, ext, N, T, monkeypatch):
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    monkeypatch.setenv("SIDWT_TCS", "0")
    rng = np.random.default_rng(9000 + fam * 7 + J + N)
    isint = fam == O.LEGALL53_INT
    if isint:
        tm = rng.integers(-2047, 2048, size=(1, T, 2)).astype(np.int16)
        rows = rng.integers(-3000, 3000, size=(2, N, 2)).astype(np.int16)
    else:
        tm = (rng.normal(size=(1, T)) + 1j * rng.normal(size=(1, T))).astype(np.complex64)
        rows = (rng.normal(size=(2, N)) + 1j * rng.normal(size=(2, N))).astype(np.complex64)
    plan = Plan(fam, J, N, 2, ext).load_templates(tm)
    assert plan.fused_available()
    g = run_gpu(plan, rows, fused=True)
    fc, fl, fv = _fused(plan, rows)
    assert np.array_equal(fc, g["corr"]) and np.array_equal(fl, g["lag"]) and np.array_equal(fv, g["val"])


def test_fused_unavailable_for_banks():
    from paper_cs_0607001_b200 import Plan, SidwtError, _native
    import torch
    _native.build()
    p = Plan(1, 3, 1024, 1, 1).load_templates(np.ones((4, 16), np.complex64))
    assert not p.fused_available()
    with pytest.raises(SidwtError) as e:
        p.analyze_correlate(torch.zeros(1, 1024, 2, device="cuda"), 1)
    assert e.value.status == 5


def test_fused_full_size_c2():
    """BASELINE C2 at full size through the fused call: equal to the two-call path on every row."""
    import torch
    cfg = W.CONFIGS[2]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, cfg.rows, tm)
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    plan = Plan(cfg.family, cfg.levels, cfg.N, cfg.rows, cfg.ext).load_templates(tm)
    assert plan.fused_available()
    d = plan.rows_to_device(rows)
    bands = plan.analyze(d, cfg.rows)
    corr, lag, val = plan.correlate_peaks(bands, cfg.rows)
    fcorr, flag, fval = plan.analyze_correlate(d, cfg.rows)
    torch.cuda.synchronize()
    assert torch.equal(corr, fcorr) and torch.equal(lag, flag) and torch.equal(val, fval)
