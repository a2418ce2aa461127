"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Small cases run every row through the oracle; the full-size cases run the whole
BASELINE batch on the GPU in the launch configuration bench.py times and check
a seeded sample of rows (first, last, and spread) against the oracle.
"""
import numpy as np
import pytest

import oracle as O
import workloads as W

from parity import compare, oracle_for, run_gpu

pytestmark = pytest.mark.gpu


def _plan(cfg, batch, templates):
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    return Plan(cfg.family, cfg.levels, cfg.N, batch, cfg.ext).load_templates(templates)


def _taps_match(plan, templates):
    """Device template pyramid (fp64 lifting on the GPU, stored fp32/int32) vs the oracle's
    Mallat pyramid: same supports; values within fp32 rounding (exact for the integer family)."""
    got = plan.template_taps()
    for t in range(templates.shape[0]):
        ref = O.template_pyramid(plan.filter, plan.levels, templates[t])
        for (k0, c), (k1, d) in zip(got[t], ref):
            assert k0 == k1 and len(c) == len(d)
            if plan.is_int:
                assert np.array_equal(np.asarray(c, np.int64), d)
            else:
                scale = max(np.abs(d).max(), 1e-30)
                assert np.abs(c - d).max() <= 2e-7 * scale


@pytest.mark.parametrize("cid,nrows", [(1, 1), (2, 4), (3, 3), (5, 4)])
@pytest.mark.parametrize("fused", [False, True])
def test_config_small(cid, nrows, fused):
    cfg = W.CONFIGS[cid]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, nrows, tm)
    plan = _plan(cfg, nrows, tm)
    _taps_match(plan, tm)
    g = run_gpu(plan, rows, fused=fused)
    r = oracle_for(plan, rows, tm)
    st = compare(plan, g, r, neartie_bound=True)
    print(cfg.name, st)


def test_config4_bank_small():
    """C4 shape (N=16384, J=4, 9/7, symmetric) against a sub-bank of 8 templates."""
    cfg = W.CONFIGS[4]
    tm = W.templates(cfg)[::8].copy()
    rows = W.make_rows(cfg, 0, 2, W.templates(cfg))
    plan = _plan(cfg, 2, tm)
    _taps_match(plan, tm)
    g = run_gpu(plan, rows, fused=True)
    r = oracle_for(plan, rows, tm)
    compare(plan, g, r)


EDGE = [
    # family, J, ext, N, T, rows-kind
    (0, 3, 0, 8, 8, "random"),        # N = 2^J, T = N
    (1, 3, 1, 8, 8, "random"),
    (2, 3, 1, 8, 3, "random"),
    (3, 3, 1, 8, 8, "random"),
    (0, 1, 0, 2, 1, "random"),        # smallest plan
    (1, 1, 1, 2, 2, "random"),
    (3, 1, 1, 2, 1, "random"),
    (1, 5, 1, 64, 1, "random"),       # T = 1
    (0, 4, 1, 256, 40, "zero"),       # all-zero rows
    (1, 4, 1, 256, 40, "dc"),         # DC rows
    (2, 4, 1, 256, 40, "impulse"),    # impulses at 0 and N-1
    (3, 4, 1, 256, 40, "impulse"),
    (1, 6, 0, 4096, 300, "random"),   # periodic, deep, multi-tile K1/K2
    (2, 7, 1, 8192, 130, "random"),
    (0, 9, 1, 2048, 100, "random"),   # 2^J = 512 > K2 tile residues
    (3, 10, 1, 4096, 64, "random"),
    (1, 2, 1, 32768, 700, "random"),  # many K1 / K2 tiles, ragged last K1 tile
]


@pytest.mark.parametrize("fam,J,ext,N,T,kind", EDGE)
def test_edge_cases(fam, J, ext, N, T, kind):
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    rng = np.random.default_rng(1000 + 7 * fam + J + N)
    nrows = 2
    isint = fam == O.LEGALL53_INT
    if isint:
        tm = rng.integers(-2047, 2048, size=(1, T, 2)).astype(np.int16)
        rows = rng.integers(-3000, 3000, size=(nrows, N, 2)).astype(np.int16)
    else:
        tm = (rng.normal(size=(1, T)) + 1j * rng.normal(size=(1, T))).astype(np.complex64)
        rows = (rng.normal(size=(nrows, N)) + 1j * rng.normal(size=(nrows, N))).astype(np.complex64)
    if kind == "zero":
        rows[...] = 0
    elif kind == "dc":
        rows[...] = (1.5 - 0.5j) if not isint else 700
    elif kind == "impulse":
        rows[...] = 0
        if isint:
            rows[0, 0] = (2047, -2047)
            rows[1, N - 1] = (-2047, 1000)
        else:
            rows[0, 0] = 1 + 1j
            rows[1, N - 1] = 2 - 1j
    plan = Plan(fam, J, N, nrows, ext).load_templates(tm)
    _taps_match(plan, tm)
    g = run_gpu(plan, rows, fused=True)
    g2 = run_gpu(plan, rows, fused=False)
    assert np.array_equal(g["corr"], g2["corr"]) and np.array_equal(g["lag"], g2["lag"])
    r = oracle_for(plan, rows, tm)
    compare(plan, g, r)


def test_status_codes_on_device():
    from paper_cs_0607001_b200 import Plan, SidwtError, _native
    import torch
    _native.build()
    p = Plan(0, 3, 64, 2, 0)
    d = torch.zeros(2, 64, 2, device="cuda")
    b = torch.zeros(1 << 16, device="cuda")
    with pytest.raises(SidwtError) as e:
        _native.sidwt_analyze(p.handle, d, 2, b)
    assert e.value.status == 6                       # STATE: no template yet
    p.load_templates(np.ones((1, 8), np.complex64))
    with pytest.raises(SidwtError) as e:
        _native.sidwt_analyze(p.handle, d, 3, b)     # rows > batch
    assert e.value.status == 3
    with pytest.raises(SidwtError) as e:
        p.load_templates(np.ones((1, 65), np.complex64))
    assert e.value.status == 2                       # T > N


def test_execute_host_matches_device_path():
    import torch
    cfg = W.CONFIGS[2]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, 8, tm)
    plan = _plan(cfg, 8, tm)
    g = run_gpu(plan, rows, fused=True)
    lag = np.zeros((8, 1, cfg.levels + 1), np.int32)
    val = np.zeros((8, 1, cfg.levels + 1, 2), np.float32)
    plan.execute_host(np.ascontiguousarray(rows), 8, lag, val)
    torch.cuda.synchronize()
    assert np.array_equal(lag, g["lag"]) and np.array_equal(val, g["val"])


# ------------------------------------------------------------------ full BASELINE sizes

def _sample_rows(cfg, n):
    """n seeded row ids spread over the batch, always the first and the last (BASELINE.md
    section 3: >= 256 rows for C2/C3/C5, 16 pulses for C4)."""
    if n >= cfg.rows:
        return list(range(cfg.rows))
    rng = np.random.default_rng(np.random.SeedSequence([W.SEED_TAG, cfg.cid, 0xB]))
    ids = set(rng.choice(np.arange(1, cfg.rows - 1), size=n - 2, replace=False).tolist())
    return sorted(ids | {0, cfg.rows - 1})


@pytest.mark.parametrize("cid", [2, 3, 5])
def test_full_size_sampled(cid):
    """The whole BASELINE batch through analyze + correlate_peaks (bench.py's launch
    configuration); 256 seeded rows compared with the oracle element by element."""
    import torch
    cfg = W.CONFIGS[cid]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, cfg.rows, tm)
    plan = _plan(cfg, cfg.rows, tm)
    d_rows = plan.rows_to_device(rows)
    bands = plan.analyze(d_rows, cfg.rows)
    corr, lag, val = plan.correlate_peaks(bands, cfg.rows)
    torch.cuda.synchronize()
    ids = _sample_rows(cfg, 256)
    it = torch.tensor(ids, device=bands.device)
    g = dict(bands=bands.index_select(0, it).cpu().numpy(), corr=corr.index_select(0, it).cpu().numpy(),
             lag=lag.index_select(0, it).cpu().numpy(), val=val.index_select(0, it).cpu().numpy())
    r = oracle_for(plan, rows[ids], tm)
    st = compare(plan, g, r, neartie_bound=True)
    assert st["lag_total"] == 256 * (cfg.levels + 1)
    # property at any size: every lag is in range
    lg = lag.cpu().numpy()
    assert lg.min() >= 0 and lg.max() < cfg.N
    print(cfg.name, "full-size, 256 rows vs oracle", st)
    del bands, corr


def test_full_size_c4_sampled():
    """C4 (2048 pulses x bank of 64) through the peaks-only bank kernel; 16 seeded pulses x all
    64 templates compared with the oracle (corr of those pulses from the same kernel)."""
    import torch
    cfg = W.CONFIGS[4]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, cfg.rows, tm)
    plan = _plan(cfg, cfg.rows, tm)
    d_rows = plan.rows_to_device(rows)
    bands = plan.analyze(d_rows, cfg.rows)
    _, lag, val = plan.correlate_peaks(bands, cfg.rows, want_corr=False)     # peaks-only mode
    torch.cuda.synchronize()
    ids = _sample_rows(cfg, 16)
    it = torch.tensor(ids, device=bands.device)
    sub_bands = bands.index_select(0, it).contiguous()
    sub = plan.correlate_peaks(sub_bands, len(ids))
    torch.cuda.synchronize()
    g = dict(bands=sub_bands.cpu().numpy(), corr=sub[0].cpu().numpy(),
             lag=lag.index_select(0, it).cpu().numpy(), val=val.index_select(0, it).cpu().numpy())
    assert np.array_equal(g["lag"], sub[1].cpu().numpy())       # peaks-only == with-corr peaks
    r = oracle_for(plan, rows[ids], tm)
    st = compare(plan, g, r, neartie_bound=True)
    assert st["lag_total"] == 16 * 64 * (cfg.levels + 1)
    print(cfg.name, "full-size, 16 pulses x 64 templates vs oracle", st)


def test_real_template_variant_equals_general_path():
    """C2's Barker template is real: the real-template correlation (t.y products skipped) gives
    the same corr and peaks as the general complex kernel (SIDWT_REALT=0)."""
    import os
    cfg = W.CONFIGS[2]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, 4, tm)
    p_real = _plan(cfg, 4, tm)
    os.environ["SIDWT_REALT"] = "0"
    try:
        p_gen = _plan(cfg, 4, tm)
    finally:
        os.environ.pop("SIDWT_REALT", None)
    assert p_real.template_is_real() and not p_gen.template_is_real()
    g1 = run_gpu(p_real, rows, fused=True)
    g2 = run_gpu(p_gen, rows, fused=True)
    assert np.array_equal(g1["corr"], g2["corr"]) and np.array_equal(g1["lag"], g2["lag"])
    compare(p_real, g1, oracle_for(p_real, rows, tm))


def test_execute_host_after_reload_grows_workspaces():
    """execute_host, then a reload with a longer template (wider band margins -> larger band
    stride) and a larger bank, then execute_host again: the plan-owned workspaces must follow
    the new layout (results equal the device path and the oracle)."""
    import torch
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    rng = np.random.default_rng(77)
    N, J, R = 1024, 4, 6
    rows = (rng.normal(size=(R, N)) + 1j * rng.normal(size=(R, N))).astype(np.complex64)
    plan = Plan(O.CDF97, J, N, R, O.SYMMETRIC)
    for n_t, T in ((1, 16), (3, 200)):
        tm = (rng.normal(size=(n_t, T)) + 1j * rng.normal(size=(n_t, T))).astype(np.complex64)
        plan.load_templates(tm)
        lag = np.zeros((R, n_t, J + 1), np.int32)
        val = np.zeros((R, n_t, J + 1, 2), np.float32)
        plan.execute_host(np.ascontiguousarray(rows), R, lag, val)
        torch.cuda.synchronize()
        g = run_gpu(plan, rows, fused=True)
        assert np.array_equal(lag, g["lag"]) and np.array_equal(val, g["val"])
        compare(plan, g, oracle_for(plan, rows, tm))


def test_rejected_reload_keeps_previous_template():
    """A reload that the layout validation rejects (RANGE) leaves the loaded template usable."""
    import torch
    from paper_cs_0607001_b200 import Plan, SidwtError, _native
    _native.build()
    rng = np.random.default_rng(5)
    N, J, R = 8192, 10, 2
    rows = (rng.normal(size=(R, N)) + 1j * rng.normal(size=(R, N))).astype(np.complex64)
    tm = (rng.normal(size=(1, 40)) + 1j * rng.normal(size=(1, 40))).astype(np.complex64)
    plan = Plan(O.LEGALL53, J, N, R, O.SYMMETRIC).load_templates(tm)
    g0 = run_gpu(plan, rows, fused=True)
    with pytest.raises(SidwtError) as e:
        # T = N at J = 10: the coarsest term's band tile no longer fits the K2 shared memory
        _native.sidwt_template_load(plan.handle, np.ones((1, N, 2), np.float32), N, 1)
    assert e.value.status == 5
    g1 = run_gpu(plan, rows, fused=True)
    torch.cuda.synchronize()
    assert np.array_equal(g0["corr"], g1["corr"]) and np.array_equal(g0["lag"], g1["lag"])
