"""GPU parity of the single-template tensor-core correlation (csrc/corr_tcs.cuh, SURVEY
8(f) NEXT 4): the template's Toeplitz matrix (M = 64 shifts x re/im) against the band
gathered per residue class (N = one column per 64-lag block), bf16x3 split, fp32
accumulation in TMEM, eq. (4) suffix sums and peaks in the epilogue.  Taken for float
families, one template, symmetric extension, N/64 in [16, 256], 2^J <= N/64
(SIDWT_TCS=1 enables it; SIDWT_TCS=0 disables).  Compared element by element with the
oracle (fp64), and with the SIMT kernel on the same inputs."""
import os

import numpy as np
import pytest

import oracle as O
import workloads as W

from parity import compare, oracle_for, run_gpu

pytestmark = pytest.mark.gpu


def _plan(fam, J, N, rows, ext, tm, tcs="1", t=None):
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    old = os.environ.get("SIDWT_TCS")
    os.environ["SIDWT_TCS"] = tcs
    try:
        return Plan(fam, J, N, rows, ext, lifting_t=t).load_templates(tm)
    finally:
        if old is None:
            os.environ.pop("SIDWT_TCS", None)
        else:
            os.environ["SIDWT_TCS"] = old


@pytest.mark.parametrize("cid,nrows", [(2, 5), (3, 3)])
def test_tcs_configs_small(cid, nrows):
    cfg = W.CONFIGS[cid]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, nrows, tm)
    plan = _plan(cfg.family, cfg.levels, cfg.N, nrows, cfg.ext, tm)
    assert plan.tensor_core_path() == 2
    g = run_gpu(plan, rows, fused=True)
    r = oracle_for(plan, rows, tm)
    print(cfg.name, compare(plan, g, r))
    # same inputs through the SIMT kernel: both within tolerance of each other
    p2 = _plan(cfg.family, cfg.levels, cfg.N, nrows, cfg.ext, tm, tcs="0")
    assert p2.tensor_core_path() == 0
    g2 = run_gpu(p2, rows, fused=True)
    c1 = g["corr"][..., 0].astype(np.float64) + 1j * g["corr"][..., 1]
    c2 = g2["corr"][..., 0].astype(np.float64) + 1j * g2["corr"][..., 1]
    peak = np.abs(c2).max(axis=-1, keepdims=True)
    assert (np.abs(c1 - c2) <= 1e-4 * peak).all()


EDGE = [
    # fam, J, N, T
    (0, 2, 1024, 1),
    (0, 4, 1024, 64),
    (1, 4, 2048, 300),
    (1, 6, 8192, 512),
    (2, 5, 4096, 130),
    (2, 3, 8192, 33),
    (1, 2, 8192, 1000),
    (1, 7, 8192, 600),      # g = 2^7 = N / 64: residue blocks of one 64-lag block, the lg = 7 epilogue
    (0, 5, 2048, 200),      # N / 64 = 32 data rows (the M = 128 MMA rows past them are ignored)
    (2, 4, 1024, 100),      # the smallest tile: N / 64 = 16 data rows
]


@pytest.mark.parametrize("fam,J,N,T", EDGE)
def test_tcs_edge(fam, J, N, T):
    rng = np.random.default_rng(31 * fam + J + N + T)
    tm = (rng.normal(size=(1, T)) + 1j * rng.normal(size=(1, T))).astype(np.complex64)
    rows = (rng.normal(size=(3, N)) + 1j * rng.normal(size=(3, N))).astype(np.complex64)
    plan = _plan(fam, J, N, 3, 1, tm)
    assert plan.tensor_core_path() == 2
    g = run_gpu(plan, rows, fused=True)
    r = oracle_for(plan, rows, tm)
    compare(plan, g, r)


def test_tcs_peaks_only_and_rows_beyond_grid():
    """More rows than SMs (persistent CTAs loop over rows) and the peaks-only mode
    (running corr row in shared memory, no corr stores): same peaks as with corr output."""
    import torch
    cfg = W.CONFIGS[2]
    tm = W.templates(cfg)
    n = 300
    rows = W.make_rows(cfg, 0, n, tm)
    plan = _plan(cfg.family, cfg.levels, cfg.N, n, cfg.ext, tm)
    d = plan.rows_to_device(rows)
    bands = plan.analyze(d, n)
    corr, lag, val = plan.correlate_peaks(bands, n)
    _, lag2, val2 = plan.correlate_peaks(bands, n, want_corr=False)
    torch.cuda.synchronize()
    assert np.array_equal(lag.cpu().numpy(), lag2.cpu().numpy())
    assert np.array_equal(val.cpu().numpy(), val2.cpu().numpy())
    ids = [0, 1, 147, 148, 149, 299]
    g = dict(bands=bands.cpu().numpy()[ids], corr=corr.cpu().numpy()[ids], lag=lag.cpu().numpy()[ids],
             val=val.cpu().numpy()[ids])
    r = oracle_for(plan, rows[ids], tm)
    compare(plan, g, r)


def test_tcs_exact_cdf97():
    cfg = W.CONFIGS[3]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, 2, tm)
    t = 1.2301741049140007
    plan = _plan(cfg.family, cfg.levels, cfg.N, 2, cfg.ext, tm, t=t)
    assert plan.tensor_core_path() == 2
    g = run_gpu(plan, rows, fused=True)
    with O.t97(t):
        r = oracle_for(plan, rows, tm)
    compare(plan, g, r)


def test_tcs_not_taken():
    """Periodic extension, banks and short rows stay on the SIMT kernel; the integer family takes
    its own int8 tensor-core kernel (tests/test_gpu_i8.py), never this one."""
    rng = np.random.default_rng(5)
    one = (rng.normal(size=(1, 40)) + 1j * rng.normal(size=(1, 40))).astype(np.complex64)
    assert _plan(1, 3, 4096, 1, 0, one).tensor_core_path() == 0                    # periodic
    assert _plan(1, 3, 512, 1, 1, one).tensor_core_path() == 0                     # N / 64 < 16
    assert _plan(1, 3, 16384, 1, 1, one).tensor_core_path() == 0                   # does not fit on chip
    assert _plan(1, 7, 4096, 1, 1, one).tensor_core_path() == 0                    # 2^J > N / 64
    assert _plan(1, 3, 4096, 1, 1, np.repeat(one, 2, 0)).tensor_core_path() == 0  # two templates
    it = rng.integers(-100, 100, size=(1, 40, 2)).astype(np.int16)
    assert _plan(3, 3, 4096, 1, 1, it).tensor_core_path() == 3                     # integer: int8 kernel
