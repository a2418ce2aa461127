"""Integer family on the int8 tensor cores (k_correlate_i8, csrc/corr_i8.cu): exact digit
GEMM, bit-identical to the oracle and to the INT32 SIMT kernel (SIDWT_I8=0) -- C5 shapes,
partial 2048-lag tiles, every depth, large-magnitude rows (three data digits), wide
templates (three template digits), peaks-only."""
import os

import numpy as np
import pytest

import oracle as O
import workloads as W

from parity import compare, oracle_for, run_gpu

pytestmark = pytest.mark.gpu


def _plans(J, N, R, tm):
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    p = Plan(O.LEGALL53_INT, J, N, R, O.SYMMETRIC).load_templates(tm)
    os.environ["SIDWT_I8"] = "0"
    try:
        q = Plan(O.LEGALL53_INT, J, N, R, O.SYMMETRIC).load_templates(tm)
    finally:
        os.environ.pop("SIDWT_I8", None)
    assert p.tensor_core_path() == 3 and q.tensor_core_path() == 0
    return p, q


def _check(J, N, rows, tm):
    p, q = _plans(J, N, rows.shape[0], tm)
    g = run_gpu(p, rows, fused=True)
    h = run_gpu(q, rows, fused=True)
    assert np.array_equal(g["corr"], h["corr"]) and np.array_equal(g["lag"], h["lag"])
    assert np.array_equal(g["val"], h["val"])
    compare(p, g, oracle_for(p, rows, tm))
    return p, g


def test_c5_rows():
    cfg = W.CONFIGS[5]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, 6, tm)
    _check(cfg.levels, cfg.N, rows, tm)


@pytest.mark.parametrize("J,N,T", [(1, 16, 3), (2, 64, 20), (3, 512, 100), (5, 1024, 64), (8, 2048, 128),
                                   (8, 4096, 200), (4, 4096, 160), (9, 4096, 128), (10, 4096, 50)])
def test_shapes(J, N, T):
    rng = np.random.default_rng(J * 1000 + N + T)
    tm = rng.integers(-2047, 2048, size=(1, T, 2)).astype(np.int16)
    rows = rng.integers(-3000, 3000, size=(3, N, 2)).astype(np.int16)
    _check(J, N, rows, tm)


def test_full_range_rows_take_three_digits():
    """Rows spanning the whole int16 range push the coarse bands past 16 bits: the builders'
    range flag selects three data digits there (still exact)."""
    rng = np.random.default_rng(11)
    N, J = 4096, 8
    tm = rng.integers(-2047, 2048, size=(1, 128, 2)).astype(np.int16)
    rows = rng.integers(-32768, 32768, size=(3, N, 2)).astype(np.int16)
    rows[1] = 32767                                   # DC extreme: U_8 = 256 * 32767
    rows[2, :, 0] = -32768
    p, g = _check(J, N, rows, tm)
    assert np.abs(g["bands"]).max() > 32767


def test_wide_template_three_digits():
    """A full-scale int16 template: pyramid taps beyond two balanced digits."""
    rng = np.random.default_rng(12)
    N, J = 2048, 6
    tm = rng.integers(-32768, 32768, size=(1, 300, 2)).astype(np.int16)
    rows = rng.integers(-4000, 4000, size=(2, N, 2)).astype(np.int16)
    _check(J, N, rows, tm)


@pytest.mark.parametrize("J,N", [(3, 4096), (8, 4096), (4, 2048), (2, 512)])
def test_peak_search_ties_and_equal_keys(J, N):
    """The two-stage peak search (32-bit high-word keys, exact 64-bit comparison for the key
    holders): rows whose |corr|^2 stays below 2^32 (every key 0: every thread is a holder), an
    all-zero row, a DC row, an impulse, and rows periodic in N/2 and N/8 (exactly equal maxima in
    different lag blocks, warps and tiles: the smallest lag must win) -- bit-identical to the
    oracle and to the SIMT kernel."""
    rng = np.random.default_rng(100 * J + N)
    T = 40
    tiny_t = rng.integers(-3, 4, size=(1, T, 2)).astype(np.int16)
    rows = np.zeros((6, N, 2), dtype=np.int16)
    rows[0] = rng.integers(-3, 4, size=(N, 2))                       # tiny: all keys 0
    rows[2, :, 0] = 5                                                # DC (row 1 stays all-zero)
    rows[3, N // 3] = (7, -2)                                        # impulse
    rows[4] = np.tile(rng.integers(-3, 4, size=(N // 2, 2)), (2, 1))   # period N/2
    rows[5] = np.tile(rng.integers(-3, 4, size=(N // 8, 2)), (8, 1))   # period N/8
    _check(J, N, rows, tiny_t)
    # the same periodic structure at full scale (keys differ, maxima still exactly equal)
    big_t = rng.integers(-2047, 2048, size=(1, T, 2)).astype(np.int16)
    rows2 = np.zeros((3, N, 2), dtype=np.int16)
    rows2[0] = np.tile(rng.integers(-3000, 3000, size=(N // 2, 2)), (2, 1))
    rows2[1] = np.tile(rng.integers(-3000, 3000, size=(N // 8, 2)), (8, 1))
    rows2[2] = np.tile(rng.integers(-3000, 3000, size=(16, 2)), (N // 16, 1))
    _check(J, N, rows2, big_t)


def test_peaks_only_and_many_rows():
    """More rows than SMs (persistent CTAs loop), peaks-only equals the with-corr peaks."""
    import torch
    cfg = W.CONFIGS[5]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, 300, tm)
    p, q = _plans(cfg.levels, cfg.N, 300, tm)
    d = p.rows_to_device(rows)
    bands = p.analyze(d, 300)
    corr, lag, val = p.correlate_peaks(bands, 300)
    _, lag2, val2 = p.correlate_peaks(bands, 300, want_corr=False)
    c2, lag3, _ = q.correlate_peaks(bands, 300)
    torch.cuda.synchronize()
    assert torch.equal(lag, lag2) and torch.equal(val, val2) and torch.equal(lag, lag3)
    assert torch.equal(corr, c2)
    ids = [0, 147, 148, 299]
    g = dict(bands=bands[ids].cpu().numpy(), corr=corr[ids].cpu().numpy(), lag=lag[ids].cpu().numpy(),
             val=val[ids].cpu().numpy())
    compare(p, g, oracle_for(p, rows[ids], tm))


def test_long_template_falls_back_to_simt():
    """Templates whose finest-term B images do not fit the shared-memory ring run on the INT32
    SIMT kernel (same results by construction; the tensor-core path is not taken)."""
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    rng = np.random.default_rng(13)
    tm = rng.integers(-2047, 2048, size=(1, 2000, 2)).astype(np.int16)
    p = Plan(O.LEGALL53_INT, 4, 4096, 2, O.SYMMETRIC).load_templates(tm)
    assert p.tensor_core_path() == 0
    rows = rng.integers(-3000, 3000, size=(2, 4096, 2)).astype(np.int16)
    compare(p, run_gpu(p, rows, fused=True), oracle_for(p, rows, tm))
