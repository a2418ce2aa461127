"""GPU synthesis (inverse lifting, coarse to fine; eq. (21)) against
the oracle's forward tree, and the perfect-reconstruction property (PAPER.md:61-63,
173-179): synthesising level 0 from the bands gives back the row itself.

Float families: relative L2 per row <= 1e-5 (the band tolerance); integer family:
bit-exact (the reversible integer lifting is exactly invertible)."""
import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu

CASES = [
    # family, J, ext, N
    (0, 3, 0, 1024),
    (0, 4, 1, 2048),
    (1, 6, 1, 8192),
    (1, 2, 0, 512),
    (2, 5, 1, 4096),
    (2, 3, 0, 256),
    (3, 8, 1, 4096),
    (3, 3, 0, 1024),
    (1, 4, 1, 16384),
]


def _rel(a, b):
    return float(np.sqrt((np.abs(a - b) ** 2).sum() / max((np.abs(b) ** 2).sum(), 1e-300)))


@pytest.mark.parametrize("fam,J,ext,N", CASES)
def test_synthesis_every_level(fam, J, ext, N):
    import torch
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    rng = np.random.default_rng(77 + fam * 13 + J + N)
    rows_n = 3
    isint = fam == O.LEGALL53_INT
    if isint:
        y = rng.integers(-3000, 3000, size=(rows_n, N, 2)).astype(np.int16)
        tm = rng.integers(-2047, 2048, size=(1, 40, 2)).astype(np.int16)
    else:
        y = (rng.normal(size=(rows_n, N)) + 1j * rng.normal(size=(rows_n, N))).astype(np.complex64)
        tm = (rng.normal(size=(1, 40)) + 1j * rng.normal(size=(1, 40))).astype(np.complex64)
    plan = Plan(fam, J, N, rows_n, ext).load_templates(tm)
    bands = plan.analyze(plan.rows_to_device(y), rows_n)
    for level in range(J):
        out = plan.synthesize(bands, rows_n, level)
        torch.cuda.synchronize()
        g = out.cpu().numpy()
        ref = O.approx(fam, ext, N, y, level)
        if isint:
            assert np.array_equal(g.astype(np.int64), ref), f"level {level}"
        else:
            gc = g[..., 0].astype(np.float64) + 1j * g[..., 1]
            for r in range(rows_n):
                assert _rel(gc[r], ref[r]) <= 1e-5, (level, r, _rel(gc[r], ref[r]))
    # perfect reconstruction: level 0 is the row itself
    g0 = plan.synthesize(bands, rows_n, 0).cpu().numpy()
    if isint:
        assert np.array_equal(g0, y.astype(np.int32))
    else:
        gc = g0[..., 0].astype(np.float64) + 1j * g0[..., 1]
        for r in range(rows_n):
            assert _rel(gc[r], y[r].astype(np.complex128)) <= 1e-5


def test_synthesis_c5_full_rows_exact():
    """BASELINE C5 shape (int 5/3, J=8, symmetric, 4096): exact reconstruction of a batch."""
    import torch
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    cfg = W.CONFIGS[5]
    tm = W.templates(cfg)
    y = W.make_rows(cfg, 0, 64, tm)
    plan = Plan(cfg.family, cfg.levels, cfg.N, 64, cfg.ext).load_templates(tm)
    bands = plan.analyze(plan.rows_to_device(y), 64)
    g0 = plan.synthesize(bands, 64, 0)
    torch.cuda.synchronize()
    assert np.array_equal(g0.cpu().numpy(), y.astype(np.int32))


def test_synthesis_status():
    from paper_cs_0607001_b200 import Plan, SidwtError, _native
    import torch
    _native.build()
    p = Plan(0, 3, 64, 2, 0).load_templates(np.ones((1, 8), np.complex64))
    b = p.empty_bands(2)
    o = torch.empty((2, 64, 2), device="cuda")
    with pytest.raises(SidwtError) as e:
        _native.sidwt_synthesize(p.handle, b, 2, 3, o)       # level must be < levels
    assert e.value.status == 4
