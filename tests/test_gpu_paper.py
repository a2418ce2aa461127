"""GPU parity of the paper's orientation (eq. (20)):
the template carries the redundant tree, the received row is critically sampled,
corr_s[tau] = <A_s (x delayed by tau), C_s ybar>.  Against oracle.run_paper (plain
definition: one Mallat pyramid of the delayed template per lag), same tolerances."""
import numpy as np
import pytest

import oracle as O
import workloads as W

from parity import CORR_TOL

pytestmark = pytest.mark.gpu


def _run(plan, rows):
    import torch
    n = rows.shape[0]
    bands = plan.analyze(plan.rows_to_device(rows), n)
    corr, lag, val = plan.correlate_peaks(bands, n)
    torch.cuda.synchronize()
    c = corr.cpu().numpy()
    return c[..., 0].astype(np.float64) + 1j * c[..., 1], lag.cpu().numpy(), val.cpu().numpy()


def _check(gc, gl, r):
    oc = r["corr"]
    peak = np.abs(oc).max(-1)
    err = np.abs(gc - oc).max(-1)
    assert (err / np.maximum(peak, 1e-300)).max() <= CORR_TOL
    same = gl == r["lag"]
    for i in np.argwhere(~same):
        i = tuple(i)
        tol = CORR_TOL * peak[i]
        assert np.abs(oc[i][gl[i]]) >= np.abs(oc[i][r["lag"][i]]) - 2 * tol


CASES = [
    # family, J, ext, N, T, n_t
    (0, 3, 0, 1024, 64, 1),
    (1, 4, 1, 1024, 100, 1),
    (2, 5, 1, 2048, 130, 1),
    (1, 6, 1, 1024, 200, 1),       # tap table too large for the kernel parameters (shared memory path)
    (0, 2, 1, 512, 1, 3),
]


@pytest.mark.parametrize("fam,J,ext,N,T,nt", CASES)
def test_paper_orientation(fam, J, ext, N, T, nt):
    from paper_cs_0607001_b200 import Plan, SIDWT_ORIENT_TEMPLATE_TREE, _native
    _native.build()
    rng = np.random.default_rng(31 + fam + J + N + T)
    tm = (rng.normal(size=(nt, T)) + 1j * rng.normal(size=(nt, T))).astype(np.complex64)
    rows = (rng.normal(size=(2, N)) + 1j * rng.normal(size=(2, N))).astype(np.complex64)
    rows[0, 50:50 + T] += 4 * tm[0]
    plan = Plan(fam, J, N, 2, ext, orientation=SIDWT_ORIENT_TEMPLATE_TREE).load_templates(tm)
    assert not plan.uses_tensor_cores()
    gc, gl, gv = _run(plan, rows)
    r = O.run_paper(fam, J, ext, N, rows, tm)
    _check(gc, gl, r)


def test_paper_orientation_c2_rows():
    """C2 shape (causal D4, J=5, symmetric, 4096, Barker-13 x10): two rows."""
    from paper_cs_0607001_b200 import Plan, SIDWT_ORIENT_TEMPLATE_TREE, _native
    _native.build()
    cfg = W.CONFIGS[2]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, 2, tm)
    plan = Plan(cfg.family, cfg.levels, cfg.N, 2, cfg.ext, orientation=SIDWT_ORIENT_TEMPLATE_TREE).load_templates(tm)
    gc, gl, gv = _run(plan, rows)
    r = O.run_paper(cfg.family, cfg.levels, cfg.ext, cfg.N, rows, tm)
    _check(gc, gl, r)


def test_orientation_rules():
    from paper_cs_0607001_b200 import Plan, SidwtError, _native
    _native.build()
    with pytest.raises(SidwtError) as e:
        Plan(3, 3, 64, 1, 1, orientation=1)                     # integer family: received tree only
    assert e.value.status == 1
    p = Plan(0, 3, 64, 1, 0).load_templates(np.ones((1, 8), np.complex64))
    with pytest.raises(SidwtError) as e:
        _native.sidwt_plan_set_orientation(p.handle, 1)         # after template_load
    assert e.value.status == 6
