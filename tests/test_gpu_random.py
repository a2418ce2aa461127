"""Seeded random sweep over the plan space (family, depth, row length, template length,
extension, bank size, rows), each case through whichever correlation kernel the plan
selects (SIMT, template-bank tensor cores, single-template tensor cores) and compared
element by element with the oracle: bands, corr at every scale, peaks."""
import numpy as np
import pytest

import oracle as O

from parity import compare, oracle_for, run_gpu

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(0xC0FFEE + seed)
    fam = int(rng.integers(0, 4))
    N = int(2 ** rng.integers(8, 14))                      # 256 .. 8192
    J = int(rng.integers(1, min(7, int(np.log2(N)) - 1) + 1))
    ext = int(rng.integers(0, 2))
    T = int(rng.integers(1, min(N, 600) + 1))
    n_t = int(rng.choice([1, 1, 2, 16])) if fam != O.LEGALL53_INT else 1
    rows = int(rng.integers(1, 4))
    return rng, fam, N, J, ext, T, n_t, rows


@pytest.mark.parametrize("seed", range(48))
def test_random_plan(seed):
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    rng, fam, N, J, ext, T, n_t, rows = _case(seed)
    if fam == O.LEGALL53_INT:
        tm = rng.integers(-2047, 2048, size=(n_t, T, 2)).astype(np.int16)
        y = rng.integers(-3000, 3000, size=(rows, N, 2)).astype(np.int16)
    else:
        tm = (rng.normal(size=(n_t, T)) + 1j * rng.normal(size=(n_t, T))).astype(np.complex64)
        y = (rng.normal(size=(rows, N)) + 1j * rng.normal(size=(rows, N))).astype(np.complex64)
    plan = Plan(fam, J, N, rows, ext).load_templates(tm)
    g = run_gpu(plan, y, fused=True)
    r = oracle_for(plan, y, tm)
    st = compare(plan, g, r)
    print(dict(fam=fam, N=N, J=J, ext=ext, T=T, n_t=n_t, rows=rows, path=plan.tensor_core_path()), st)
