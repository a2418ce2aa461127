"""Memory-safety checks of every kernel without compute-sanitizer (closed on this GPU pool:
runs under it have left GPUs needing a reset).  For each entry point, on small and ragged
plans of every family:

  * out-of-bounds writes: every output lives in the middle of a larger device buffer whose
    guard regions (before and after) hold a fixed byte pattern; the pattern must survive;
  * unwritten outputs (initcheck): the call runs twice, the output pre-filled with two
    different byte patterns; an element the kernels do not write keeps its pattern and the
    two results differ;
  * races: the same call repeated gives bit-identical outputs (a shared-memory or TMEM race
    shows up as run-to-run differences), and the result matches the oracle.
"""
import numpy as np
import pytest

import oracle as O
import workloads as W

from parity import compare, oracle_for

pytestmark = pytest.mark.gpu

GUARD = 1 << 16        # bytes of guard before and after each output


def _guarded(torch, nbytes, dev):
    buf = torch.empty(nbytes + 2 * GUARD, dtype=torch.uint8, device=dev)
    return buf


def _fill(buf, nbytes, pat):
    buf[:GUARD].fill_(0xA5)
    buf[GUARD + nbytes:].fill_(0x5A)
    buf[GUARD:GUARD + nbytes].fill_(pat)


def _guards_ok(buf, nbytes):
    b = buf.cpu().numpy()
    return bool((b[:GUARD] == 0xA5).all() and (b[GUARD + nbytes:] == 0x5A).all())


PLANS = [
    # (family, J, N, ext, T, n_t, rows)
    (0, 3, 1024, 0, 64, 1, 3),          # C1-like, periodic
    (2, 5, 4096, 1, 130, 1, 5),         # C2: real-template FFMA2 kernel
    (1, 6, 8192, 1, 512, 1, 3),         # C3: single-template tensor cores
    (1, 4, 2048, 1, 256, 16, 2),        # bank: template-bank tensor cores
    (3, 8, 4096, 1, 128, 1, 5),         # C5: int8 tensor cores
    (3, 4, 512, 1, 40, 1, 3),           # int8, partial tile (N < 2048), direct stores
    (0, 4, 256, 1, 40, 3, 2),           # small SIMT bank of 3
]


@pytest.mark.parametrize("fam,J,N,ext,T,nt,R", PLANS)
def test_guards_initcheck_determinism(fam, J, N, ext, T, nt, R):
    import torch
    from paper_cs_0607001_b200 import Plan, _native
    _native.build()
    dev = torch.device("cuda")
    rng = np.random.default_rng(fam * 100 + J + N)
    isint = fam == O.LEGALL53_INT
    if isint:
        tm = rng.integers(-2047, 2048, size=(nt, T, 2)).astype(np.int16)
        rows = rng.integers(-3000, 3000, size=(R, N, 2)).astype(np.int16)
    else:
        tm = (rng.normal(size=(nt, T)) + 1j * rng.normal(size=(nt, T))).astype(np.complex64)
        rows = (rng.normal(size=(R, N)) + 1j * rng.normal(size=(R, N))).astype(np.complex64)
    plan = Plan(fam, J, N, R, ext).load_templates(tm)
    d_rows = plan.rows_to_device(rows)
    S, nterm = plan.band_stride, J + 1
    nb = R * nterm * 2 * S * 4
    nc = R * nt * nterm * N * 8
    npk = R * nt * nterm
    B, Cb, Lb, Vb = (_guarded(torch, n, dev) for n in (nb, nc, npk * 4, npk * 8))
    dt = torch.int32 if isint else torch.float32

    def views():
        bands = B[GUARD:GUARD + nb].view(dt).view(R, nterm, 2, S)
        corr = Cb[GUARD:GUARD + nc].view(dt).view(R, nt, nterm, N, 2)
        lag = Lb[GUARD:GUARD + npk * 4].view(torch.int32).view(R, nt, nterm)
        val = Vb[GUARD:GUARD + npk * 8].view(dt).view(R, nt, nterm, 2)
        return bands, corr, lag, val

    outs = []
    for pat in (0x00, 0xFF, 0x3C):
        for buf, n in ((B, nb), (Cb, nc), (Lb, npk * 4), (Vb, npk * 8)):
            _fill(buf, n, pat)
        bands, corr, lag, val = views()
        plan.analyze(d_rows, R, bands)
        plan.correlate_peaks(bands, R, corr, lag, val)
        torch.cuda.synchronize()
        for buf, n in ((B, nb), (Cb, nc), (Lb, npk * 4), (Vb, npk * 8)):
            assert _guards_ok(buf, n), "a kernel wrote outside its output"
        outs.append([x.cpu().numpy().copy() for x in (bands, corr, lag, val)])
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b), "an output element is never written (or a race)"
    for a, b in zip(outs[0], outs[2]):
        assert np.array_equal(a, b), "run-to-run difference (race)"
    g = dict(bands=outs[0][0], corr=outs[0][1], lag=outs[0][2], val=outs[0][3])
    compare(plan, g, oracle_for(plan, rows, tm))

    # standalone peaks and synthesis, same checks on their outputs
    for pat in (0x00, 0xFF):
        _fill(Lb, npk * 4, pat)
        _fill(Vb, npk * 8, pat)
        bands, corr, lag, val = views()
        plan.peaks(corr, R, lag, val)
        torch.cuda.synchronize()
        assert _guards_ok(Lb, npk * 4) and _guards_ok(Vb, npk * 8)
        assert np.array_equal(lag.cpu().numpy(), outs[0][2])
    if plan.fused_available():                                  # k_fused: corr, lag, val
        fo = []
        for pat in (0x00, 0xFF):
            for buf, n in ((Cb, nc), (Lb, npk * 4), (Vb, npk * 8)):
                _fill(buf, n, pat)
            _, corr, lag, val = views()
            plan.analyze_correlate(d_rows, R, corr, lag, val)
            torch.cuda.synchronize()
            for buf, n in ((Cb, nc), (Lb, npk * 4), (Vb, npk * 8)):
                assert _guards_ok(buf, n)
            fo.append([x.cpu().numpy().copy() for x in (corr, lag, val)])
        for a, b in zip(fo[0], fo[1]):
            assert np.array_equal(a, b)
    ns = R * N * 8
    Sb = _guarded(torch, ns, dev)
    syn = []
    for pat in (0x00, 0xFF):
        _fill(Sb, ns, pat)
        out = Sb[GUARD:GUARD + ns].view(dt).view(R, N, 2)
        plan.synthesize(views()[0], R, 0, out)
        torch.cuda.synchronize()
        assert _guards_ok(Sb, ns)
        syn.append(out.cpu().numpy().copy())
    assert np.array_equal(syn[0], syn[1])
