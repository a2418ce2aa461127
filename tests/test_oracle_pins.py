"""Pins of the CPU oracle against what the paper and the mathematics fix.

Every check here pins oracle/ to something other than itself:
  * printed values (tests/golden/*.txt, each line cited),
  * the paper's printed lifting factorizations (a different printed object than
    the filter polynomials the oracle uses) -- "the lifting factorization
    reproduces the filterbank outputs exactly" (BASELINE north star),
  * closed forms (Table I from t = 5/4, D4 orthonormality, vanishing moments),
  * invariants (perfect reconstruction / biorthogonality eq. (11),(13), energy
    (PAPER.md:61-63), shift-circulance, eq. (4) telescoping),
  * brute force on small inputs (textbook correlation at s = 0, the a-trous
    definition of the fine-grid bands).
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import workloads as W

FAMS_FLOAT = (O.LEGALL53, O.CDF97, O.DAUB4)
RNG = np.random.default_rng(12345)


def _golden(golden_dir, name):
    out = {}
    with open(os.path.join(golden_dir, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                k, *v = line.split()
                out[k] = v
    return out


# ---------------------------------------------------------------- Table I / constants

def test_table1_from_free_variable(golden_dir):
    """PAPER.md:217-219 formulas at t = 5/4 give Table I."""
    g = _golden(golden_dir, "table1.txt")
    t = Fraction(g["t"][0])
    alpha = (-2 * t + 1) / (4 * (t - 1))
    beta = -(t - 1) ** 2
    gamma = 1 / (4 * t * (t - 1))
    delta = t ** 3 - Fraction(7, 4) * t ** 2 + t
    zeta2 = Fraction(2) / t ** 2
    assert alpha == Fraction(g["alpha"][0])
    assert beta == Fraction(g["beta"][0])
    assert gamma == Fraction(g["gamma"][0])
    assert delta == Fraction(g["delta"][0])
    assert zeta2 == Fraction(g["zeta^2"][0])


def _table1(golden_dir):
    g = _golden(golden_dir, "table1.txt")
    return (float(Fraction(g["alpha"][0])), float(Fraction(g["beta"][0])), float(Fraction(g["gamma"][0])),
            float(Fraction(g["delta"][0])), math.sqrt(float(Fraction(g["zeta^2"][0]))))


# ---------------------------------------------------------------- printed filter values

def test_printed_filters(golden_dir):
    g = _golden(golden_dir, "filters_printed.txt")

    def tab(key):
        lo = int(g[key][0])
        return lo, np.array([float(Fraction(v)) for v in g[key][1:]])

    lo, t = O.filt(O.LEGALL53, O.ANALYSIS, O.LOWPASS)
    assert (lo, list(t)) == (tab("legall53_analysis_low")[0], list(tab("legall53_analysis_low")[1]))
    lo, t = O.filt(O.LEGALL53, O.ANALYSIS, O.HIGHPASS)
    assert (lo, list(t)) == (tab("legall53_analysis_high")[0], list(tab("legall53_analysis_high")[1]))
    # dual analysis = 2 x time-reversed synthesis filters
    for which, key in ((O.LOWPASS, "legall53_synth_low"), (O.HIGHPASS, "legall53_synth_high")):
        lo_s, h = tab(key)
        lo, t = O.filt(O.LEGALL53, O.DUAL, which)
        n_hi = lo_s + len(h) - 1
        assert lo == -n_hi
        np.testing.assert_array_equal(t, 2.0 * h[::-1])
    # 9/7 lowpass listings, symmetric, outermost -> centre
    half = np.array([float(v) for v in g["cdf97_analysis_low_x160sqrt2"]]) / (160 * math.sqrt(2))
    lo, t = O.filt(O.CDF97, O.ANALYSIS, O.LOWPASS)
    assert lo == -4
    np.testing.assert_allclose(t, np.concatenate([half, half[-2::-1]]), rtol=0, atol=4e-16)
    half = np.array([float(v) for v in g["cdf97_synth_low_x64_over_sqrt2"]]) * math.sqrt(2) / 64
    lo, t = O.filt(O.CDF97, O.DUAL, O.LOWPASS)
    assert lo == -3
    np.testing.assert_allclose(t, np.concatenate([half, half[-2::-1]]), rtol=0, atol=4e-16)


def test_eq7_reproduces_printed_53_highpass(golden_dir):
    """Eq. (7) applied to the printed 5/3 lowpasses gives the printed
    5/3 highpasses -- validates the Eq. (7) route the oracle uses for the 9/7 highpass."""
    g = _golden(golden_dir, "filters_printed.txt")
    h = {n: float(Fraction(v)) for n, v in zip(range(-1, 2), g["legall53_synth_low"][1:])}
    ht = {m: float(Fraction(v)) for m, v in zip(range(-2, 3), g["legall53_analysis_low"][1:])}
    # gt(z^-1) = z h(-z): coefficient of z^-m is (-1)^(m+1) h[m+1]
    gt = [(-1) ** ((m + 1) & 1) * h.get(m + 1, 0.0) for m in range(-2, 1)]
    assert gt == [float(Fraction(v)) for v in g["legall53_analysis_high"][1:]]
    # g(z^-1) = z ht(-z) (ht symmetric): coefficient of z^-m is (-1)^(m+1) ht[m+1]
    gd = [(-1) ** ((m + 1) & 1) * ht.get(m + 1, 0.0) for m in range(-3, 2)]
    synth_high = [float(Fraction(v)) for v in g["legall53_synth_high"][1:]]   # n = -1..3
    assert gd == synth_high[::-1]


# ---------------------------------------------------------------- lifting == filterbank

def _nxt(a):
    return np.roll(a, -1)


def _prv(a):
    return np.roll(a, 1)


def lift(prog, v, consts):
    """The paper's printed lifting factorizations, applied right-to-left on a periodic sequence.
    Pairing: x_e[k] = x[2k], x_o[k] = x[2k+1] except causal D4 (x[2k-1], reading R-D1)."""
    al, be, ga, de, ze = consts
    v = np.asarray(v, dtype=np.complex128)
    if prog == "d4":
        e, o = v[0::2].copy(), np.roll(v, 1)[0::2].copy()
    else:
        e, o = v[0::2].copy(), v[1::2].copy()
    if prog == "53a":
        o = o - 0.5 * (e + _nxt(e))
        e = e + 0.25 * (o + _prv(o))
        return e, 0.5 * o
    if prog == "53d":
        e = e + 0.5 * (o + _prv(o))
        o = o - 0.25 * (e + _nxt(e))
        return e, 2.0 * o
    if prog == "97a":      # PAPER.md:238, reading R-D3
        o = o + al * (e + _nxt(e))
        e = e + be * (o + _prv(o))
        o = o + ga * (e + _nxt(e))
        e = e + de * (o + _prv(o))
        return ze * e, o / ze
    if prog == "97d":      # PAPER.md:240-242, reading R-D3 (mechanical dual of 97a)
        e = e - al * (o + _prv(o))
        o = o - be * (e + _nxt(e))
        e = e - ga * (o + _prv(o))
        o = o - de * (e + _nxt(e))
        return e / ze, ze * o
    if prog == "d4":       # eq. (17), reading R-D2
        r3 = math.sqrt(3.0)
        o = o - r3 * e
        e = e + (r3 / 4) * o + ((r3 - 2) / 4) * _prv(o)
        o = e + _prv(o)
        return ((r3 + 1) / math.sqrt(2)) * e, ((r3 - 1) / math.sqrt(2)) * o
    raise ValueError(prog)


@pytest.mark.parametrize("fam,role,prog", [
    (O.LEGALL53, O.ANALYSIS, "53a"), (O.LEGALL53, O.DUAL, "53d"),
    (O.CDF97, O.ANALYSIS, "97a"), (O.CDF97, O.DUAL, "97d"),
    (O.DAUB4, O.ANALYSIS, "d4"), (O.DAUB4, O.DUAL, "d4")])
def test_lifting_reproduces_filterbank(fam, role, prog, golden_dir):
    consts = _table1(golden_dir)
    for P in (8, 16, 64):
        for _ in range(20):
            v = RNG.normal(size=P) + 1j * RNG.normal(size=P)
            c, d = O.mallat_level(fam, role, v)
            a, b = lift(prog, v, consts)
            np.testing.assert_allclose(c, a, rtol=0, atol=1e-13)
            np.testing.assert_allclose(d, b, rtol=0, atol=1e-13)


def test_d4_eq17_product_equals_polyphase():
    """Eq. (17) (reading R-D2) multiplies out to Pt'(z^-1)
    with the textbook Daubechies-4 coefficients the oracle uses; det = z^-1."""
    sp = pytest.importorskip("sympy")
    z = sp.symbols("z")
    r3, r2 = sp.sqrt(3), sp.sqrt(2)
    K = sp.diag((r3 + 1) / r2, (r3 - 1) / r2)
    M1 = sp.Matrix([[1, 0], [1, 1 / z]])
    M2 = sp.Matrix([[1, r3 / 4 + (r3 - 2) / 4 / z], [0, 1]])
    M3 = sp.Matrix([[1, 0], [-r3, 1]])
    Pp = sp.simplify(K * M1 * M2 * M3)
    lo, hlo = O.filt(O.DAUB4, O.ANALYSIS, O.LOWPASS)
    h = [(1 + r3) / (4 * r2), (3 + r3) / (4 * r2), (3 - r3) / (4 * r2), (1 - r3) / (4 * r2)]
    np.testing.assert_allclose([float(v) for v in h], hlo, atol=1e-15)
    target = sp.Matrix([[h[0] + h[2] / z, h[1] + h[3] / z], [-h[3] - h[1] / z, h[2] + h[0] / z]])
    diff = sp.simplify(sp.expand(Pp - target))
    assert diff == sp.zeros(2, 2)
    assert sp.simplify(Pp.det() - 1 / z) == 0


def test_d4_orthonormal_and_moments():
    lo, h = O.filt(O.DAUB4, O.ANALYSIS, O.LOWPASS)
    _, g = O.filt(O.DAUB4, O.ANALYSIS, O.HIGHPASS)
    assert abs(np.dot(h, h) - 1) < 1e-15 and abs(h[0] * h[2] + h[1] * h[3]) < 1e-15
    m = np.arange(4)
    assert abs(np.sum(g)) < 1e-15 and abs(np.sum(g * m)) < 1e-14   # 2 vanishing moments
    assert abs(np.sum(g * m ** 2)) > 0.1


@pytest.mark.parametrize("fam,role,nvm", [
    (O.LEGALL53, O.ANALYSIS, 2), (O.LEGALL53, O.DUAL, 2),
    (O.CDF97, O.ANALYSIS, 4), (O.CDF97, O.DUAL, 2), (O.DAUB4, O.DUAL, 2)])
def test_vanishing_moments(fam, role, nvm):
    """PAPER.md:187 (5/3: two), PAPER.md:215 (9/7: four -- holds for the analysis
    highpass; with Table I's rational parameters the dual highpass keeps two)."""
    lo, g = O.filt(fam, role, O.HIGHPASS)
    m = np.arange(lo, lo + len(g), dtype=np.float64)
    for p in range(nvm):
        assert abs(np.sum(g * m ** p)) < 1e-12, p
    assert abs(np.sum(g * m ** nvm)) > 1e-3


# ---------------------------------------------------------------- PR / biorthogonality / energy

def _dense(fam, role, P):
    cols = []
    for n in range(P):
        e = np.zeros(P, np.complex128)
        e[n] = 1
        c, d = O.mallat_level(fam, role, e)
        cols.append(np.concatenate([c, d]))
    return np.array(cols).T.real


@pytest.mark.parametrize("fam", FAMS_FLOAT)
def test_perfect_reconstruction_biorthogonal(fam):
    """eq. (11)/(13): dual-analysis^T x analysis = I (perfect reconstruction, and the
    one-level inner-product identity of eq. (4)/(15))."""
    for P in (8, 16, 32):
        Ma = _dense(fam, O.ANALYSIS, P)
        Md = _dense(fam, O.DUAL, P)
        np.testing.assert_allclose(Md.T @ Ma, np.eye(P), atol=1e-13)
        x = RNG.normal(size=P) + 1j * RNG.normal(size=P)
        y = RNG.normal(size=P) + 1j * RNG.normal(size=P)
        a, b = O.mallat_level(fam, O.ANALYSIS, x)
        c, d = O.mallat_level(fam, O.DUAL, y)
        lhs = np.vdot(x, y)
        rhs = np.vdot(a, c) + np.vdot(b, d)
        assert abs(lhs - rhs) < 1e-12 * (1 + abs(lhs))


def test_d4_energy():
    """PAPER.md:61-63 energy equivalence for the orthogonal (Daubechies-4) filterbank."""
    for P in (8, 32, 128):
        v = RNG.normal(size=P) + 1j * RNG.normal(size=P)
        c, d = O.mallat_level(O.DAUB4, O.DUAL, v)
        assert abs(np.vdot(c, c).real + np.vdot(d, d).real - np.vdot(v, v).real) < 1e-12 * P


def test_d4_tight_frame_bands():
    """Energy over the fine-grid bands of the orthogonal D4 tree: one period of y
    gives ||y||^2 = sum_s 2^-s ||W_s||^2 + 2^-J ||U_J||^2."""
    N, J = 64, 4
    y = RNG.normal(size=N) + 1j * RNG.normal(size=N)
    x = np.ones(4, np.complex128)
    r = O.run(O.DAUB4, J, O.PERIODIC, N, y[None], x[None], p_lo=0, p_hi=N, corr=False)
    B = r["bands"][0]
    e = sum(2.0 ** -(s + 1) * np.vdot(B[s], B[s]).real for s in range(J)) + 2.0 ** -J * np.vdot(B[J], B[J]).real
    assert abs(e - np.vdot(y, y).real) < 1e-10 * np.vdot(y, y).real


# ---------------------------------------------------------------- shift-circulance

@pytest.mark.parametrize("fam", FAMS_FLOAT)
def test_shift_circulance_one_level(fam):
    """shifting the input by 2p shifts the DWT coefficients by p."""
    P = 32
    v = RNG.normal(size=P) + 1j * RNG.normal(size=P)
    c, d = O.mallat_level(fam, O.DUAL, v)
    for p in (1, 3, 7):
        c2, d2 = O.mallat_level(fam, O.DUAL, np.roll(v, -2 * p))
        np.testing.assert_allclose(c2, np.roll(c, -p), atol=1e-13)
        np.testing.assert_allclose(d2, np.roll(d, -p), atol=1e-13)


@pytest.mark.parametrize("fam", FAMS_FLOAT)
def test_shift_equivariance_bands_and_corr(fam):
    """SIDWT is shift-invariant at every lag: bands and corr of the
    row circularly shifted by d are the originals shifted by d (periodic extension)."""
    N, J, T = 64, 3, 9
    y = RNG.normal(size=N) + 1j * RNG.normal(size=N)
    x = RNG.normal(size=T) + 1j * RNG.normal(size=T)
    r0 = O.run(fam, J, O.PERIODIC, N, y[None], x[None], p_lo=0, p_hi=N)
    for d in (1, 5, 13):
        r1 = O.run(fam, J, O.PERIODIC, N, np.roll(y, -d)[None], x[None], p_lo=0, p_hi=N)
        np.testing.assert_allclose(r1["bands"][0], np.roll(r0["bands"][0], -d, axis=-1), atol=1e-12)
        np.testing.assert_allclose(r1["corr"][0], np.roll(r0["corr"][0], -d, axis=-1), atol=1e-11)


@pytest.mark.parametrize("fam", FAMS_FLOAT + (O.LEGALL53_INT,))
def test_template_pyramid_shift(fam):
    """Critically sampled template: a_s(S_{2^s m} x)[k] = a_s(x)[k - m] (zero-extended)."""
    J, T, m = 3, 12, 1
    if fam == O.LEGALL53_INT:
        x = RNG.integers(-2000, 2000, size=(T, 2)).astype(np.int16)
        xs = np.concatenate([np.zeros((2 ** J * m, 2), np.int16), x])
    else:
        x = RNG.normal(size=T) + 1j * RNG.normal(size=T)
        xs = np.concatenate([np.zeros(2 ** J * m), x])
    p0 = O.template_pyramid(fam, J, x)
    p1 = O.template_pyramid(fam, J, xs)
    # a_J is the last entry; coefficients equal after trimming the (zero) support ends
    k0, a0 = p0[-1]
    k1, a1 = p1[-1]
    full0 = {k0 + i: a0[i] for i in range(len(a0))}
    full1 = {k1 + i: a1[i] for i in range(len(a1))}
    for k, v in full0.items():
        np.testing.assert_array_equal(np.asarray(full1.get(k + m, 0 * v)), np.asarray(v))


# ---------------------------------------------------------------- tree == a trous (P11)

def _extend(y, ext, n):
    N = len(y)
    if ext == O.PERIODIC:
        return y[np.mod(n, N)]
    m = np.mod(n, 2 * N - 2)
    return y[np.where(m < N, m, 2 * N - 2 - m)]


@pytest.mark.parametrize("fam", FAMS_FLOAT)
@pytest.mark.parametrize("ext", (O.PERIODIC, O.SYMMETRIC))
def test_tree_equals_a_trous(fam, ext):
    """The paper's even/odd shift tree (Fig. 1/5) re-indexed on the fine
    grid (branch r, coefficient k <-> tau = r + 2^s k) equals the undecimated transform
    U_s[tau] = sum_m f[m] U_{s-1}[tau - 2^{s-1} m] (reading R-D5)."""
    N, J = 32, 3
    y = RNG.normal(size=N) + 1j * RNG.normal(size=N)
    p_lo, p_hi = -40, N + 70
    r = O.run(fam, J, ext, N, y[None], np.ones((1, 2)), p_lo=p_lo, p_hi=p_hi, corr=False)
    lo_l, fl = O.filt(fam, O.DUAL, O.LOWPASS)
    lo_h, fh = O.filt(fam, O.DUAL, O.HIGHPASS)
    span = 400
    pos = np.arange(-span, span + 1)
    U = _extend(y, ext, pos)
    for s in range(1, J + 1):
        h = 2 ** (s - 1)
        Un = np.zeros_like(U)
        Wn = np.zeros_like(U)
        for i, m in enumerate(range(lo_l, lo_l + len(fl))):
            Un += fl[i] * np.roll(U, h * m)
        for i, m in enumerate(range(lo_h, lo_h + len(fh))):
            Wn += fh[i] * np.roll(U, h * m)
        sel = slice(p_lo + span, p_hi + span)
        np.testing.assert_allclose(r["bands"][0, s - 1], Wn[sel], atol=1e-12)
        U = Un
    np.testing.assert_allclose(r["bands"][0, J], U[sel], atol=1e-12)


# ---------------------------------------------------------------- correlation pins

@pytest.mark.parametrize("fam", FAMS_FLOAT)
@pytest.mark.parametrize("ext", (O.PERIODIC, O.SYMMETRIC))
def test_scale0_is_textbook_correlation(fam, ext):
    """P9: corr_0[tau] = sum_n conj(x[n]) ybar[n + tau] (brute force)."""
    N, J, T = 64, 3, 20
    y = RNG.normal(size=N) + 1j * RNG.normal(size=N)
    x = RNG.normal(size=T) + 1j * RNG.normal(size=T)
    r = O.run(fam, J, ext, N, y[None], x[None])
    ref = np.array([sum(np.conj(x[n]) * _extend(y, ext, np.array([n + tau]))[0] for n in range(T))
                    for tau in range(N)])
    np.testing.assert_allclose(r["corr"][0, 0, 0], ref, atol=1e-12)


@pytest.mark.parametrize("fam", FAMS_FLOAT)
@pytest.mark.parametrize("ext", (O.PERIODIC, O.SYMMETRIC))
def test_eq4_telescoping(fam, ext):
    """P10: the oracle's approximation-domain corr_s equals the eq. (4) telescoped form
    A_J + sum_{i>s} D_i computed here from the oracle's template pyramid and bands."""
    N, J, T = 64, 4, 23
    y = RNG.normal(size=N) + 1j * RNG.normal(size=N)
    x = RNG.normal(size=T) + 1j * RNG.normal(size=T)
    pyr = O.template_pyramid(fam, J, x)
    lo = min(2 ** (i + 1) * k for i, (k, _) in enumerate(pyr[:-1]))
    lo = min(lo, 2 ** J * pyr[-1][0])
    hi = max(2 ** (i + 1) * (k + len(c) - 1) for i, (k, c) in enumerate(pyr[:-1]))
    hi = max(hi, 2 ** J * (pyr[-1][0] + len(pyr[-1][1]) - 1))
    p_lo, p_hi = lo, N + hi + 1
    r = O.run(fam, J, ext, N, y[None], x[None], p_lo=p_lo, p_hi=p_hi)
    B = r["bands"][0]
    terms = []
    for i in range(J + 1):
        k0, c = pyr[i]
        lev = i + 1 if i < J else J
        t = np.zeros(N, np.complex128)
        for j, cc in enumerate(c):
            idx = np.arange(N) + 2 ** lev * (k0 + j) - p_lo
            t += np.conj(cc) * B[i, idx]
        terms.append(t)
    corr = np.zeros(N, np.complex128) + terms[J]
    np.testing.assert_allclose(r["corr"][0, 0, J], corr, atol=1e-10)
    for s in range(J - 1, -1, -1):
        corr = corr + terms[s]
        np.testing.assert_allclose(r["corr"][0, 0, s], corr, atol=1e-10)


def test_peak_clean_chirp_and_tie_rule():
    """P15: a clean row holding the template at lag d peaks at d with value sum |x|^2 = T
    (unit-modulus LFM); two equal echoes -> the smaller lag wins."""
    N, J, T = 256, 3, 32
    x = W.lfm(T, 16.0)
    for fam in FAMS_FLOAT:
        for d in (0, 17, N - T):
            y = np.zeros(N, np.complex128)
            y[d:d + T] = x
            r = O.run(fam, J, O.PERIODIC, N, y[None], x[None])
            assert r["lag"][0, 0, 0] == d
            assert abs(r["val"][0, 0, 0] - T) < 1e-9
        y = np.zeros(N, np.complex128)
        y[40:40 + T] += x
        y[140:140 + T] += x
        r = O.run(fam, J, O.PERIODIC, N, y[None], x[None])
        assert r["lag"][0, 0, 0] == 40


def test_zero_row_and_degenerate_sizes():
    """All-zero rows give zero correlation and lag 0; N = 2^J and T = N are accepted."""
    for fam in FAMS_FLOAT:
        N, J = 8, 3
        r = O.run(fam, J, O.SYMMETRIC, N, np.zeros((1, N)), np.ones((1, N)))
        assert np.all(r["corr"] == 0) and np.all(r["lag"] == 0)
    r = O.run(O.LEGALL53_INT, 3, O.SYMMETRIC, 8, np.zeros((1, 8, 2), np.int16), np.ones((1, 8, 2), np.int16))
    assert np.all(r["corr"] == 0) and np.all(r["lag"] == 0)
    with pytest.raises(ValueError):
        O.run(O.LEGALL53, 4, O.PERIODIC, 8, np.zeros((1, 8)), np.ones((1, 3)))    # 2^J > N


# ---------------------------------------------------------------- integer 5/3

def test_int53_golden(golden_dir):
    g = _golden(golden_dir, "int53_levels.txt")
    for role, key in ((O.DUAL, "dual"), (O.ANALYSIS, "analysis")):
        v = g[key]
        vi = np.array([int(t) for t in v[0:4]])
        c = [int(t) for t in v[5:7]]
        d = [int(t) for t in v[8:10]]
        cc, dd = O.int_level(role, vi)
        assert list(cc) == c and list(dd) == d


def _inv_int(role, c, d):
    """Inverse lifting steps (reverse order, opposite sign) -- exact reversibility."""
    c = np.asarray(c, np.int64)
    d = np.asarray(d, np.int64)
    fl = lambda a, b: np.floor_divide(a, b)
    if role == O.DUAL:
        o = d + fl(c + np.roll(c, -1) + 2, 4)
        e = c - fl(o + np.roll(o, 1), 2)
    else:
        e = c - fl(np.roll(d, 1) + d + 2, 4)
        o = d + fl(e + np.roll(e, -1), 2)
    v = np.empty(2 * len(c), np.int64)
    v[0::2], v[1::2] = e, o
    return v


@pytest.mark.parametrize("role", (O.DUAL, O.ANALYSIS))
def test_int53_reversible(role):
    for P in (4, 16, 64):
        for _ in range(50):
            v = RNG.integers(-30000, 30000, size=P)
            c, d = O.int_level(role, v)
            np.testing.assert_array_equal(_inv_int(role, c, d), v)


def test_int53_equals_rational_53_when_floors_exact():
    """With every sample a multiple of 2^(2J+2) all floors are exact, so the integer
    path (scales 1 and 1 instead of 1/2 and 2, DESIGN.md R-INT) equals the rational
    LeGall 5/3 path exactly: bands up to the detail factor 2, correlations exactly."""
    N, J, T = 64, 2, 8
    q = 2 ** (2 * J + 2)
    y = RNG.integers(-40, 40, size=(N, 2)) * q
    x = RNG.integers(-40, 40, size=(T, 2)) * q
    ri = O.run(O.LEGALL53_INT, J, O.SYMMETRIC, N, y.astype(np.int16)[None], x.astype(np.int16)[None],
               p_lo=-20, p_hi=N + 20)
    yc = (y[:, 0] + 1j * y[:, 1]).astype(np.complex128)
    xc = (x[:, 0] + 1j * x[:, 1]).astype(np.complex128)
    rf = O.run(O.LEGALL53, J, O.SYMMETRIC, N, yc[None], xc[None], p_lo=-20, p_hi=N + 20)
    bi = ri["bands"][0][..., 0] + 1j * ri["bands"][0][..., 1]
    bf = rf["bands"][0]
    np.testing.assert_array_equal(bi[J], bf[J])
    np.testing.assert_array_equal(2 * bi[:J], bf[:J])
    ci = ri["corr"][0][..., 0].astype(np.float64) + 1j * ri["corr"][0][..., 1]
    np.testing.assert_allclose(ci, rf["corr"][0], atol=1e-6 * np.abs(rf["corr"][0]).max())
    assert np.abs(rf["corr"][0]).max() < 2 ** 31


def test_int53_close_to_exact_correlation():
    """C5-like rows: the integer scale-0 correlation stays within the rounding of the
    floor-based lifting of the exact correlation (~4e-4 x peak)."""
    cfg = W.CONFIGS[5]
    tm = W.templates(cfg)
    y, truth = W.make_row(cfg, 0, tm)
    J = cfg.levels
    ri = O.run(O.LEGALL53_INT, J, O.SYMMETRIC, cfg.N, y[None], tm)
    yc = y[:, 0].astype(np.float64) + 1j * y[:, 1]
    xc = tm[0, :, 0].astype(np.float64) + 1j * tm[0, :, 1]
    ext = _extend(yc, O.SYMMETRIC, np.arange(cfg.N + cfg.T))
    ref = np.array([np.vdot(xc, ext[t:t + cfg.T]) for t in range(cfg.N)])
    ci = ri["corr"][0, 0, 0, :, 0] + 1j * ri["corr"][0, 0, 0, :, 1]
    assert np.abs(ci - ref).max() < 1e-3 * np.abs(ref).max()
    assert ri["lag"][0, 0, 0] == truth[0][1]


# ---------------------------------------------------------------- approximation bands (synthesis checks)

@pytest.mark.parametrize("fam", FAMS_FLOAT)
@pytest.mark.parametrize("ext", (O.PERIODIC, O.SYMMETRIC))
def test_approx_bands_are_a_trous_lowpass(fam, ext):
    """oracle.approx (the forward tree's U_s, used to check the GPU synthesis of eq. (21),
    PAPER.md:296-298): U_0 is the extended row (O1), U_J equals oracle_run's band J, and every
    level is the undecimated lowpass U_s[tau] = sum_m f[m] U_{s-1}[tau - 2^{s-1} m] (R-D5)."""
    N, J = 32, 3
    y = RNG.normal(size=N) + 1j * RNG.normal(size=N)
    p_lo, p_hi = -40, N + 70
    lo_l, fl = O.filt(fam, O.DUAL, O.LOWPASS)
    span = 400
    pos = np.arange(-span, span + 1)
    U = _extend(y, ext, pos)
    sel = slice(p_lo + span, p_hi + span)
    np.testing.assert_allclose(O.approx(fam, ext, N, y[None], 0, p_lo, p_hi)[0], U[sel], atol=0)
    for s in range(1, J + 1):
        h = 2 ** (s - 1)
        Un = np.zeros_like(U)
        for i, m in enumerate(range(lo_l, lo_l + len(fl))):
            Un += fl[i] * np.roll(U, h * m)
        U = Un
        np.testing.assert_allclose(O.approx(fam, ext, N, y[None], s, p_lo, p_hi)[0], U[sel], atol=1e-12)
    r = O.run(fam, J, ext, N, y[None], np.ones((1, 2)), p_lo=p_lo, p_hi=p_hi, corr=False)
    np.testing.assert_allclose(O.approx(fam, ext, N, y[None], J, p_lo, p_hi)[0], r["bands"][0, J], atol=0)


@pytest.mark.parametrize("ext", (O.PERIODIC, O.SYMMETRIC))
def test_approx_bands_integer(ext):
    """Integer family: U_0 is the extended I/Q row exactly; U_J equals oracle_run's band J."""
    N, J = 64, 4
    y = RNG.integers(-3000, 3000, size=(1, N, 2)).astype(np.int16)
    p_lo, p_hi = -20, N + 30
    u0 = O.approx(O.LEGALL53_INT, ext, N, y, 0, p_lo, p_hi)[0]
    idx = np.array([_ext_index(ext, N, p) for p in range(p_lo, p_hi)])
    assert np.array_equal(u0, y[0][idx].astype(np.int64))
    r = O.run(O.LEGALL53_INT, J, ext, N, y, np.ones((1, 2, 2), np.int16), p_lo=p_lo, p_hi=p_hi, corr=False)
    assert np.array_equal(O.approx(O.LEGALL53_INT, ext, N, y, J, p_lo, p_hi)[0], r["bands"][0, J])


def _ext_index(ext, N, n):
    if ext == O.PERIODIC:
        return n % N
    m = n % (2 * N - 2)
    return m if m < N else 2 * N - 2 - m


# ---------------------------------------------------------------- the paper's orientation (NEXT 3)

@pytest.mark.parametrize("fam", FAMS_FLOAT)
@pytest.mark.parametrize("ext", (O.PERIODIC, O.SYMMETRIC))
def test_paper_orientation_pins(fam, ext):
    """corr^P_s[tau] = <A_s S_{-tau} x, C_s ybar>: equal to the textbook
    correlation at s = 0 (brute force), equal to this build's orientation <A_s x, C_s S_tau ybar>
    at tau = 0 mod 2^s, and shift-consistent: the lag 2^s m corresponds to shifting
    the critically sampled coefficients by m (P12)."""
    N, J, T = 64, 3, 12
    y = RNG.normal(size=N) + 1j * RNG.normal(size=N)
    x = RNG.normal(size=T) + 1j * RNG.normal(size=T)
    rp = O.run_paper(fam, J, ext, N, y[None], x[None])
    ro = O.run(fam, J, ext, N, y[None], x[None])
    ref = np.array([sum(np.conj(x[n]) * _extend(y, ext, np.array([n + tau]))[0] for n in range(T))
                    for tau in range(N)])
    np.testing.assert_allclose(rp["corr"][0, 0, 0], ref, atol=1e-12)
    for s in range(J + 1):
        sel = np.arange(0, N, 2 ** s)
        np.testing.assert_allclose(rp["corr"][0, 0, s, sel], ro["corr"][0, 0, s, sel], atol=1e-11)
    # off the 2^s grid the two orientations differ (D7): at least one lag at every s >= 1
    for s in range(1, J + 1):
        off = np.setdiff1d(np.arange(N), np.arange(0, N, 2 ** s))
        assert np.abs(rp["corr"][0, 0, s, off] - ro["corr"][0, 0, s, off]).max() > 1e-6


def test_paper_orientation_dense_matrices():
    """Brute force on a tiny periodic case: A_s and C_s as explicit matrices (level-by-level
    Mallat operators of the printed filters), corr^P_s[tau] = (A_s S_{-tau} x)^H (C_s y)."""
    fam, J, N, T = O.LEGALL53, 2, 16, 5
    y = RNG.normal(size=N) + 1j * RNG.normal(size=N)
    x = RNG.normal(size=T) + 1j * RNG.normal(size=T)
    rp = O.run_paper(fam, J, O.PERIODIC, N, y[None], x[None])
    # analysis operator on a zero-padded line long enough to hold every delayed template
    L = 64
    def op(role, Lin):
        lo, f = O.filt(fam, role, O.LOWPASS)
        M = np.zeros((Lin // 2, Lin))
        for k in range(Lin // 2):
            for i, m in enumerate(range(lo, lo + len(f))):
                n = 2 * k - m
                if 0 <= n < Lin:
                    M[k, n] += f[i]
        return M
    # dual operator on the N-periodic received row
    def op_per(Lin):
        lo, f = O.filt(fam, O.DUAL, O.LOWPASS)
        M = np.zeros((Lin // 2, Lin))
        for k in range(Lin // 2):
            for i, m in enumerate(range(lo, lo + len(f))):
                M[k, (2 * k - m) % Lin] += f[i]
        return M
    off = 16                                  # origin of the zero-padded template line
    for s in range(J + 1):
        A = np.eye(L)
        C = np.eye(N)
        for l in range(s):
            A = op(O.ANALYSIS, L >> l) @ A
            C = op_per(N >> l) @ C
        cy = C @ y
        for tau in range(N):
            xt = np.zeros(L, complex)
            xt[off + tau: off + tau + T] = x
            ax = A @ xt
            # coefficient k of the padded line <-> k - off / 2^s of the true line (off multiple of 2^s)
            ks = np.arange(ax.shape[0]) - off // (2 ** s)
            val = np.sum(np.conj(ax) * cy[np.mod(ks, N >> s)])
            assert abs(val - rp["corr"][0, 0, s, tau]) < 1e-10, (s, tau)


# ---------------------------------------------------------------- the free-t 9/7 family

T_EXACT = 1.2301741049140007        # include/sidwt.h SIDWT_CDF97_T_EXACT


def _cdf97_spectral():
    """The irrational CDF 9/7 lowpass pair (ref. [28] of the paper) built from scratch by
    spectral factorisation, independent of any lifting: |H|^2-type product
    cos^8(w/2) P(sin^2(w/2)) with P(y) = sum_{k<4} C(3+k, k) y^k; the complex root pair of P
    goes to the 9-tap filter, the real root to the 7-tap one; both normalised to DC gain sqrt2."""
    r = np.roots([math.comb(3 + k, k) for k in range(3, -1, -1)])
    y0 = r[np.argmin(abs(r.imag))].real
    yc = r[np.argmax(r.imag)]
    Y = np.array([-1, 2, -1]) / 4.0                       # sin^2(w/2) as a Laurent polynomial
    cos4 = np.convolve([1, 2, 1], [1, 2, 1]) / 16.0       # cos^4(w/2)
    one = np.array([0, 1.0, 0])
    f9 = np.convolve(cos4, np.real(np.convolve(one - Y / yc, one - Y / np.conj(yc))))
    f7 = np.convolve(cos4, one - Y / y0)
    f9, f7 = f9[np.abs(f9) > 1e-15], f7[np.abs(f7) > 1e-15]
    return f9 * math.sqrt(2) / f9.sum(), f7 * math.sqrt(2) / f7.sum()


def test_t97_lifting_expansion_reproduces_printed_filters():
    """At t = 5/4 the oracle's expansion of the lifting factorisations
    gives the printed 9/7 listings and their eq. (7) highpass filters."""
    for role in (O.ANALYSIS, O.DUAL):
        for which in (O.LOWPASS, O.HIGHPASS):
            lo_p, printed = O.filt(O.CDF97, role, which)
            lo_t, derived = O.filt_t97(1.25, role, which)
            assert lo_p == lo_t
            np.testing.assert_allclose(derived, printed, atol=1e-15)


def test_t97_exact_cdf_equals_spectral_factorisation():
    """At t = t* (alpha(t*) = the CDF value) the free-t family is the irrational CDF 9/7
    filterbank: both lowpass filters equal the spectral factorisation,
    and both highpass filters have four vanishing moments -- Table I's dual
    highpass has only two."""
    f9, f7 = _cdf97_spectral()
    lo, a = O.filt_t97(T_EXACT, O.ANALYSIS, O.LOWPASS)
    assert lo == -4 and len(a) == 9
    np.testing.assert_allclose(a, f9, atol=1e-14)
    lo, d = O.filt_t97(T_EXACT, O.DUAL, O.LOWPASS)
    assert lo == -3 and len(d) == 7
    np.testing.assert_allclose(d, f7, atol=1e-14)
    for role in (O.ANALYSIS, O.DUAL):
        lo, g = O.filt_t97(T_EXACT, role, O.HIGHPASS)
        m = np.arange(lo, lo + len(g), dtype=np.float64)
        for p in range(4):
            assert abs(np.sum(g * m ** p)) < 1e-12, (role, p)
        assert abs(np.sum(g * m ** 4)) > 1.0
    lo, g = O.filt_t97(1.25, O.DUAL, O.HIGHPASS)
    m = np.arange(lo, lo + len(g), dtype=np.float64)
    assert abs(np.sum(g * m ** 2)) > 0.1


@pytest.mark.parametrize("t", (0.8, T_EXACT, 1.6, 1.85))
def test_t97_biorthogonal_and_inner_product(t):
    """Any t of the family is a biorthogonal pair: dual^T analysis = I (eq. (11)/(13)) and
    the one-level inner-product identity <x, y> = <a, c> + <b, d> (eq. (4)/(15))."""
    with O.t97(t):
        for P in (8, 16, 32):
            Ma = _dense(O.CDF97, O.ANALYSIS, P)
            Md = _dense(O.CDF97, O.DUAL, P)
            np.testing.assert_allclose(Md.T @ Ma, np.eye(P), atol=1e-12)
            x = RNG.normal(size=P) + 1j * RNG.normal(size=P)
            y = RNG.normal(size=P) + 1j * RNG.normal(size=P)
            a, b = O.mallat_level(O.CDF97, O.ANALYSIS, x)
            c, d = O.mallat_level(O.CDF97, O.DUAL, y)
            assert abs(np.vdot(x, y) - np.vdot(a, c) - np.vdot(b, d)) < 1e-11 * (1 + abs(np.vdot(x, y)))
        # the setting is scoped
    lo, f = O.filt(O.CDF97, O.ANALYSIS, O.LOWPASS)
    np.testing.assert_allclose(f, O.filt_t97(1.25, O.ANALYSIS, O.LOWPASS)[1], atol=1e-15)


@pytest.mark.parametrize("ext", (O.PERIODIC, O.SYMMETRIC))
def test_t97_full_path_pins(ext):
    """Exact CDF 9/7 through the whole oracle: corr_0 is the textbook correlation (P9) and
    the telescoped eq. (4) form equals the approximation-domain form (P10) at every scale."""
    N, J, T = 64, 4, 23
    y = RNG.normal(size=N) + 1j * RNG.normal(size=N)
    x = RNG.normal(size=T) + 1j * RNG.normal(size=T)
    with O.t97(T_EXACT):
        r = O.run(O.CDF97, J, ext, N, y[None], x[None])
        pyr = O.template_pyramid(O.CDF97, J, x)
        lo = min(min(2 ** (i + 1) * k for i, (k, _) in enumerate(pyr[:-1])), 2 ** J * pyr[-1][0])
        hi = max(max(2 ** (i + 1) * (k + len(c) - 1) for i, (k, c) in enumerate(pyr[:-1])),
                 2 ** J * (pyr[-1][0] + len(pyr[-1][1]) - 1))
        rb = O.run(O.CDF97, J, ext, N, y[None], x[None], p_lo=lo, p_hi=N + hi + 1)
    ref = np.array([sum(np.conj(x[n]) * _extend(y, ext, np.array([n + tau]))[0] for n in range(T))
                    for tau in range(N)])
    np.testing.assert_allclose(r["corr"][0, 0, 0], ref, atol=1e-12)
    B = rb["bands"][0]
    corr = np.zeros(N, np.complex128)
    for i in range(J, -1, -1):
        k0, c = pyr[i]
        lev = i + 1 if i < J else J
        for j, cc in enumerate(c):
            corr = corr + np.conj(cc) * B[i, np.arange(N) + 2 ** lev * (k0 + j) - lo]
        s = i if i < J else J
        if i == J:
            np.testing.assert_allclose(r["corr"][0, 0, J], corr, atol=1e-10)
        else:
            np.testing.assert_allclose(r["corr"][0, 0, s], corr, atol=1e-10)
    # and it differs from Table I away from s = 0
    r125 = O.run(O.CDF97, J, ext, N, y[None], x[None])
    assert np.max(np.abs(r125["corr"][0, 0, 2] - r["corr"][0, 0, 2])) > 1e-6
