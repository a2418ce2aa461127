"""ctypes wrapper of the CPU oracle (oracle/oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with
the CUDA library (paper_cs_0607001_b200); the only common dependency is the
seeded input generator module ``workloads`` (which holds none of the method's
arithmetic).  Parity: see the header of oracle.c and DESIGN.md.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

LEGALL53, CDF97, DAUB4, LEGALL53_INT = 0, 1, 2, 3
ANALYSIS, DUAL = 0, 1
LOWPASS, HIGHPASS = 0, 1
PERIODIC, SYMMETRIC = 0, 1


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, OpenMP)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", SRC, "-o", LIB, "-lm"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        P = C.c_void_p
        i = C.c_int
        L.oracle_filter.argtypes = [i, i, i, C.POINTER(i), C.POINTER(i), P]
        L.oracle_support.argtypes = [i, i, i, i, C.POINTER(i), C.POINTER(i)]
        L.oracle_mallat_level.argtypes = [i, i, i, P, P, P]
        L.oracle_int_level.argtypes = [i, i, P, P, P]
        L.oracle_template_pyramid.argtypes = [i, i, i, P, P]
        L.oracle_run.argtypes = [i, i, i, i, i, P, i, i, P, i, i, P, P, P, P, i]
        L.oracle_max_threads.restype = i
        L.oracle_approx.argtypes = [i, i, i, i, P, i, i, i, P, i]
        L.oracle_run_paper.argtypes = [i, i, i, i, i, P, i, i, P, P, P, P, i]
        L.oracle_set_t97.argtypes = [C.c_double]
        L.oracle_get_t97.restype = C.c_double
        L.oracle_filter_t97.argtypes = [C.c_double, i, i, C.POINTER(i), C.POINTER(i), P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def filt(family: int, role: int, which: int):
    """(lo, taps) with taps[m - lo] the coefficient of z^-m (Mallat: out[k] = sum f[m] v[2k-m])."""
    lo, hi = C.c_int(), C.c_int()
    taps = np.zeros(32, dtype=np.float64)
    assert lib().oracle_filter(family, role, which, C.byref(lo), C.byref(hi), _p(taps)) == 0
    return lo.value, taps[: hi.value - lo.value + 1].copy()


class t97:
    """Context manager: CDF 9/7 free parameter t for every CDF97 call
    inside the block (default 5/4 = Table I).  Process-wide; not thread-safe."""

    def __init__(self, t: float):
        self.t = float(t)

    def __enter__(self):
        self.prev = lib().oracle_get_t97()
        lib().oracle_set_t97(self.t)
        return self

    def __exit__(self, *exc):
        lib().oracle_set_t97(self.prev)
        return False


def filt_t97(t: float, role: int, which: int):
    """The 9/7 filter of parameter t from the lifting factorisation (not the printed listing)."""
    lo, hi = C.c_int(), C.c_int()
    taps = np.zeros(32, dtype=np.float64)
    assert lib().oracle_filter_t97(float(t), role, which, C.byref(lo), C.byref(hi), _p(taps)) == 0
    return lo.value, taps[: hi.value - lo.value + 1].copy()


def support(family: int, T: int, s: int, which: int):
    a, b = C.c_int(), C.c_int()
    assert lib().oracle_support(family, T, s, which, C.byref(a), C.byref(b)) == 0
    return a.value, b.value


def mallat_level(family: int, role: int, v: np.ndarray):
    v = np.ascontiguousarray(v, dtype=np.complex128)
    P = v.shape[0]
    Po = P // 2 if P % 2 == 0 else P
    c = np.zeros(Po, np.complex128)
    d = np.zeros(Po, np.complex128)
    assert lib().oracle_mallat_level(family, role, P, _p(v), _p(c), _p(d)) == 0
    return c, d


def int_level(role: int, v: np.ndarray):
    v = np.ascontiguousarray(v, dtype=np.int64)
    P = v.shape[0]
    Po = P // 2 if P % 2 == 0 else P
    c = np.zeros(Po, np.int64)
    d = np.zeros(Po, np.int64)
    assert lib().oracle_int_level(role, P, _p(v), _p(c), _p(d)) == 0
    return c, d


def supports(family: int, J: int, T: int):
    """[(kmin,kmax) of b_1..b_J] + [(kmin,kmax) of a_J]."""
    out = [support(family, T, s, HIGHPASS) for s in range(1, J + 1)]
    out.append(support(family, T, J, LOWPASS))
    return out


def template_pyramid(family: int, J: int, x: np.ndarray):
    """List of (kmin, coeffs) for b_1..b_J, a_J (complex128, or int64 [n][2] for the int family)."""
    T = x.shape[0]
    sup = supports(family, J, T)
    total = sum(b - a + 1 for a, b in sup)
    if family == LEGALL53_INT:
        x = np.ascontiguousarray(x, dtype=np.int16)
        out = np.zeros((total, 2), np.int64)
    else:
        x = np.ascontiguousarray(x, dtype=np.complex128)
        out = np.zeros(total, np.complex128)
    n = lib().oracle_template_pyramid(family, J, T, _p(x), _p(out))
    assert n == total, (n, total)
    res, off = [], 0
    for a, b in sup:
        res.append((a, out[off: off + b - a + 1].copy()))
        off += b - a + 1
    return res


def run(family: int, J: int, ext: int, N: int, y: np.ndarray, x: np.ndarray,
        p_lo: int | None = None, p_hi: int | None = None, corr: bool = True,
        nthreads: int = 0):
    """Full oracle path over rows y against templates x.

    y: complex [rows][N] (float families) or int16 [rows][N][2]
    x: complex [n_t][T]                   or int16 [n_t][T][2]
    Returns dict(bands=[rows][J+1][p_hi-p_lo] (complex128 / int64 [..][2]) or None,
                 corr=[rows][n_t][J+1][N] complex128 / int32 [..][2] or None,
                 lag=[rows][n_t][J+1] int32, val=... )
    """
    isint = family == LEGALL53_INT
    if isint:
        y = np.ascontiguousarray(y, dtype=np.int16)
        x = np.ascontiguousarray(x, dtype=np.int16)
        if y.ndim == 2:
            y = y[None]
        if x.ndim == 2:
            x = x[None]
    else:
        y = np.ascontiguousarray(y, dtype=np.complex128)
        x = np.ascontiguousarray(x, dtype=np.complex128)
        if y.ndim == 1:
            y = y[None]
        if x.ndim == 1:
            x = x[None]
    rows, n_t, T = y.shape[0], x.shape[0], x.shape[1]
    bands = None
    if p_lo is not None:
        nb = p_hi - p_lo
        bands = np.zeros((rows, J + 1, nb, 2), np.int64) if isint else np.zeros((rows, J + 1, nb), np.complex128)
    else:
        p_lo, p_hi = 0, 0
    cr = None
    if corr:
        cr = np.zeros((rows, n_t, J + 1, N, 2), np.int32) if isint else np.zeros((rows, n_t, J + 1, N), np.complex128)
    lag = np.zeros((rows, n_t, J + 1), np.int32)
    val = np.zeros((rows, n_t, J + 1, 2), np.int32) if isint else np.zeros((rows, n_t, J + 1), np.complex128)
    rc = lib().oracle_run(family, J, ext, N, rows, _p(y), T, n_t, _p(x), p_lo, p_hi, _p(bands),
                          _p(cr), _p(lag), _p(val), nthreads)
    if rc != 0:
        raise ValueError("oracle_run rejected its arguments")
    return dict(bands=bands, corr=cr, lag=lag, val=val)


def approx(family: int, ext: int, N: int, y: np.ndarray, s: int, p_lo: int = 0, p_hi: int | None = None,
           nthreads: int = 0):
    """Approximation band U_s of each row at positions [p_lo, p_hi) (default [0, N)):
    complex128 [rows][n] (float families) or int64 [rows][n][2] (integer family)."""
    isint = family == LEGALL53_INT
    p_hi = N if p_hi is None else p_hi
    if isint:
        y = np.ascontiguousarray(y, dtype=np.int16)
        if y.ndim == 2:
            y = y[None]
        out = np.zeros((y.shape[0], p_hi - p_lo, 2), np.int64)
    else:
        y = np.ascontiguousarray(y, dtype=np.complex128)
        if y.ndim == 1:
            y = y[None]
        out = np.zeros((y.shape[0], p_hi - p_lo), np.complex128)
    if lib().oracle_approx(family, ext, N, y.shape[0], _p(y), s, p_lo, p_hi, _p(out), nthreads) != 0:
        raise ValueError("oracle_approx rejected its arguments")
    return out


def run_paper(family: int, J: int, ext: int, N: int, y: np.ndarray, x: np.ndarray, nthreads: int = 0):
    """The paper's orientation: corr[rows][n_t][J+1][N] of
    <A_s (x delayed by tau), C_s ybar>, lag and val; float families only."""
    y = np.ascontiguousarray(y, dtype=np.complex128)
    x = np.ascontiguousarray(x, dtype=np.complex128)
    if y.ndim == 1:
        y = y[None]
    if x.ndim == 1:
        x = x[None]
    rows, n_t, T = y.shape[0], x.shape[0], x.shape[1]
    cr = np.zeros((rows, n_t, J + 1, N), np.complex128)
    lag = np.zeros((rows, n_t, J + 1), np.int32)
    val = np.zeros((rows, n_t, J + 1), np.complex128)
    if lib().oracle_run_paper(family, J, ext, N, rows, _p(y), T, n_t, _p(x), _p(cr), _p(lag), _p(val), nthreads) != 0:
        raise ValueError("oracle_run_paper rejected its arguments")
    return dict(corr=cr, lag=lag, val=val)


def max_threads() -> int:
    return lib().oracle_max_threads()
