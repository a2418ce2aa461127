"""Thin ctypes binding of libsidwt (include/sidwt.h): argument marshalling only.

Every step of the path runs in the CUDA kernels of csrc/; this module never
computes anything and has no CPU fallback: if the shared library is missing or
fails to load, the import raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "libsidwt.so")
CSRC = os.path.join(HERE, "csrc")
HEADERS = [os.path.join(CSRC, f) for f in ("kernels.cuh", "lifting.cuh", "corr_tc.cuh", "corr_tcs.cuh", "fused.cuh",
                                           "corr_i8.h")] + [os.path.join(ROOT, "include", "sidwt.h")]
# translation units (compiled separately, in parallel, then linked into one shared library)
UNITS = [os.path.join(CSRC, "sidwt.cu"), os.path.join(CSRC, "corr_i8.cu")]
SOURCES = UNITS + HEADERS
BUILD_DIR = os.path.join(ROOT, "build")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC"]

SIDWT_LEGALL53, SIDWT_CDF97, SIDWT_DAUB4_CAUSAL, SIDWT_LEGALL53_INT = 0, 1, 2, 3
SIDWT_EXT_PERIODIC, SIDWT_EXT_SYMMETRIC = 0, 1
SIDWT_ORIENT_RECEIVED_TREE, SIDWT_ORIENT_TEMPLATE_TREE = 0, 1

CDF97_T_EXACT = 1.2301741049140007   # include/sidwt.h SIDWT_CDF97_T_EXACT (irrational CDF 9/7)
STATUS = {0: "SIDWT_OK", 1: "SIDWT_ERR_PARAM", 2: "SIDWT_ERR_LENGTH", 3: "SIDWT_ERR_DIMENSION",
          4: "SIDWT_ERR_DEPTH", 5: "SIDWT_ERR_RANGE", 6: "SIDWT_ERR_STATE", 7: "SIDWT_ERR_OOM",
          8: "SIDWT_ERR_CUDA"}

# every symbol include/sidwt.h declares
EXPORTS = ["sidwt_plan_create", "sidwt_plan_set_orientation", "sidwt_plan_set_lifting_t", "sidwt_plan_destroy", "sidwt_template_load", "sidwt_analyze",
           "sidwt_correlate", "sidwt_peaks", "sidwt_correlate_peaks", "sidwt_run", "sidwt_analyze_correlate", "sidwt_synthesize",
           "sidwt_execute_host", "sidwt_fused_available",
           "sidwt_band_stride", "sidwt_band_offset", "sidwt_bands_bytes", "sidwt_corr_bytes",
           "sidwt_template_taps", "sidwt_last_launches", "sidwt_uses_tensor_cores", "sidwt_template_is_real",
           "sidwt_status_string"]


def build(force: bool = False, verbose: bool = False) -> str:
    """nvcc -gencode arch=compute_100a,code=sm_100a: each translation unit of csrc/ -> build/*.o
    (rebuilt when it or a header changed), linked into paper_cs_0607001_b200/libsidwt.so."""
    os.makedirs(BUILD_DIR, exist_ok=True)
    newest_hdr = max(os.path.getmtime(h) for h in HEADERS)
    procs, objs = [], []
    for src in UNITS:
        obj = os.path.join(BUILD_DIR, os.path.basename(src).replace(".cu", ".o"))
        objs.append(obj)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), newest_hdr):
            cmd = ["nvcc", *NVCC_FLAGS, "-c", "-o", obj, src]
            if os.environ.get("SIDWT_TC_PROFILE"):        # debug: timed role waits in the tensor-core kernels
                cmd.insert(1, "-DSIDWT_TC_PROFILE")
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            procs.append((subprocess.Popen(cmd), cmd))
    for pr, cmd in procs:
        if pr.wait() != 0:
            raise subprocess.CalledProcessError(pr.returncode, cmd)
    if force or procs or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(map(os.path.getmtime, objs)):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB_PATH, *objs])
    return LIB_PATH


class SidwtError(RuntimeError):
    def __init__(self, fn, status):
        super().__init__(f"{fn} -> {STATUS.get(status, status)}")
        self.status = status


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libsidwt.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        P, I64, I = C.c_void_p, C.c_int64, C.c_int
        L.sidwt_plan_create.argtypes = [C.POINTER(P), I, I, I64, I64, I]
        L.sidwt_plan_destroy.argtypes = [P]
        L.sidwt_plan_set_orientation.argtypes = [P, I]
        L.sidwt_plan_set_lifting_t.argtypes = [P, C.c_double]
        L.sidwt_template_load.argtypes = [P, P, I64, I]
        L.sidwt_analyze.argtypes = [P, P, I64, P, P]
        L.sidwt_correlate.argtypes = [P, P, I64, P, P]
        L.sidwt_peaks.argtypes = [P, P, I64, P, P, P]
        L.sidwt_correlate_peaks.argtypes = [P, P, I64, P, P, P, P]
        L.sidwt_execute_host.argtypes = [P, P, I64, P, P, P]
        L.sidwt_run.argtypes = [P, P, I64, P, P, P, P, P]
        L.sidwt_synthesize.argtypes = [P, P, I64, I, P, P]
        L.sidwt_analyze_correlate.argtypes = [P, P, I64, P, P, P, P]
        L.sidwt_fused_available.argtypes = [P]
        L.sidwt_fused_available.restype = I
        for f in ("sidwt_band_stride", "sidwt_band_offset"):
            getattr(L, f).argtypes = [P]
            getattr(L, f).restype = I64
        for f in ("sidwt_bands_bytes", "sidwt_corr_bytes"):
            getattr(L, f).argtypes = [P, I64]
            getattr(L, f).restype = I64
        L.sidwt_template_taps.argtypes = [P, P, P, P]
        L.sidwt_template_taps.restype = I64
        L.sidwt_last_launches.argtypes = [P]
        L.sidwt_last_launches.restype = I
        L.sidwt_uses_tensor_cores.argtypes = [P]
        L.sidwt_uses_tensor_cores.restype = I
        L.sidwt_template_is_real.argtypes = [P]
        L.sidwt_template_is_real.restype = I
        L.sidwt_status_string.argtypes = [I]
        L.sidwt_status_string.restype = C.c_char_p
        _lib = L
    return _lib


def _ptr(x):
    """Device/host pointer of a torch tensor / numpy array / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    raise TypeError(type(x))


def _stream(s):
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


def _check(fn, st):
    if st != 0:
        raise SidwtError(fn, st)


# ---- functions with the C names -------------------------------------------------------

def sidwt_plan_create(filter: int, levels: int, N: int, batch: int, ext: int) -> int:
    h = C.c_void_p()
    _check("sidwt_plan_create", lib().sidwt_plan_create(C.byref(h), filter, levels, N, batch, ext))
    return h.value


def sidwt_plan_set_orientation(plan: int, orientation: int) -> None:
    _check("sidwt_plan_set_orientation", lib().sidwt_plan_set_orientation(plan, orientation))


def sidwt_plan_set_lifting_t(plan: int, t: float) -> None:
    _check("sidwt_plan_set_lifting_t", lib().sidwt_plan_set_lifting_t(plan, float(t)))


def sidwt_plan_destroy(plan: int) -> None:
    _check("sidwt_plan_destroy", lib().sidwt_plan_destroy(plan))


def sidwt_template_load(plan: int, host_templates, T: int, n_templates: int) -> None:
    _check("sidwt_template_load", lib().sidwt_template_load(plan, _ptr(host_templates), T, n_templates))


def sidwt_analyze(plan, d_rows, rows, d_bands, stream=None):
    _check("sidwt_analyze", lib().sidwt_analyze(plan, _ptr(d_rows), rows, _ptr(d_bands), _stream(stream)))


def sidwt_correlate(plan, d_bands, rows, d_corr, stream=None):
    _check("sidwt_correlate", lib().sidwt_correlate(plan, _ptr(d_bands), rows, _ptr(d_corr), _stream(stream)))


def sidwt_peaks(plan, d_corr, rows, d_lag, d_val=None, stream=None):
    _check("sidwt_peaks", lib().sidwt_peaks(plan, _ptr(d_corr), rows, _ptr(d_lag), _ptr(d_val), _stream(stream)))


def sidwt_correlate_peaks(plan, d_bands, rows, d_corr, d_lag, d_val=None, stream=None):
    _check("sidwt_correlate_peaks", lib().sidwt_correlate_peaks(
        plan, _ptr(d_bands), rows, _ptr(d_corr), _ptr(d_lag), _ptr(d_val), _stream(stream)))


def sidwt_run(plan, d_rows, rows, d_bands, d_corr, d_lag, d_val=None, stream=None):
    _check("sidwt_run", lib().sidwt_run(
        plan, _ptr(d_rows), rows, _ptr(d_bands), _ptr(d_corr), _ptr(d_lag), _ptr(d_val), _stream(stream)))


def sidwt_analyze_correlate(plan, d_rows, rows, d_corr, d_lag, d_val=None, stream=None):
    _check("sidwt_analyze_correlate", lib().sidwt_analyze_correlate(
        plan, _ptr(d_rows), rows, _ptr(d_corr), _ptr(d_lag), _ptr(d_val), _stream(stream)))


def sidwt_fused_available(plan) -> int:
    return lib().sidwt_fused_available(plan)


def sidwt_synthesize(plan, d_bands, rows, level, d_out, stream=None):
    _check("sidwt_synthesize", lib().sidwt_synthesize(plan, _ptr(d_bands), rows, level, _ptr(d_out), _stream(stream)))


def sidwt_execute_host(plan, h_rows, rows, h_lag, h_val=None, stream=None):
    _check("sidwt_execute_host", lib().sidwt_execute_host(
        plan, _ptr(h_rows), rows, _ptr(h_lag), _ptr(h_val), _stream(stream)))


def sidwt_band_stride(plan) -> int:
    return lib().sidwt_band_stride(plan)


def sidwt_band_offset(plan) -> int:
    return lib().sidwt_band_offset(plan)


def sidwt_bands_bytes(plan, rows) -> int:
    return lib().sidwt_bands_bytes(plan, rows)


def sidwt_corr_bytes(plan, rows) -> int:
    return lib().sidwt_corr_bytes(plan, rows)


def sidwt_template_taps(plan, host_taps=None, kmin=None, count=None) -> int:
    return lib().sidwt_template_taps(plan, _ptr(host_taps), _ptr(kmin), _ptr(count))


def sidwt_last_launches(plan) -> int:
    return lib().sidwt_last_launches(plan)


def sidwt_uses_tensor_cores(plan) -> int:
    return lib().sidwt_uses_tensor_cores(plan)


def sidwt_template_is_real(plan) -> int:
    return lib().sidwt_template_is_real(plan)


def sidwt_status_string(st: int) -> str:
    return lib().sidwt_status_string(st).decode()
