"""CPU-side checks of the C ABI: the library builds for sm_100a, loads, exports
every symbol include/sidwt.h declares, and validates arguments before touching
the device (so the status codes can be checked without a GPU)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def native():
    from paper_cs_0607001_b200 import _native
    _native.build()
    return _native


def test_header_symbols_exported(native):
    hdr = open(os.path.join(ROOT, "include", "sidwt.h")).read()
    declared = set(re.findall(r"^\s*(?:sidwt_status|int64_t|int|const char\*)\s+(sidwt_\w+)\s*\(", hdr, re.M))
    assert declared == set(native.EXPORTS), declared ^ set(native.EXPORTS)
    lib = native.lib()
    for name in declared:
        assert hasattr(lib, name), name
    out = os.popen(f"nm -D --defined-only {native.LIB_PATH}").read()
    for name in declared:
        assert re.search(rf"\bT {name}\b", out), f"{name} not exported with C linkage"


def test_sass_is_sm100a(native):
    """The library is sm_100a code and each kernel family carries its Blackwell-native
    instructions (tools/sass_evidence.py; summary in profiles/)."""
    import collections
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import sass_evidence as SE
    out = os.popen(f"cuobjdump --list-elf {native.LIB_PATH}").read()
    assert "sm_100a" in out
    per = collections.defaultdict(collections.Counter)
    for name, lines in SE.kernels(native.LIB_PATH).items():
        per[SE.short(name)].update(SE.counts(lines))
    # template-bank tensor-core correlation: tcgen05.mma, tcgen05.ld, TMA tensor stores of corr
    for k in ("UTCHMMA", "LDTM", "UTMASTG", "UBLKCP"):
        assert per["k_correlate_tc"][k] > 0, ("k_correlate_tc", k)
    # single-template tensor-core correlation: tcgen05.mma, tcgen05.ld, bulk copies
    for k in ("UTCHMMA", "LDTM", "UBLKCP"):
        assert per["k_correlate_tcs"][k] > 0, ("k_correlate_tcs", k)
    # integer family: int8 tcgen05.mma (UTCIMMA), tcgen05.ld, bulk loads, TMA tensor stores of corr
    for k in ("UTCIMMA", "LDTM", "UTMASTG", "UBLKCP"):
        assert per["k_correlate_i8"][k] > 0, ("k_correlate_i8", k)
    # per-role register budgets (setmaxnreg) in the three warp-specialised tensor-core kernels
    for kern in ("k_correlate_tc", "k_correlate_tcs", "k_correlate_i8"):
        assert per[kern]["USETMAXREG"] >= 2, (kern, "USETMAXREG")
    assert per["k_analyze"]["UBLKCP"] > 0                  # TMA bulk stores of the bands
    assert per["k_correlate"]["FFMA2"] > 0                 # packed FP32 real-template correlation


def test_plan_validation_without_gpu(native):
    L = native.lib()
    h = C.c_void_p()
    cases = [
        ((0, 3, 1000, 1, 0), 1),     # N not a power of two -> PARAM
        ((0, 3, 1, 1, 0), 1),        # N < 2
        ((9, 3, 64, 1, 0), 1),       # bad filter
        ((0, 3, 64, 1, 7), 1),       # bad ext
        ((0, 0, 64, 1, 0), 4),       # levels < 1 -> DEPTH
        ((0, 7, 64, 1, 0), 4),       # 2^J > N
        ((0, 17, 1 << 20, 1, 0), 4), # J > 16
        ((0, 3, 64, 0, 0), 3),       # batch < 1 -> DIMENSION
    ]
    for args, want in cases:
        assert L.sidwt_plan_create(C.byref(h), *args) == want, args
    assert L.sidwt_plan_create(C.byref(h), 0, 3, 64, 4, 0) == 0
    plan = h.value
    assert L.sidwt_band_stride(plan) == -1          # before template_load
    P = C.c_void_p
    assert L.sidwt_analyze(plan, P(1), 1, P(1), None) == 6      # STATE
    assert L.sidwt_correlate(plan, P(1), 1, P(1), None) == 6
    assert L.sidwt_peaks(plan, P(1), 1, P(1), None, None) == 6
    assert L.sidwt_run(plan, P(1), 1, P(1), P(1), P(1), None, None) == 6
    assert L.sidwt_plan_set_lifting_t(plan, 1.3) == 1                # PARAM: not a 9/7 plan
    assert L.sidwt_analyze(plan, None, 1, P(1), None) == 1      # PARAM
    assert L.sidwt_run(plan, P(1), 1, None, P(1), P(1), None, None) == 1
    x = (C.c_float * 2)()
    assert L.sidwt_template_load(plan, x, 0, 1) == 2            # LENGTH
    assert L.sidwt_template_load(plan, x, 65, 1) == 2
    assert L.sidwt_template_load(plan, x, 1, 0) == 3            # DIMENSION
    assert L.sidwt_plan_destroy(plan) == 0
    assert L.sidwt_plan_destroy(None) == 0
    # J = 11: the deepest analysis level needs 1024 branch threads > 512 -> RANGE, detected
    # before any device work (so also without a GPU)
    assert L.sidwt_plan_create(C.byref(h), 0, 11, 4096, 1, 0) == 0
    assert L.sidwt_template_load(h.value, x, 1, 1) == 5
    assert L.sidwt_band_stride(h.value) == -1
    assert L.sidwt_plan_destroy(h.value) == 0
    assert native.sidwt_status_string(6) == "state error"


def test_no_cpu_fallback_in_binding():
    """The binding must not import the oracle or compute anything itself."""
    src = open(os.path.join(ROOT, "paper_cs_0607001_b200", "_native.py")).read()
    src += open(os.path.join(ROOT, "paper_cs_0607001_b200", "__init__.py")).read()
    assert "oracle" not in src.replace("no CPU fallback", "")
