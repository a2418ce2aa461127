"""SIDWT-domain multiresolution correlation by lifting, B200 (sm_100a).

Python face of libsidwt (include/sidwt.h).  ``_native`` holds the functions with
the C names (argument marshalling only); ``Plan`` is a convenience wrapper that
allocates the device buffers with PyTorch (memory and streams only) and calls
the C ABI.  Nothing here computes any part of the path: no CPU fallback exists.
"""
from __future__ import annotations

import numpy as np

from . import _native
from ._native import (CDF97_T_EXACT, SIDWT_CDF97, SIDWT_DAUB4_CAUSAL, SIDWT_EXT_PERIODIC, SIDWT_EXT_SYMMETRIC,  # noqa: F401
                      SIDWT_LEGALL53, SIDWT_LEGALL53_INT, SIDWT_ORIENT_RECEIVED_TREE, SIDWT_ORIENT_TEMPLATE_TREE,
                      SidwtError)

__all__ = ["Plan", "SidwtError", "SIDWT_LEGALL53", "SIDWT_CDF97", "SIDWT_DAUB4_CAUSAL",
           "SIDWT_LEGALL53_INT", "SIDWT_EXT_PERIODIC", "SIDWT_EXT_SYMMETRIC", "SIDWT_ORIENT_RECEIVED_TREE",
           "SIDWT_ORIENT_TEMPLATE_TREE", "CDF97_T_EXACT"]


class Plan:
    """Owns one sidwt_plan.  Device tensors are torch tensors on ``device``."""

    def __init__(self, filter: int, levels: int, N: int, batch: int, ext: int, device="cuda", orientation: int = 0,
                 lifting_t: float | None = None):
        import torch  # plumbing only
        self.torch = torch
        self.filter, self.levels, self.N, self.batch, self.ext = filter, levels, N, batch, ext
        self.device = torch.device(device)
        self.handle = _native.sidwt_plan_create(filter, levels, N, batch, ext)
        self.orientation = orientation
        if orientation:
            _native.sidwt_plan_set_orientation(self.handle, orientation)
        self.lifting_t = 1.25 if lifting_t is None else float(lifting_t)
        if lifting_t is not None:
            _native.sidwt_plan_set_lifting_t(self.handle, lifting_t)
        self.n_templates = 0
        self.T = 0

    @property
    def is_int(self) -> bool:
        return self.filter == SIDWT_LEGALL53_INT

    def close(self):
        if self.handle:
            _native.sidwt_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- templates
    def load_templates(self, templates: np.ndarray):
        """templates: complex64 [n][T] (float families) or int16 [n][T][2] (integer family)."""
        t = np.ascontiguousarray(templates)
        if self.is_int:
            assert t.dtype == np.int16 and t.ndim == 3 and t.shape[2] == 2
        else:
            t = t.astype(np.complex64)
            if t.ndim == 1:
                t = t[None]
        n, T = t.shape[0], t.shape[1]
        _native.sidwt_template_load(self.handle, t, T, n)
        self.n_templates, self.T = n, T
        return self

    @property
    def band_stride(self) -> int:
        return _native.sidwt_band_stride(self.handle)

    @property
    def band_offset(self) -> int:
        return _native.sidwt_band_offset(self.handle)

    def template_taps(self):
        """List over templates of [(kmin, taps complex / int [n][2]) for b_1..b_J, a_J]."""
        J = self.levels
        kmin = np.zeros(J + 1, np.int32)
        cnt = np.zeros(J + 1, np.int32)
        per_t = _native.sidwt_template_taps(self.handle, None, kmin, cnt)
        raw = np.zeros((self.n_templates, per_t, 2), np.int32 if self.is_int else np.float32)
        _native.sidwt_template_taps(self.handle, raw, kmin, cnt)
        out = []
        for t in range(self.n_templates):
            off, terms = 0, []
            for i in range(J + 1):
                c = raw[t, off:off + cnt[i]]
                terms.append((int(kmin[i]), c.copy() if self.is_int else (c[:, 0] + 1j * c[:, 1])))
                off += cnt[i]
            out.append(terms)
        return out

    # ---- buffers
    def empty_bands(self, rows: int):
        dt = self.torch.int32 if self.is_int else self.torch.float32
        return self.torch.empty((rows, self.levels + 1, 2, self.band_stride), dtype=dt, device=self.device)

    def empty_corr(self, rows: int):
        dt = self.torch.int32 if self.is_int else self.torch.float32
        return self.torch.empty((rows, self.n_templates, self.levels + 1, self.N, 2), dtype=dt, device=self.device)

    def empty_peaks(self, rows: int):
        dt = self.torch.int32 if self.is_int else self.torch.float32
        lag = self.torch.empty((rows, self.n_templates, self.levels + 1), dtype=self.torch.int32, device=self.device)
        val = self.torch.empty((rows, self.n_templates, self.levels + 1, 2), dtype=dt, device=self.device)
        return lag, val

    def rows_to_device(self, rows: np.ndarray):
        r = np.ascontiguousarray(rows)
        if self.is_int:
            t = self.torch.from_numpy(r.view(np.int16)).to(self.device)
        else:
            t = self.torch.from_numpy(r.astype(np.complex64).view(np.float32)).to(self.device)
        return t

    # ---- the path
    def _stream(self, stream):
        return stream if stream is not None else self.torch.cuda.current_stream(self.device)

    def analyze(self, d_rows, rows: int, bands=None, stream=None):
        bands = self.empty_bands(rows) if bands is None else bands
        _native.sidwt_analyze(self.handle, d_rows, rows, bands, self._stream(stream))
        return bands

    def correlate(self, bands, rows: int, corr=None, stream=None):
        corr = self.empty_corr(rows) if corr is None else corr
        _native.sidwt_correlate(self.handle, bands, rows, corr, self._stream(stream))
        return corr

    def peaks(self, corr, rows: int, lag=None, val=None, stream=None):
        if lag is None:
            lag, val = self.empty_peaks(rows)
        _native.sidwt_peaks(self.handle, corr, rows, lag, val, self._stream(stream))
        return lag, val

    def correlate_peaks(self, bands, rows: int, corr=None, lag=None, val=None, want_corr=True, stream=None):
        if corr is None and want_corr:
            corr = self.empty_corr(rows)
        if lag is None:
            lag, val = self.empty_peaks(rows)
        _native.sidwt_correlate_peaks(self.handle, bands, rows, corr, lag, val, self._stream(stream))
        return corr, lag, val

    def run(self, d_rows, rows: int, bands=None, corr=None, lag=None, val=None, want_corr=True, stream=None):
        """Whole path (analyze -> correlate -> peaks) with the analysis of the next row chunk
        overlapping the correlation of the current one; same outputs as analyze + correlate_peaks."""
        if bands is None:
            bands = self.empty_bands(rows)
        if corr is None and want_corr:
            corr = self.empty_corr(rows)
        if lag is None:
            lag, val = self.empty_peaks(rows)
        _native.sidwt_run(self.handle, d_rows, rows, bands, corr, lag, val, self._stream(stream))
        return corr, lag, val

    def fused_available(self) -> bool:
        return _native.sidwt_fused_available(self.handle) == 1

    def analyze_correlate(self, d_rows, rows: int, corr=None, lag=None, val=None, want_corr=True, stream=None):
        """Fused analyze -> correlate -> peaks (no band round trip); single-template plans."""
        if corr is None and want_corr:
            corr = self.empty_corr(rows)
        if lag is None:
            lag, val = self.empty_peaks(rows)
        _native.sidwt_analyze_correlate(self.handle, d_rows, rows, corr, lag, val, self._stream(stream))
        return corr, lag, val

    def synthesize(self, bands, rows: int, level: int = 0, out=None, stream=None):
        """Inverse lifting: U_level at positions 0..N-1 ([rows][N][2] float32 / int32)."""
        if out is None:
            dt = self.torch.int32 if self.is_int else self.torch.float32
            out = self.torch.empty((rows, self.N, 2), dtype=dt, device=self.device)
        _native.sidwt_synthesize(self.handle, bands, rows, level, out, self._stream(stream))
        return out

    def execute_host(self, h_rows, rows: int, h_lag, h_val=None, stream=None):
        _native.sidwt_execute_host(self.handle, h_rows, rows, h_lag, h_val, self._stream(stream))

    def template_is_real(self) -> bool:
        return _native.sidwt_template_is_real(self.handle) == 1

    def uses_tensor_cores(self) -> bool:
        """True when the correlation runs on the tensor cores (template bank or single template)."""
        return _native.sidwt_uses_tensor_cores(self.handle) > 0

    def tensor_core_path(self) -> int:
        """0: SIMT correlation; 1: template-bank tcgen05 kernel; 2: single-template tcgen05 kernel."""
        return _native.sidwt_uses_tensor_cores(self.handle)

    def last_launches(self) -> int:
        return _native.sidwt_last_launches(self.handle)
