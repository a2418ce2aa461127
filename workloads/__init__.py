"""Seeded synthetic workloads for the five BASELINE.json configurations.

This module is shared by the oracle-side tests and the CUDA-side harness, and it
holds NONE of the method's arithmetic (no lifting, no filtering, no
correlation): only the signal model of the paper's Section IV/V and the
parameters of each configuration.

* LFM chirp, Eq. (18): x(t) = exp(i*pi*K*t^2) rect(t/T_p),
  sampled at B samples/s over T_p, i.e. BT_p = beta is the time-bandwidth
  product. Reading (DESIGN.md R-D12): with N_c samples,
  x[n] = exp(i*pi*beta*(n - N_c/2)^2 / N_c^2), n = 0..N_c-1.
* Point-target backscatter: y[n] = sum_k sigma_k x[n - d_k],
  plus circular complex Gaussian noise.

Every row r of configuration c is drawn from its own generator
``np.random.default_rng(np.random.SeedSequence([0x51D7, c, r]))`` so any subset
of rows can be regenerated independently. The order in
which a row's random numbers are drawn is fixed here and documented per config.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED_TAG = 0x51D7

# Filter families / extensions, same integer codes as include/sidwt.h.
LEGALL53, CDF97, DAUB4_CAUSAL, LEGALL53_INT = 0, 1, 2, 3
PERIODIC, SYMMETRIC = 0, 1

FAMILY_NAMES = {LEGALL53: "legall53", CDF97: "cdf97",
                DAUB4_CAUSAL: "daub4_causal", LEGALL53_INT: "legall53_int"}

BARKER13 = (1, 1, 1, 1, 1, -1, -1, 1, 1, -1, 1, -1, 1)


@dataclasses.dataclass(frozen=True)
class Config:
    cid: int            # 1..5 (BASELINE.json configs[cid-1])
    name: str
    family: int
    levels: int
    ext: int
    N: int
    rows: int
    T: int
    n_templates: int
    description: str

    @property
    def is_int(self) -> bool:
        return self.family == LEGALL53_INT


CONFIGS = {
    1: Config(1, "C1", LEGALL53, 3, PERIODIC, 1024, 1, 64, 1,
              "single pulse, LeGall 5/3, J=3, periodic; LFM N_c=64, BT=32; 10 dB"),
    2: Config(2, "C2", DAUB4_CAUSAL, 5, SYMMETRIC, 4096, 4096, 130, 1,
              "causal Daubechies-4, J=5, symmetric; Barker-13 x10; 0 dB"),
    3: Config(3, "C3", CDF97, 6, SYMMETRIC, 8192, 16384, 512, 1,
              "CDF 9/7 (Table I), J=6, symmetric; LFM N_c=512, BT=100; 1-4 Rayleigh echoes; -5 dB"),
    4: Config(4, "C4", CDF97, 4, SYMMETRIC, 16384, 2048, 256, 64,
              "CDF 9/7, J=4, symmetric; bank of 64 Doppler-shifted LFM (256, BT=64); 1-3 members; 0 dB"),
    5: Config(5, "C5", LEGALL53_INT, 8, SYMMETRIC, 4096, 65536, 128, 1,
              "reversible integer 5/3, J=8, symmetric; 12-bit LFM N_c=128, BT=50; sigma=200 LSB"),
}


def lfm(n_c: int, beta: float) -> np.ndarray:
    """Eq. (18) sampled: exp(i*pi*beta*(n - N_c/2)^2 / N_c^2), complex128."""
    n = np.arange(n_c, dtype=np.float64)
    return np.exp(1j * math.pi * beta * (n - n_c / 2.0) ** 2 / float(n_c) ** 2)


def templates(cfg: Config) -> np.ndarray:
    """Template bank [n_templates][T]: complex64 for float configs, int16 [n][T][2] (I,Q) for C5."""
    c = cfg.cid
    if c == 1:
        return lfm(64, 32.0).astype(np.complex64)[None, :]
    if c == 2:
        chips = np.repeat(np.array(BARKER13, dtype=np.float64), 10)
        return chips.astype(np.complex64)[None, :]
    if c == 3:
        return lfm(512, 100.0).astype(np.complex64)[None, :]
    if c == 4:
        base = lfm(256, 64.0)
        n = np.arange(256, dtype=np.float64)
        bank = np.stack([base * np.exp(2j * math.pi * k * n / (64.0 * 256.0)) for k in range(64)])
        return bank.astype(np.complex64)
    if c == 5:
        ph = np.angle(lfm(128, 50.0))
        iq = np.stack([np.round(2047.0 * np.cos(ph)), np.round(2047.0 * np.sin(ph))], axis=-1)
        return iq.astype(np.int16)[None, :, :]
    raise ValueError(c)


def row_rng(cid: int, r: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([SEED_TAG, cid, r]))


def _noise(rng, n, var):
    s = math.sqrt(var / 2.0)
    return rng.normal(0.0, s, n) + 1j * rng.normal(0.0, s, n)


def make_row(cfg: Config, r: int, tmpl=None):
    """One received row and its ground truth.

    Returns (row, truth) with row complex64 [N] (float configs) or int16 [N][2]
    (C5), truth a list of (template_index, lag, amplitude).
    Draw order per row: echo count (C3/C4), then per echo (template index (C4),
    lag, amplitude), then noise re[N], noise im[N].
    """
    if tmpl is None:
        tmpl = templates(cfg)
    rng = row_rng(cfg.cid, r)
    N, T = cfg.N, cfg.T
    c = cfg.cid
    truth = []
    if c == 5:
        lag = int(rng.integers(0, N - T))
        y = np.zeros((N, 2), dtype=np.float64)
        y[lag:lag + T] += tmpl[0].astype(np.float64)
        y[:, 0] += np.round(rng.normal(0.0, 200.0, N))
        y[:, 1] += np.round(rng.normal(0.0, 200.0, N))
        y = np.clip(y, -32768, 32767).astype(np.int16)
        truth.append((0, lag, 1.0))
        return y, truth
    y = np.zeros(N, dtype=np.complex128)
    t64 = tmpl.astype(np.complex128)
    if c == 1:
        lag = int(rng.integers(0, N - T))
        y[lag:lag + T] += t64[0]
        truth.append((0, lag, 1.0))
        y += _noise(rng, N, 0.1)
    elif c == 2:
        lag = int(rng.integers(0, N - T))
        amp = np.exp(1j * rng.uniform(0.0, 2 * math.pi))
        y[lag:lag + T] += amp * t64[0]
        truth.append((0, lag, amp))
        y += _noise(rng, N, 1.0)
    elif c == 3:
        p = int(rng.integers(1, 5))
        for _ in range(p):
            lag = int(rng.integers(0, N - T))
            amp = (rng.normal(0.0, math.sqrt(0.5)) + 1j * rng.normal(0.0, math.sqrt(0.5)))
            y[lag:lag + T] += amp * t64[0]
            truth.append((0, lag, amp))
        y += _noise(rng, N, 10.0 ** 0.5)
    elif c == 4:
        p = int(rng.integers(1, 4))
        for _ in range(p):
            k = int(rng.integers(0, 64))
            lag = int(rng.integers(0, N - T))
            amp = np.exp(1j * rng.uniform(0.0, 2 * math.pi))
            y[lag:lag + T] += amp * t64[k]
            truth.append((k, lag, amp))
        y += _noise(rng, N, 1.0)
    return y.astype(np.complex64), truth


def make_rows(cfg: Config, start: int, count: int, tmpl=None) -> np.ndarray:
    """Rows [start, start+count): complex64 [count][N] or int16 [count][N][2]."""
    if tmpl is None:
        tmpl = templates(cfg)
    if cfg.is_int:
        out = np.empty((count, cfg.N, 2), dtype=np.int16)
    else:
        out = np.empty((count, cfg.N), dtype=np.complex64)
    for i in range(count):
        out[i], _ = make_row(cfg, start + i, tmpl)
    return out


def shard(n_rows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row block of rank `rank` out of `world` (weak-scaling partition)."""
    base, rem = divmod(n_rows, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)
