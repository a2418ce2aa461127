#!/usr/bin/env python
"""Benchmark: SIDWT lifting + correlation throughput (complex samples/s) on B200.

One step = one pass of the whole hot path over one batch:
sidwt_analyze (fused J-level lifting, all shift branches) + sidwt_correlate_peaks
(correlation at every scale and lag, written to HBM, plus the per-scale peak
search), on inputs already resident in HBM.  Workload: BASELINE.json configs[4]
(C5: reversible integer 5/3, J=8, symmetric, 65536 x 4096 int16 I/Q rows, 12-bit
LFM template) -- the largest single-GPU configuration by samples per step, the
metric naming no config; override with --config.  The line carries `parity`: the
GPU outputs of the rows the cpu_baseline oracle processed (>= 256 seeded rows;
C4: 16 pulses x 64 templates) compared with the oracle's.  Multi-GPU (torchrun):
weak scaling, each rank its own batch of rows, no collective on the data path
(DESIGN.md section 8).

--impl reference times the CPU oracle (oracle/, fp64 C, OpenMP) on the host
cores, each step a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "complex samples/s through SIDWT lifting+correlation"
UNIT = "complex samples/s"
FP32_LANES_PER_SM = 128
N_SMS = 148


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return dict(hbm=float(d["hbm_gbs"]), sm_mhz=float(d.get("sm_max_mhz", 1965.0)),
                    bf16_sustained=float(d.get("bf16_tflops_sustained", d.get("bf16_tflops", 1400.0))), src="measured")
    except Exception:
        return dict(hbm=6650.0, sm_mhz=1965.0, bf16_sustained=1400.0, src="fallback")


def fp32_peak_tflops(sm_mhz):
    # derived from the unit counts: 148 SMs x 128 FP32 lanes x 2 flop/FFMA x clock
    return N_SMS * FP32_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12


IMAD_PER_CLK_PER_SM = 64    # measured (tools/micro/fma_rate.cu, profiles/r1d_micro_fma_imad.txt): half the FFMA rate


def int32_peak_tops(sm_mhz):
    # 148 SMs x 64 IMAD/clk x 2 int ops (multiply + add) x clock
    return N_SMS * IMAD_PER_CLK_PER_SM * 2 * sm_mhz * 1e6 / 1e12


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 10 and self.proc.poll() is None:
                time.sleep(0.05)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def algorithmic(cfg, plan):
    """Per-row algorithmic bytes / flops of each kernel."""
    J, N = cfg.levels, cfg.N
    sb = 4 if cfg.is_int else 8
    stride = plan.band_stride
    k1_bytes = N * sb + (J + 1) * 2 * stride * 4
    taps = sum(c for c in plan_counts(plan))
    # complex MAC = 8 real flops; a real template (zero imaginary taps, e.g. C2's Barker
    # code) needs 4 (real x complex), and the real-template kernel does exactly those
    k2_flops = cfg.n_templates * N * taps * (4 if plan.template_is_real() else 8)
    k2_bytes = (J + 1) * 2 * stride * 4 + cfg.n_templates * (J + 1) * N * 8
    return dict(k1_bytes=k1_bytes, k2_flops=k2_flops, k2_bytes=k2_bytes, taps=taps)


BF16_SPLIT_PRODUCTS = 3     # tensor-core bank path: fp32 = bf16 hi + lo, hi.hi + hi.lo + lo.hi


def plan_counts(plan):
    from paper_cs_0607001_b200 import _native
    J = plan.levels
    kmin = np.zeros(J + 1, np.int32)
    cnt = np.zeros(J + 1, np.int32)
    _native.sidwt_template_taps(plan.handle, None, kmin, cnt)
    return [int(c) for c in cnt]


def step_roofline(stages, ms):
    t = {}
    for name, st in stages.items():
        if "bytes_per_row" in st:                               # analyze: HBM only
            t[name] = st["ms"] * st["frac"]
        else:
            t[name] = st["ms"] * max(v["frac"] for k, v in st.items() if isinstance(v, dict) and "frac" in v)
    lb = sum(t.values())
    return {"lower_bound_ms": lb, "measured_ms": ms, "frac": lb / ms,
            "per_stage_lower_bound_ms": t,
            "note": "per stage max(algorithmic bytes / HBM peak, algorithmic work / compute peak)"}


def traffic_from_profiles(cfg_name, kernel, rows=None):
    """DRAM bytes per launch of `kernel` from profiles/ncu_traffic.json (ncu --set full:
    dram__bytes_read.sum + dram__bytes_write.sum).  A capture on a reduced batch is stored
    under "<cfg>_<R>rows" and scaled to `rows` (the kernels' traffic is linear in rows)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
    except Exception:
        return None
    if kernel in d.get(cfg_name, {}):
        return d[cfg_name][kernel]
    for key, kern in d.items():
        if key.startswith(cfg_name + "_") and key.endswith("rows") and kernel in kern and rows:
            r = int(key[len(cfg_name) + 1:-4])
            return kern[kernel] * rows / r
    return None


def parity_rows(cfg, n, total):
    """Seeded spread sample of n of the `total` row ids (always the first and the last row)."""
    if n >= total:
        return list(range(total))
    rng = np.random.default_rng(np.random.SeedSequence([W.SEED_TAG, cfg.cid, 0xB]))
    ids = set(rng.choice(np.arange(1, total - 1), size=n - 2, replace=False).tolist())
    return sorted(ids | {0, total - 1})


def oracle_sample(cfg, tm, rows_total, budget_s=15.0, min_rows=None):
    """The row sample the oracle runs on: >= 256 seeded rows (C4: 16 pulses x all 64
    templates), grown to ~budget_s of CPU work on the host cores.
    Returns (rows, ids, threads); run_oracle_sample times the oracle on them and the same
    rows are compared with the GPU's outputs."""
    import oracle as O
    threads = O.max_threads()
    if min_rows is None:
        min_rows = 16 if cfg.n_templates > 1 else 256
    min_rows = min(min_rows, rows_total)
    probe_ids = parity_rows(cfg, min(rows_total, max(2, threads)), rows_total)
    probe = np.stack([W.make_rows(cfg, r, 1, tm)[0] for r in probe_ids])
    t0 = time.perf_counter()
    O.run(cfg.family, cfg.levels, cfg.ext, cfg.N, probe, tm, corr=True, nthreads=threads)
    per_row = max(time.perf_counter() - t0, 1e-6) / probe.shape[0]
    n = int(max(min_rows, min(rows_total, budget_s / per_row)))
    ids = parity_rows(cfg, n, rows_total)
    rows = np.stack([W.make_rows(cfg, r, 1, tm)[0] for r in ids])
    return rows, ids, threads


def run_oracle_sample(cfg, tm, rows, ids, threads, ML, stride):
    import oracle as O
    t0 = time.perf_counter()
    ref = O.run(cfg.family, cfg.levels, cfg.ext, cfg.N, rows, tm, p_lo=-ML, p_hi=stride - ML, corr=True,
                nthreads=threads)
    dt = time.perf_counter() - t0
    cpu = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    rec = {"value": len(ids) * cfg.N / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
           "sample": f"{len(ids)} of {cfg.rows} rows of {cfg.name} (seeded spread sample incl. first and last; full "
                     f"N={cfg.N}, bands + all {cfg.levels + 1} scales + peaks, {cfg.n_templates} template(s)), "
                     f"fp64/int64 C oracle, {dt:.1f} s, cpu '{cpu}'"}
    return rec, ref


BAND_RTOL, CORR_TOL = 1e-5, 1e-4     # BASELINE.json north star (tests/parity.py uses the same)


def parity_record(cfg, ids, ref, g):
    """GPU outputs g (bands [n][J+1][2][stride], corr [n][n_t][J+1][N][2], lag, val) of the rows
    `ids` against the oracle's: the north-star bars (fp32: band rel L2 <= 1e-5 per (row, band),
    corr max|err| <= 1e-4 x peak per (row, template, scale), lags exact or counted near ties;
    integer family: everything bit-exact)."""
    out = {"rows": len(ids), "row_ids": f"{len(ids)} seeded ids in [0, {cfg.rows}), first {ids[:4]}, last {ids[-1]}"}
    gb, gc, gl, gv = g["bands"], g["corr"], g["lag"], g["val"]
    if cfg.is_int:
        ob = ref["bands"]
        gbb = np.stack([gb[:, :, 0, :], gb[:, :, 1, :]], axis=-1).astype(np.int64)
        bands_ok = bool(np.array_equal(gbb, ob))
        corr_ok = bool(np.array_equal(gc, ref["corr"]))
        lags_exact = int((gl == ref["lag"]).sum())
        vals_ok = bool(np.array_equal(gv, ref["val"]))
        out.update({"bit_exact_bands": bands_ok, "bit_exact_corr": corr_ok, "bit_exact_vals": vals_ok,
                    "lags_total": int(gl.size), "lags_exact": lags_exact, "near_ties": 0,
                    "pass": bands_ok and corr_ok and vals_ok and lags_exact == gl.size})
        return out
    ob = ref["bands"]
    gbc = gb[:, :, 0, :].astype(np.float64) + 1j * gb[:, :, 1, :]
    num = np.sqrt((np.abs(gbc - ob) ** 2).sum(-1))
    den = np.sqrt((np.abs(ob) ** 2).sum(-1))
    zero = den <= 1e-9 * den[:, -1:]                 # numerically-zero bands (reading R-TOL)
    rel = np.where(zero, num / np.maximum(den[:, -1:], 1e-300), num / np.maximum(den, 1e-300))
    oc = ref["corr"]
    gcc = gc[..., 0].astype(np.float64) + 1j * gc[..., 1]
    peak = np.abs(oc).max(-1)
    err = np.abs(gcc - oc).max(-1) / np.maximum(peak, 1e-300)
    ol = ref["lag"]
    same = gl == ol
    near, bad = 0, 0
    for i in map(tuple, np.argwhere(~same)):
        tol = CORR_TOL * peak[i]
        if np.abs(oc[i][gl[i]]) >= np.abs(oc[i][ol[i]]) - 2 * tol:
            near += 1
        else:
            bad += 1
    out.update({"band_rel_l2_max": float(rel.max()), "band_rtol": BAND_RTOL,
                "corr_err_over_peak_max": float(err.max()), "corr_tol": CORR_TOL,
                "lags_total": int(gl.size), "lags_exact": int(same.sum()), "near_ties": near, "lag_failures": bad,
                "pass": bool(rel.max() <= BAND_RTOL and err.max() <= CORR_TOL and bad == 0)})
    return out


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU oracle on this workload (rank 0 only)."""
    if rank != 0:
        return
    import oracle as O
    tm = W.templates(cfg)
    threads = O.max_threads()
    probe = W.make_rows(cfg, 0, min(cfg.rows, threads), tm)
    t0 = time.perf_counter()
    O.run(cfg.family, cfg.levels, cfg.ext, cfg.N, probe, tm, nthreads=threads)
    per_row = max((time.perf_counter() - t0) / probe.shape[0], 1e-6)
    total_budget = 120.0
    n = int(max(1, min(cfg.rows, total_budget / (args.steps + args.warmup) / per_row)))
    rows = W.make_rows(cfg, 0, n, tm)
    for _ in range(args.warmup):
        O.run(cfg.family, cfg.levels, cfg.ext, cfg.N, rows, tm, nthreads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.run(cfg.family, cfg.levels, cfg.ext, cfg.N, rows, tm, nthreads=threads)
    dt = (time.perf_counter() - t0) / args.steps
    v = n * cfg.N / dt
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "i64" if cfg.is_int else "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{cfg.name}: {cfg.description}", "rows_per_step": n, "N": cfg.N},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"{n} rows of {cfg.name} per step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5,
                    help="BASELINE.json config (default 5: C5, the largest single-GPU workload by samples per step)")
    ap.add_argument("--rows", type=int, default=0, help="override batch rows (default: the config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the non-headline variant timings")
    ap.add_argument("--two-call", action="store_true", help="time analyze + correlate_peaks as two plain calls")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = W.CONFIGS[args.config]

    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import torch
    import torch.distributed as dist
    from paper_cs_0607001_b200 import Plan, _native

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_cs_0607001_b200 import dist as D
    R = args.rows or cfg.rows
    tm = W.templates(cfg)
    r0, R = D.weak_rows(rank, R)                        # weak scaling: each rank its own batch
    rows_h = W.make_rows(cfg, r0, R, tm)
    plan = Plan(cfg.family, cfg.levels, cfg.N, R, cfg.ext, device=dev).load_templates(tm)
    stream = torch.cuda.current_stream(dev)
    d_rows = plan.rows_to_device(rows_h)
    bands = plan.empty_bands(R)
    corr = plan.empty_corr(R)
    lag, val = plan.empty_peaks(R)

    def step_two_call():
        plan.analyze(d_rows, R, bands, stream)
        plan.correlate_peaks(bands, R, corr, lag, val, stream=stream)

    def step_run():
        # the library's whole-path call: analysis of row chunk k+1 overlaps correlation of chunk k
        plan.run(d_rows, R, bands, corr, lag, val, stream=stream)

    step = step_two_call if args.two_call else step_run
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = plan.last_launches()

    # per-kernel timing (CUDA events on the launching stream), separate pass
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    k1_ms, k2_ms = [], []
    for _ in range(max(3, min(args.steps, 10))):
        ev[0].record(stream)
        plan.analyze(d_rows, R, bands, stream)
        ev[1].record(stream)
        plan.correlate_peaks(bands, R, corr, lag, val, stream=stream)
        ev[2].record(stream)
        torch.cuda.synchronize()
        k1_ms.append(ev[0].elapsed_time(ev[1]))
        k2_ms.append(ev[1].elapsed_time(ev[2]))
    k1_ms = float(np.median(k1_ms))
    k2_ms = float(np.median(k2_ms))

    # variants (not the headline): fused analyze->correlate->peaks without the band round
    # trip and the peaks-only mode, CUDA events on the same stream
    variants = {}

    def time_fn(fn, n):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n
    nv = max(3, min(args.steps, 20))
    if not args.no_variants:
        variants["two_call_ms"] = time_fn(step_two_call, nv)
        variants["run_ms"] = time_fn(step_run, nv)
        variants["peaks_only_ms"] = time_fn(lambda: (plan.analyze(d_rows, R, bands, stream),
                                                     plan.correlate_peaks(bands, R, None, lag, val, want_corr=False,
                                                                          stream=stream)), nv)
        if plan.fused_available():
            variants["fused_ms"] = time_fn(lambda: plan.analyze_correlate(d_rows, R, corr, lag, val, stream=stream),
                                           nv)
            variants["fused_peaks_only_ms"] = time_fn(
                lambda: plan.analyze_correlate(d_rows, R, None, lag, val, want_corr=False, stream=stream), nv)
    for k in list(variants):
        variants[k.replace("_ms", "_samples_per_s")] = world * R * cfg.N / (variants[k] * 1e-3)

    # timed region: K steps, barrier + sync on both sides, CUDA events on the launching
    # stream, max over ranks (paper_cs_0607001_b200.dist.timed_steps, also driven by the
    # world-size-2 gloo test)
    def cuda_timer():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        return (lambda: e0.record(stream)), (lambda: e1.record(stream)), (lambda: e0.elapsed_time(e1))
    with ClockSampler(local) as clk:
        ms = D.timed_steps(step, args.steps, torch.cuda.synchronize, cuda_timer, device=dev)
    value = world * R * cfg.N / (ms * 1e-3)
    # optional collective of the path: the per-row peak tables of every rank,
    # all-gathered outside the timed region
    gathered_rows = int(D.gather_weak(lag).shape[0]) if world > 1 else R

    # e2e: host rows (pinned) -> device -> path -> lag/val back to host, through the C ABI
    e2e = None
    if not args.no_e2e:
        sb = 4 if cfg.is_int else 8
        h_rows = torch.from_numpy(np.ascontiguousarray(rows_h).view(np.uint8).reshape(-1)).pin_memory()
        h_lag = torch.empty(lag.shape, dtype=torch.int32).pin_memory()
        h_val = torch.empty(val.shape, dtype=val.dtype).pin_memory()
        plan.execute_host(h_rows, R, h_lag, h_val, stream)
        torch.cuda.synchronize()
        for _ in range(2):
            plan.execute_host(h_rows, R, h_lag, h_val, stream)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            plan.execute_host(h_rows, R, h_lag, h_val, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = D.max_over_ranks(e0.elapsed_time(e1) / args.steps, device=dev)
        assert np.array_equal(h_lag.numpy(), lag.cpu().numpy()), "e2e lags differ from the device path"
        e2e = {"value": world * R * cfg.N / (ems * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": R * cfg.N * sb,
               "d2h_bytes_per_step": int(h_lag.numel() * 4 + h_val.numel() * 4),
               "ms_per_step": ems}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    pk = load_peaks()
    alg = algorithmic(cfg, plan)
    tc_path = plan.tensor_core_path()            # 0 SIMT, 1 template bank, 2 single template
    tc = tc_path > 0
    k1_gbs = R * alg["k1_bytes"] / (k1_ms * 1e-3) / 1e9
    k2_tflops = R * alg["k2_flops"] / (k2_ms * 1e-3) / 1e12
    k2_gbs = R * alg["k2_bytes"] / (k2_ms * 1e-3) / 1e9
    fp32_peak = fp32_peak_tflops(pk["sm_mhz"])
    k2_kernel = ("k_correlate", "k_correlate_tc", "k_correlate_tcs", "k_correlate_i8")[tc_path]
    if tc_path == 3:
        # int8 tensor pipe (exact digit GEMM): algorithmic integer ops (4 multiplies + 4 adds per
        # complex MAC) against the int8 dense peak = measured sustained bf16 x the nominal
        # int8 / bf16 ratio (4.5 / 2.25 PFLOP/s, B200_PROFILING.md)
        i8_peak = 2.0 * pk["bf16_sustained"]
        comp = {"achieved": k2_tflops, "peak": i8_peak, "unit": "Tops/s (int8 tensor)", "frac": k2_tflops / i8_peak,
                "flops_per_row": alg["k2_flops"],
                "note": "algorithmic int ops of the complex MACs; the kernel issues 4 real products x "
                        "(2 or 3 data digits) x (template digits) int8 MACs per complex MAC",
                "peak_source": f"{pk['src']} MEASURED_PEAKS.json bf16_tflops_sustained x 2 (int8/bf16 nominal ratio)"}
        comp_key, comp_bound = "tensor", "tensor"
    elif tc:
        # tensor pipe: the algorithmic complex MACs run as 3 bf16 products (split precision);
        # peak = measured sustained cuBLAS bf16 (the kernel runs inside a long power-capped step)
        comp = {"achieved": k2_tflops * BF16_SPLIT_PRODUCTS, "peak": pk["bf16_sustained"], "unit": "TFLOP/s",
                "frac": k2_tflops * BF16_SPLIT_PRODUCTS / pk["bf16_sustained"], "flops_per_row": alg["k2_flops"],
                "note": "bf16 tensor flops = 3 x algorithmic complex-MAC flops (hi.hi + hi.lo + lo.hi)",
                "peak_source": f"{pk['src']} MEASURED_PEAKS.json bf16_tflops_sustained"}
        comp_key, comp_bound = "tensor", "tensor"
    elif cfg.is_int:
        ipk = int32_peak_tops(pk["sm_mhz"])
        comp = {"achieved": k2_tflops, "peak": ipk, "unit": "Tops/s (int32 mul+add)", "frac": k2_tflops / ipk,
                "flops_per_row": alg["k2_flops"],
                "peak_source": "measured IMAD rate 64/clk/SM (tools/micro/fma_rate.cu) x 148 SM x 2 x %.0f MHz"
                               % pk["sm_mhz"]}
        comp_key, comp_bound = "alu", "alu"
    else:
        comp = {"achieved": k2_tflops, "peak": fp32_peak, "unit": "TFLOP/s", "frac": k2_tflops / fp32_peak,
                "flops_per_row": alg["k2_flops"],
                "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x %.0f MHz" % pk["sm_mhz"]}
        comp_key, comp_bound = "alu", "alu"
    stages = {
        "analyze": {"kernel": "k_analyze", "ms": k1_ms, "bound": "hbm", "achieved": k1_gbs, "peak": pk["hbm"],
                    "unit": "GB/s", "frac": k1_gbs / pk["hbm"], "bytes_per_row": alg["k1_bytes"]},
        "correlate_peaks": {"kernel": k2_kernel + ("" if tc_path in (2, 3) else "+k_peaks_finalize"), "ms": k2_ms,
                            comp_key: comp,
                            "hbm": {"achieved": k2_gbs, "peak": pk["hbm"], "unit": "GB/s",
                                    "frac": k2_gbs / pk["hbm"], "bytes_per_row": alg["k2_bytes"]}},
    }
    if k2_ms >= k1_ms:
        a2, h2 = stages["correlate_peaks"][comp_key], stages["correlate_peaks"]["hbm"]
        use = a2 if a2["frac"] >= h2["frac"] else h2
        roof = {"kernel": k2_kernel, "bound": comp_bound if use is a2 else "hbm", "achieved": use["achieved"],
                "peak": use["peak"], "unit": use["unit"], "frac": use["frac"],
                "traffic": traffic_from_profiles(cfg.name, k2_kernel, R),
                "peak_source": use["peak_source"] if use is a2 else f"{pk['src']} MEASURED_PEAKS.json hbm_gbs"}
    else:
        a1 = stages["analyze"]
        roof = {"kernel": "k_analyze", "bound": "hbm", "achieved": a1["achieved"], "peak": a1["peak"],
                "unit": "GB/s", "frac": a1["frac"], "traffic": traffic_from_profiles(cfg.name, "k_analyze", R),
                "peak_source": f"{pk['src']} MEASURED_PEAKS.json hbm_gbs"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "i32" if cfg.is_int else "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.description}", "rows_per_gpu": R, "N": cfg.N,
                   "levels": cfg.levels, "templates": cfg.n_templates, "parallelism": f"rows x{world} (weak)",
                   "l2": "no flush: per-step working set (bands %.2f GB + corr %.2f GB) >> 126 MB L2" % (
                       R * (cfg.levels + 1) * 2 * plan.band_stride * 4 / 1e9,
                       R * cfg.n_templates * (cfg.levels + 1) * cfg.N * 8 / 1e9)},
        "roofline": roof,
        # end-to-end roofline fraction = sum over stages of the algorithmic lower
        # bound max(t_bytes, t_compute) / the measured step
        "roofline_step": step_roofline(stages, ms),
        "stages": stages,
        "tensor_cores": tc,
        "variants": variants,
        "gpu_launches": launches_per_step * args.steps,
        "peaks_gathered_rows": gathered_rows,
        "clocks": clk.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline and world == 1:
        # the oracle on a bounded seeded sample of this rank's rows, timed on the host cores;
        # the GPU outputs of the same rows (last timed step) are compared with it element by
        # element (parity on the oracle's rows)
        o_rows, ids, threads = oracle_sample(cfg, tm, R)
        rec, ref = run_oracle_sample(cfg, tm, o_rows, ids, threads, plan.band_offset, plan.band_stride)
        line["cpu_baseline"] = rec
        it = torch.tensor(ids, dtype=torch.long, device=dev)
        g = {"bands": bands.index_select(0, it).cpu().numpy(), "corr": corr.index_select(0, it).cpu().numpy(),
             "lag": lag.index_select(0, it).cpu().numpy(), "val": val.index_select(0, it).cpu().numpy()}
        line["parity"] = parity_record(cfg, ids, ref, g)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
