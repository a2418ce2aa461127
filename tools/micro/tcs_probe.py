"""Time the single-template tensor-core correlation on C3-shaped rows, with and without the corr
write (the epilogue's store cost), for kernel experiments.  usage: python tools/micro/tcs_probe.py [rows]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import workloads as W
from paper_cs_0607001_b200 import Plan

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 2960
cfg = W.CONFIGS[3]
tm = W.templates(cfg)
y = W.make_rows(cfg, 0, min(rows, 64), tm)
y = np.concatenate([y] * (rows // y.shape[0] + 1))[:rows]
plan = Plan(cfg.family, cfg.levels, cfg.N, rows, cfg.ext, device="cuda:0").load_templates(tm)
d = plan.rows_to_device(y)
bands = plan.analyze(d, rows)
corr = plan.empty_corr(rows)
for want in (True, False):
    for _ in range(2): plan.correlate_peaks(bands, rows, corr=corr, want_corr=want)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): plan.correlate_peaks(bands, rows, corr=corr, want_corr=want)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"want_corr={want}: {ms:.3f} ms for {rows} rows -> C3 16384 rows ~ {ms * 16384 / rows:.2f} ms")
