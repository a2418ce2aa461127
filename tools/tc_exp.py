"""Time the correlation variants on a C4 batch: corr+peaks, corr only, peaks only.
usage: python tools/tc_exp.py [rows]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_cs_0607001_b200 import Plan

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 512
cfg = W.CONFIGS[4]
tm = W.templates(cfg)
y = W.make_rows(cfg, 0, rows, tm)
plan = Plan(cfg.family, cfg.levels, cfg.N, rows, cfg.ext).load_templates(tm)
print("tensor cores:", plan.uses_tensor_cores())
d = plan.rows_to_device(y)
bands = plan.analyze(d, rows)
corr = plan.empty_corr(rows)
lag, val = plan.empty_peaks(rows)
def timeit(fn, n=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
out_gb = rows * 64 * (cfg.levels + 1) * cfg.N * 8 / 1e9
for name, fn in [("corr+peaks", lambda: plan.correlate_peaks(bands, rows, corr, lag, val)),
                 ("corr only", lambda: plan.correlate(bands, rows, corr)),
                 ("peaks only", lambda: plan.correlate_peaks(bands, rows, None, lag, val, want_corr=False))]:
    ms = timeit(fn)
    print(f"{name:12s} {ms:8.3f} ms  -> full C4 {ms * 2048 / rows:7.2f} ms   write {out_gb / ms * 1e3:7.1f} GB/s")
