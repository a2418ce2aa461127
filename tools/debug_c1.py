import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import workloads as W, oracle as O
from paper_cs_0607001_b200 import Plan
from parity import run_gpu, oracle_for
for cid in (1, 2):
    cfg = W.CONFIGS[cid]; tm = W.templates(cfg); rows = W.make_rows(cfg, 0, 1, tm)
    plan = Plan(cfg.family, cfg.levels, cfg.N, 1, cfg.ext).load_templates(tm)
    g = run_gpu(plan, rows); r = oracle_for(plan, rows, tm)
    gc = g['corr'][..., 0] + 1j * g['corr'][..., 1]
    for s in range(cfg.levels + 1):
        d = np.abs(gc[0, 0, s] - r['corr'][0, 0, s]); pk = np.abs(r['corr'][0, 0, s]).max()
        bad = np.nonzero(d > 1e-4 * pk)[0]
        print(cfg.name, 's', s, 'err/peak %.2e' % (d.max() / pk), 'nbad', len(bad), bad[:8], bad[-4:] if len(bad) else '')
