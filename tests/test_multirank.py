"""World-size-2 gloo test of the multi-rank host logic (CPU): row partition,
per-rank processing, gather of the peak tables, and the max-over-ranks timing
reduction.  Each rank runs the CPU oracle on its row block as the stand-in for
its GPU; the result must equal a single-process run over all rows."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, per_rank, out_q):
    import time

    import torch
    import torch.distributed as dist

    import oracle as O
    import workloads as W
    from paper_cs_0607001_b200 import dist as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = W.CONFIGS[2]
    tm = W.templates(cfg)

    # --- bench.py's weak-scaling flow: rank k owns rows [k R, (k+1) R), times K steps with
    # D.timed_steps (barrier + sync on both sides, max over ranks), peak tables gathered with
    # D.gather_weak.  The per-rank step is the CPU oracle on the rank's rows (the stand-in for
    # the GPU path, which needs a device).
    r0, R = D.weak_rows(rank, per_rank)
    rows = W.make_rows(cfg, r0, R, tm)
    out = {}

    def step():
        out["r"] = O.run(cfg.family, cfg.levels, cfg.ext, cfg.N, rows, tm, corr=False, nthreads=2)
        if rank == 1:
            time.sleep(0.05)                     # the slower rank must set the max

    def cpu_timer():
        t = {}
        return (lambda: t.__setitem__(0, time.perf_counter())), (lambda: t.__setitem__(1, time.perf_counter())), \
            (lambda: (t[1] - t[0]) * 1e3)
    ms = D.timed_steps(step, 2, lambda: None, cpu_timer)
    lag_w = D.gather_weak(torch.from_numpy(out["r"]["lag"]))

    # --- strong partition (ragged) + gather_rows
    start, n = D.strong_rows(rank, world, total)
    srows = W.make_rows(cfg, start, n, tm)
    r = O.run(cfg.family, cfg.levels, cfg.ext, cfg.N, srows, tm, corr=False, nthreads=2)
    lag = torch.from_numpy(r["lag"])
    val = torch.from_numpy(r["val"].view(np.float64).reshape(n, 1, cfg.levels + 1, 2))
    g_lag = D.gather_rows(lag, total)
    g_val = D.gather_rows(val, total)
    t = D.max_over_ranks(10.0 + rank)
    if rank == 0:
        out_q.put((g_lag.numpy(), g_val.numpy(), t, lag_w.numpy(), ms))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharding():
    import multiprocessing as mp

    import oracle as O
    import workloads as W

    total = 7                       # ragged strong partition: 4 + 3 rows
    per_rank = 3                    # weak scaling: 3 rows per rank
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, per_rank, q)) for r in range(2)]
    for p in procs:
        p.start()
    g_lag, g_val, tmax, lag_w, ms = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = W.CONFIGS[2]
    tm = W.templates(cfg)
    rows = W.make_rows(cfg, 0, total, tm)
    ref = O.run(cfg.family, cfg.levels, cfg.ext, cfg.N, rows, tm, corr=False, nthreads=2)
    assert np.array_equal(g_lag, ref["lag"])
    assert np.array_equal(g_val.reshape(-1), ref["val"].view(np.float64).reshape(-1))
    assert tmax == 11.0
    # weak scaling: the gathered peak tables are those of global rows 0 .. 2 R - 1
    ref_w = O.run(cfg.family, cfg.levels, cfg.ext, cfg.N, W.make_rows(cfg, 0, 2 * per_rank, tm), tm, corr=False,
                  nthreads=2)
    assert np.array_equal(lag_w, ref_w["lag"])
    assert ms >= 25.0               # max over ranks: rank 1 sleeps 50 ms per 2 steps


def test_partitions_cover_rows_once():
    from paper_cs_0607001_b200 import dist as D
    for world in (1, 2, 3, 8):
        for total in (1, 7, 4096, 65536):
            spans = [D.strong_rows(r, world, total) for r in range(world)]
            assert spans[0][0] == 0
            for (s0, n0), (s1, _) in zip(spans, spans[1:]):
                assert s0 + n0 == s1
            assert sum(n for _, n in spans) == total
            assert max(n for _, n in spans) - min(n for _, n in spans) <= 1
