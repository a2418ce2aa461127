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


def _worker(rank, world, port, total, out_q):
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
    start, n = D.strong_rows(rank, world, total)
    rows = W.make_rows(cfg, start, n, tm)
    r = O.run(cfg.family, cfg.levels, cfg.ext, cfg.N, rows, tm, corr=False, nthreads=2)
    lag = torch.from_numpy(r["lag"])
    val = torch.from_numpy(r["val"].view(np.float64).reshape(n, 1, cfg.levels + 1, 2))
    g_lag = D.gather_rows(lag, total)
    g_val = D.gather_rows(val, total)
    t = D.max_over_ranks(10.0 + rank)
    # weak-scaling row ownership is disjoint and contiguous
    w0 = D.weak_rows(rank, 16)
    if rank == 0:
        out_q.put((g_lag.numpy(), g_val.numpy(), t, w0))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharding():
    import multiprocessing as mp

    import oracle as O
    import workloads as W

    total = 7                       # ragged: 4 + 3 rows
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    g_lag, g_val, tmax, w0 = q.get(timeout=300)
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
    assert w0 == (0, 16)


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
