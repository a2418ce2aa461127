"""Host-side pieces of bench.py (no GPU): the reference arm's JSON line (the oracle timed on
the host cores, same metric / unit / config as the GPU arm), the step roofline arithmetic,
and the scaling of reduced-batch ncu traffic to the bench batch."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["unit"] == bench.UNIT
    assert line["higher_is_better"] is True and line["value"] > 0 and line["steps"] == 1
    assert line["config"]["workload"].startswith("C1")
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["unit"] == line["unit"]


def test_step_roofline():
    stages = {"analyze": {"ms": 0.2, "frac": 0.8, "bytes_per_row": 1},
              "correlate_peaks": {"ms": 0.5, "alu": {"frac": 0.3}, "hbm": {"frac": 0.5}}}
    r = bench.step_roofline(stages, 0.7)
    assert abs(r["lower_bound_ms"] - (0.16 + 0.25)) < 1e-12
    assert abs(r["frac"] - 0.41 / 0.7) < 1e-12


def test_traffic_scaling(tmp_path, monkeypatch):
    prof = tmp_path / "profiles"
    prof.mkdir()
    (prof / "ncu_traffic.json").write_text(json.dumps({"C2": {"k": 10.0}, "C3_100rows": {"k": 50.0}}))
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    assert bench.traffic_from_profiles("C2", "k", 7) == 10.0                 # exact batch
    assert bench.traffic_from_profiles("C3", "k", 400) == 200.0              # scaled 100 -> 400 rows
    assert bench.traffic_from_profiles("C4", "k", 1) is None


def _gpu_like(ref, J, is_int):
    """The oracle's outputs cast to what the GPU returns (fp32 split planes / int32)."""
    import numpy as np
    b = ref["bands"]
    if is_int:
        bands = np.stack([b[..., 0], b[..., 1]], axis=2).astype(np.int32)
        return {"bands": bands, "corr": ref["corr"].copy(), "lag": ref["lag"].copy(), "val": ref["val"].copy()}
    bands = np.stack([b.real, b.imag], axis=2).astype(np.float32)
    corr = np.stack([ref["corr"].real, ref["corr"].imag], axis=-1).astype(np.float32)
    val = np.take_along_axis(corr, ref["lag"][..., None, None].astype(np.int64), -2)[..., 0, :]
    return {"bands": bands, "corr": corr, "lag": ref["lag"].copy(), "val": val}


def test_parity_record_on_the_oracle_sample():
    """bench.py's `parity` object: the rows of the oracle sample, the tolerances of the north
    star; a perturbed band / corr / lag fails it (float and integer families)."""
    import numpy as np
    import workloads as W
    for cid in (2, 5):
        cfg = W.CONFIGS[cid]
        tm = W.templates(cfg)
        rows, ids, threads = bench.oracle_sample(cfg, tm, 40, budget_s=0.0, min_rows=6)
        assert len(ids) == 6 and ids[0] == 0 and ids[-1] == 39 and ids == sorted(set(ids))
        assert np.array_equal(rows[1], W.make_rows(cfg, ids[1], 1, tm)[0])
        ML, stride = 256, 4096 + 768
        rec, ref = bench.run_oracle_sample(cfg, tm, rows, ids, 2, ML, stride)
        assert rec["kind"] == "oracle" and rec["value"] > 0 and "6 of" in rec["sample"]
        g = _gpu_like(ref, cfg.levels, cfg.is_int)
        p = bench.parity_record(cfg, ids, ref, g)
        assert p["pass"] and p["rows"] == 6 and p["lags_exact"] == p["lags_total"] == 6 * (cfg.levels + 1), p
        bad = {k: v.copy() for k, v in g.items()}
        bad["bands"][3, 1, 0, 300] += 1 if cfg.is_int else 1e-2
        assert not bench.parity_record(cfg, ids, ref, bad)["pass"]
        bad = {k: v.copy() for k, v in g.items()}
        bad["corr"][2, 0, 0, 7, 0] += 1 if cfg.is_int else 1e3
        assert not bench.parity_record(cfg, ids, ref, bad)["pass"]
        bad = {k: v.copy() for k, v in g.items()}
        bad["lag"][0, 0, 0] = (bad["lag"][0, 0, 0] + 1000) % cfg.N
        assert not bench.parity_record(cfg, ids, ref, bad)["pass"]
