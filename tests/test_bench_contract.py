"""bench.py's host logic (weak tiling, workload, the reference arm's fallback) on CPU,
and the JSON line of one short bench run on the GPU (the keys the driver reads)."""

import argparse
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _args(**kw):
    a = dict(gpus=1, steps=10, warmup=3, config=1, kernel=None, drive=None, seed=1,
             grid=None, scaling="weak")
    a.update(kw)
    return argparse.Namespace(**a)


def test_weak_tiling_series():
    assert [bench.weak_tiling(n) for n in (1, 2, 4, 8)] == [(1, 1), (2, 1), (2, 2), (4, 2)]
    for n in range(1, 17):
        a, b = bench.weak_tiling(n)
        assert a * b == n and a >= b


def test_workload_weak_and_strong(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    one = bench.workload(_args())
    assert (one.grid.nx, one.grid.ny) == (8, 8)
    assert one.grid.n_neurons == 79360
    assert bench.scaling_of(_args()) == "strong"        # one GPU: nothing to scale
    eight = bench.workload(_args(gpus=8))
    assert (eight.grid.nx, eight.grid.ny) == (32, 16)   # config-1 grid once per GPU
    assert bench.scaling_of(_args(gpus=8)) == "weak"
    strong = bench.workload(_args(gpus=8, scaling="strong"))
    assert (strong.grid.nx, strong.grid.ny) == (8, 8)
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert (bench.workload(_args()).grid.nx, bench.workload(_args()).grid.ny) == (16, 16)
    grid = bench.workload(_args(config=4, grid="48x24"))
    assert (grid.grid.nx, grid.grid.ny) == (96, 48)     # --grid is one GPU's block
    monkeypatch.delenv("WORLD_SIZE")
    grid = bench.workload(_args(config=4, grid="48x24"))
    assert (grid.grid.nx, grid.grid.ny) == (48, 24)


def test_reference_workers_tile_the_grid():
    from paper_1803_08833_b200.partition import map_columns_to_workers
    cfg = bench.workload(_args())
    k = bench.reference_workers(cfg)
    assert 1 <= k <= min(bench.host_threads(), cfg.grid.n_columns)
    map_columns_to_workers(cfg.grid, k)                 # raises if k does not tile


def _run_bench(*argv, timeout=600, env=None):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv],
                       capture_output=True, text=True, timeout=timeout, cwd=ROOT,
                       env=dict(os.environ, **(env or {})))
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, p.stdout                   # exactly one JSON line on stdout
    return json.loads(lines[0])


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="CPU-only fallback line")
def test_reference_arm_without_gpu_prints_unavailable():
    line = _run_bench("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert line["impl"] == "reference" and "unavailable" in line


@pytest.mark.gpu
def test_bench_line_contract():
    line = _run_bench("--steps", "20", "--warmup", "5", "--instrument-steps", "5",
                      env={"CC_CPU_BUDGET_S": "2"})
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "clocks", "e2e", "gpu_launches", "cpu_baseline"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["steps"] == 20 and line["warmup"] == 5
    assert line["value"] > 0 and line["ms_per_step"] > 0 and line["higher_is_better"]
    assert line["config"]["workload"].startswith("BASELINE config 1")
    assert line["config"]["neurons"] == 79360
    r = line["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert 0 < r["frac"] <= 1 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    e = line["e2e"]
    assert e["value"] > 0 and e["unit"] == line["unit"]
    # the inputs are the config and seed (network and drive are generated on the
    # device); the raster and the per-chunk counters come back every step
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] > 0
    c = line["cpu_baseline"]
    assert c["kind"] == "port" and c["cores"] == 1 and c["value"] > 0
    assert line["gpu_launches"] >= 3 * 20               # k_deliver, k_plan, k_stage per step
    assert line["clocks"]["sm_mhz"] > 0
