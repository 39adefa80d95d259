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
    a = dict(gpus=1, steps=10, warmup=3, config=None, kernel=None, drive=None, seed=1,
             grid=None, scaling="strong", regime="calibrated", settle=None)
    a.update(kw)
    ns = argparse.Namespace(**a)
    bench.resolve_defaults(ns)
    return ns


def test_weak_tiling_series():
    assert [bench.weak_tiling(n) for n in (1, 2, 4, 8)] == [(1, 1), (2, 1), (2, 2), (4, 2)]
    for n in range(1, 17):
        a, b = bench.weak_tiling(n)
        assert a * b == n and a >= b


def test_workload_defaults_and_scaling(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    one = bench.workload(_args())
    assert (one.grid.nx, one.grid.ny) == (8, 8)          # N = 1: BASELINE config 1
    assert one.grid.n_neurons == 79360
    assert bench.scaling_of(_args()) == "strong"        # one GPU: nothing to scale
    eight = bench.workload(_args(gpus=8))
    assert (eight.grid.nx, eight.grid.ny) == (24, 24)   # N > 1: config 2 split over the GPUs
    assert eight.kernel.kind == "exponential"
    assert bench.scaling_of(_args(gpus=8)) == "strong"
    weak = bench.workload(_args(gpus=8, config=1, scaling="weak"))
    assert (weak.grid.nx, weak.grid.ny) == (32, 16)     # config-1 grid once per GPU
    assert bench.scaling_of(_args(gpus=8, scaling="weak")) == "weak"
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert bench.workload(_args()).grid.nx == 24
    grid = bench.workload(_args(config=4, grid="48x24", scaling="weak"))
    assert (grid.grid.nx, grid.grid.ny) == (96, 48)     # weak: --grid is one GPU's block
    monkeypatch.delenv("WORLD_SIZE")
    grid = bench.workload(_args(config=4, grid="48x24"))
    assert (grid.grid.nx, grid.grid.ny) == (48, 24)
    stress = bench.workload(_args(config=2, regime="stress"))
    assert stress.external.rate_per_synapse_hz == 200.0 and stress.genspec.j_inh_inh == -8.0


def test_reference_arm_config_is_the_gpu_arm_config(monkeypatch):
    """The CPU reference arm builds its run description without the product
    package (oracle/configs.py); it must describe the same workload."""
    from oracle.configs import baseline_config as oc
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    for idx, regime in ((1, "calibrated"), (2, "calibrated"), (2, "stress"), (0, "literal")):
        a = _args(config=idx, regime=regime)
        g = bench.workload(a)
        assert a.settle == 200 - a.warmup                 # 200 untimed steps before the window
        o = oc(idx, regime, duration_s=(a.settle + a.warmup + a.steps) / 1000.0)
        assert (o.grid.nx, o.grid.ny, o.grid.n_neurons) == (g.grid.nx, g.grid.ny, g.grid.n_neurons)
        for k in ("kind", "amplitude_A", "scale", "cutoff_p", "local_p"):
            assert getattr(o.kernel, k) == getattr(g.kernel, k), k
        for k in ("j_exc_exc", "j_exc_inh", "j_inh_exc", "j_inh_inh", "weight_sd_frac",
                  "delay_kind", "delay_min_ms", "delay_max_ms", "timestep_ms", "d_max_steps"):
            assert getattr(o.genspec, k) == getattr(g.genspec, k), k
        for k in ("tau_m", "C_m", "E", "tau_c", "g_c", "V_theta", "V_r", "tau_arp", "alpha_c"):
            assert getattr(o.exc_params, k) == getattr(g.exc_params, k), k
            assert getattr(o.inh_params, k) == getattr(g.inh_params, k), k
        assert vars(o.external) == {k: getattr(g.external, k) for k in vars(o.external)}
        assert (o.timestep_ms, o.seed, o.n_steps) == (g.timestep_ms, g.seed, g.n_steps)


def test_reference_arm_tiling():
    from oracle.mp_runner import tiles
    from paper_1803_08833_b200.partition import map_columns_to_workers
    cfg = bench.workload(_args())
    for k in range(1, 33):
        try:
            map_columns_to_workers(cfg.grid, k)
            ok = True
        except ValueError:
            ok = False
        assert tiles(cfg.grid, k) == ok, k


def _run_bench(*argv, timeout=600, env=None):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv],
                       capture_output=True, text=True, timeout=timeout, cwd=ROOT,
                       env=dict(os.environ, **(env or {})))
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, p.stdout                   # exactly one JSON line on stdout
    return json.loads(lines[0])


def test_reference_arm_runs_without_the_product_package():
    """--impl reference on a tiny workload: one JSON line from the CPU oracle
    (W + K steps, last K timed), and the product package never imported."""
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--config', '0', "
            "'--steps', '4', '--warmup', '3', '--grid', '2x1']; "
            "import bench; bench.main(); "
            "bad = [m for m in sys.modules if m.startswith('paper_1803_08833_b200')]; "
            "assert not bad, bad")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       timeout=600, cwd=ROOT, env=dict(os.environ, CC_REF_BUDGET_S="120"))
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, p.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["steps"] == 4 and line["warmup"] == 3
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_bench_line_contract():
    line = _run_bench("--steps", "20", "--warmup", "5", "--instrument-steps", "5",
                      env={"CC_CPU_BUDGET_S": "2"})
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "clocks", "e2e", "gpu_launches", "cpu_baseline"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["steps"] == 20 and line["warmup"] == 5
    assert line["settle_steps"] == 195                    # timed window: steps 200 .. 219
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
    # the end-to-end run steps on connectivity uploaded from a host store in the
    # reference's layout (import_csr): a one-time copy, reported as such
    assert e["connectivity"]["h2d_bytes_once"] > 13 * 94_000_000
    assert 0 < e["value_including_import"] < e["value"]
    c = line["cpu_baseline"]
    assert c["kind"] == "port" and c["cores"] == 1 and c["value"] > 0
    assert line["gpu_launches"] >= 3 * 20               # k_deliver, k_plan, k_stage per step
    assert line["clocks"]["sm_mhz"] > 0
    # the device-timed value replays warm graphs: not below the end-to-end rate
    assert line["value"] >= 0.9 * e["value"]


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun_bench(n, *argv, timeout=900, env=None):
    """bench.py under the driver's launch command for N > 1."""
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", str(n), "--master-addr", "127.0.0.1",
                        "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
                        "--gpus", str(n), *argv],
                       capture_output=True, text=True, timeout=timeout, cwd=ROOT,
                       env=dict(os.environ, **(env or {})))
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, p.stdout                   # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_under_torchrun_two_ranks():
    """The driver's N = 2 launch on a one-GPU box: the two ranks share cuda:0
    (host-synchronised peer exchange), rank 0 prints the line with the
    exchange figures; config 1 split into two 4x8 column blocks."""
    line = _torchrun_bench(2, "--config", "1", "--steps", "100", "--warmup", "10")
    assert line["n_gpus"] == 2 and line["steps"] == 100 and line["scaling"] == "strong"
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["config"]["neurons"] == 79360
    assert 0 <= line["exchange_fraction"] < 1
    assert line["exchange"]["per_rank_bytes_per_step_max"] > 0
    assert line["gpu_launches"] >= 3 * 100
    assert 0 < line["roofline"]["frac"] <= 1


def test_reference_arm_under_torchrun_two_ranks():
    """--impl reference under torchrun: rank 0 alone runs the CPU oracle and
    prints; the other rank exits 0 without work."""
    line = _torchrun_bench(2, "--impl", "reference", "--config", "0", "--grid", "2x1",
                           "--steps", "4", "--warmup", "3", env={"CC_REF_BUDGET_S": "120"})
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["cpu_baseline"]["value"] == line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_bench_exchange_falls_back_to_nccl(monkeypatch):
    """A peer-store exchange that fails during the warm-up (injected on every
    rank here; CC_ERR_XWAIT on a box whose GPUs cannot reach each other's
    windows) makes the multi-GPU bench fall back to the NCCL slots transport,
    and the line says which transport ran."""
    line = _run_bench("--exchange", "--steps", "100", "--warmup", "10",
                      env={"CC_TEST_P2P_FAIL": "1"})
    assert "nccl exchange" in line["config"]["parallelism"]
    assert line["value"] > 0 and 0 <= line["exchange_fraction"] < 1
    line = _run_bench("--exchange", "--steps", "100", "--warmup", "10")
    assert "p2p exchange" in line["config"]["parallelism"]
