"""Full-length parity at the bench configuration, on the driver's clock:
BASELINE config 1 (8x8 x 1240 neurons, 95 M synapses) over 1 s of simulated
time, calibrated operating point.  The CUDA engine - on one GPU, and as 4
column-block workers exchanging spikes over the peer windows - against the
CPU oracle on 16 processes (oracle/mp_runner.py, the reference loop restated
and pinned to the reference's own fixtures) on the same connectivity: every
spike's gid and float64 time and both event counts identical (BASELINE
north star: "spike rasters match the CPU reference exactly over 1 s")."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def config1_run():
    from paper_1803_08833_b200.engine import run_b200
    from paper_1803_08833_b200.network import build_b200
    from paper_1803_08833_b200.presets import baseline_config
    from oracle.mp_runner import run_oracle_mp, tiles
    cfg = baseline_config(1, "calibrated")                 # 1 s
    net = build_b200(cfg)
    gpu = run_b200(cfg, 1, net=net)
    row_off, tgt, w, d = net.host_csr()                    # one shard: local target == gid
    del net
    k = next(k for k in range(min(len(os.sched_getaffinity(0)), 16), 0, -1) if tiles(cfg.grid, k))
    ref = run_oracle_mp(cfg, row_off, tgt.astype(np.int32), d, w, k, cfg.n_steps, 1e9,
                        collect_raster=True)
    return cfg, gpu, ref


def _same(res, ref):
    assert res.n_spikes == len(ref["raster_gids"]) > 100_000
    assert np.array_equal(res.raster_gids, ref["raster_gids"].astype(np.uint64))
    assert np.array_equal(res.raster_times.view(np.uint64), ref["raster_times"].view(np.uint64))
    assert res.recurrent_events == ref["recurrent_events"]
    assert res.external_events == ref["external_events"]


def test_config1_one_second_single_gpu(cuda, config1_run):
    cfg, gpu, ref = config1_run
    assert ref["steps"] == cfg.n_steps == 1000
    _same(gpu, ref)


def test_config1_one_second_four_workers(cuda, config1_run):
    """run_b200(config, 4): four processes, column blocks of 4x4 columns, the
    peer exchange every step (host-synchronised: one GPU)."""
    from paper_1803_08833_b200.engine import run_b200
    cfg, gpu, ref = config1_run
    four = run_b200(cfg, 4)
    assert four.worker_count == 4
    assert four.construction_checksum == gpu.construction_checksum
    _same(four, ref)
