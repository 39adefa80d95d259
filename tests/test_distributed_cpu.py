"""Multi-shard path on CPU: world_size-2/4 gloo groups run the real exchange
layer (paper_1803_08833_b200.distributed) with the CPU oracle as each shard's
compute; the merged raster must equal the single-shard run and the
reference's golden raster (partition invariance, pkg/tests/test_engine.py:184-192)."""

import os
import socket
import sys

import numpy as np
import pytest

from conftest import ROOT, golden_run, tiny_config


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, size, port, cfg, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle import corticarc_oracle as O
    from paper_1803_08833_b200.distributed import SpikeExchange, dest_masks_from_rows
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        net = O.build_shard(cfg.grid, cfg.kernel, cfg.genspec, cfg.seed, rank, size)
        sim = O.ShardSim(cfg, net, rank, size)
        has = np.zeros(cfg.grid.n_neurons, np.uint8)
        has[net.sources.astype(np.int64)] = 1
        allh = [torch.empty(cfg.grid.n_neurons, dtype=torch.uint8) for _ in range(size)]
        dist.all_gather(allh, torch.from_numpy(has))
        masks = dest_masks_from_rows([h.numpy().astype(bool) for h in allh],
                                     sim.gids.astype(np.int64))
        x = SpikeExchange(rank, size, masks, "cpu")
        rg, rt = [], []
        for t in range(cfg.n_steps):
            li = torch.from_numpy(sim.prev_idx.astype(np.int64))
            g = torch.from_numpy(sim.gids[sim.prev_idx].astype(np.int64))
            tm = torch.from_numpy(sim.prev_t.astype(np.float64))
            if t == 0:
                li, g, tm = li[:0], g[:0], tm[:0]
            in_g, in_t = x.exchange(li, g, tm)
            inc = [(in_g.numpy().astype(np.uint64), in_t.numpy())] if in_g.numel() else []
            gg, tt = sim.step(t, inc)
            if len(gg):
                rg.append(np.asarray(gg)); rt.append(np.asarray(tt))
        out_q.put((rank, np.concatenate(rg) if rg else np.empty(0, np.uint64),
                   np.concatenate(rt) if rt else np.empty(0), sim.rec, sim.ext, net.checksum,
                   x.stats["spikes_sent"]))
    finally:
        dist.destroy_process_group()


def _run_sharded(cfg, size):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, cfg, q)) for r in range(size)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(size)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    g = np.concatenate([r[1] for r in res]).astype(np.uint64)
    t = np.concatenate([r[2] for r in res])
    o = np.lexsort((g, t))
    return dict(g=g[o], t=t[o], rec=sum(r[3] for r in res), ext=sum(r[4] for r in res),
                checksum=sum(r[5] for r in res) % 2 ** 64, sent=sum(r[6] for r in res))


@pytest.mark.parametrize("size", [2, 4])
def test_sharded_oracle_matches_reference_golden(size):
    cfg, meta, arr = golden_run("tiny_gauss")
    out = _run_sharded(cfg, size)
    assert out["checksum"] == meta["construction_checksum"]
    assert np.array_equal(out["g"], arr["raster_gids"].astype(np.uint64))
    assert np.array_equal(out["t"].view(np.uint64), arr["raster_times"].view(np.uint64))
    assert out["rec"] == meta["recurrent_events"]
    assert out["ext"] == meta["external_events"]
    assert out["sent"] > 0


def test_sharded_exponential_kernel_two_ranks():
    cfg, meta, arr = golden_run("tiny_exp")
    out = _run_sharded(cfg, 2)
    assert np.array_equal(out["g"], arr["raster_gids"].astype(np.uint64))
    assert out["rec"] == meta["recurrent_events"]


def test_dest_masks_from_rows():
    from paper_1803_08833_b200.distributed import dest_masks_from_rows
    has = [np.array([1, 0, 1, 0], bool), np.array([1, 1, 0, 0], bool)]
    m = dest_masks_from_rows(has, np.array([0, 1, 2, 3]))
    assert m.tolist() == [3, 2, 1, 0]


def test_partition_tiling_matches_reference_rule():
    from paper_1803_08833_b200.partition import map_columns_to_workers
    from paper_1803_08833_b200.spec import GridSpec
    g = GridSpec(nx=24, ny=24, neurons_per_column=10)
    assert (map_columns_to_workers(g, 6).px, map_columns_to_workers(g, 6).py) == (3, 2)
    assert (map_columns_to_workers(g, 8).px, map_columns_to_workers(g, 8).py) == (4, 2)
    pm = map_columns_to_workers(GridSpec(nx=11, ny=6, neurons_per_column=4), 6)
    owned = np.concatenate([pm.owned_columns(w) for w in range(6)])
    assert sorted(owned.tolist()) == list(range(66))
    with pytest.raises(ValueError):
        map_columns_to_workers(GridSpec(nx=2, ny=2, neurons_per_column=4), 5)


def test_multiprocess_oracle_runner_event_totals():
    """oracle/mp_runner.py (the bench's CPU reference arm) on 4 processes
    reproduces the reference's event totals on shared connectivity."""
    from oracle import corticarc_oracle as O
    from oracle.mp_runner import run_oracle_mp
    cfg, meta, arr = golden_run("tiny_gauss")
    net = O.build_shard(cfg.grid, cfg.kernel, cfg.genspec, cfg.seed)
    counts = np.zeros(cfg.grid.n_neurons, np.int64)
    counts[net.sources.astype(np.int64)] = np.diff(net.offsets)
    row_off = np.concatenate([[0], np.cumsum(counts)])
    r = run_oracle_mp(cfg, row_off, net.target_local.astype(np.int64), net.delay, net.weight,
                      4, cfg.n_steps, 1e9)
    assert r["steps"] == cfg.n_steps
    assert r["events"] == meta["recurrent_events"] + meta["external_events"]
