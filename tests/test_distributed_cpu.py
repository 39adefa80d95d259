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
    """oracle/mp_runner.py (the bench's CPU reference arm) on 4 processes, on
    connectivity the oracle generates on 3 processes, reproduces the
    reference's golden run: raster, event totals, and the CSR equals the
    single-process oracle build."""
    from oracle import corticarc_oracle as O
    from oracle.mp_runner import build_global_csr, run_oracle_mp
    cfg, meta, arr = golden_run("tiny_gauss")
    row_off, tgt, dly, wgt, _ = build_global_csr(cfg, 3)
    net = O.build_shard(cfg.grid, cfg.kernel, cfg.genspec, cfg.seed)
    counts = np.zeros(cfg.grid.n_neurons, np.int64)
    counts[net.sources.astype(np.int64)] = np.diff(net.offsets)
    assert np.array_equal(np.diff(row_off), counts)
    assert np.array_equal(tgt, net.target_local.astype(np.int32))     # one shard: local == gid
    assert np.array_equal(dly, net.delay.astype(np.uint8))
    assert np.array_equal(wgt.view(np.uint32), net.weight.view(np.uint32))
    r = run_oracle_mp(cfg, row_off, tgt, dly, wgt, 4, cfg.n_steps, 1e9, collect_raster=True,
                      warmup=10)
    assert r["steps"] == cfg.n_steps and r["timed_steps"] == cfg.n_steps - 10
    assert r["events"] == meta["recurrent_events"] + meta["external_events"]
    assert r["timed_events"] < r["events"]
    assert np.array_equal(r["raster_gids"], arr["raster_gids"].astype(np.uint64))
    assert np.array_equal(r["raster_times"].view(np.uint64), arr["raster_times"].view(np.uint64))


# ------------------------------------------------- host logic of the exchange
def test_send_caps_and_window_layout():
    from paper_1803_08833_b200.distributed import (FLAG_SLOTS, REC_BYTES, send_caps,
                                                   window_layout)
    masks = np.array([0b011, 0b110, 0b000, 0b100, 0b010], np.int64)
    assert send_caps(masks, 3).tolist() == [1, 3, 2]
    lay = window_layout([4, 0, 7])
    base = 2 * FLAG_SLOTS * 8
    assert lay.rec_off[0] == (base, base + 4 * REC_BYTES, base + 4 * REC_BYTES)
    assert lay.rec_off[1][0] == base + 11 * REC_BYTES
    assert lay.nbytes == base + 2 * 11 * REC_BYTES
    assert lay.flag_off(1, 2) == (FLAG_SLOTS + 2) * 8
    # regions never overlap and stay inside the window, 16 B aligned
    spans = sorted((lay.rec_off[p][s], lay.rec_off[p][s] + lay.cap[s] * REC_BYTES)
                   for p in range(2) for s in range(3))
    assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:]))
    assert spans[-1][1] <= lay.nbytes and all(a % 16 == 0 for a, _ in spans)
    with pytest.raises(ValueError):
        window_layout([1] * (FLAG_SLOTS + 1))


def test_exact_caps_bound_every_step():
    """The per-pair capacity (neurons with the destination bit) bounds what a
    rank can send in one step: a neuron spikes at most once per step."""
    from paper_1803_08833_b200.engine import _spikes_per_step_bound
    cfg = tiny_config()
    assert _spikes_per_step_bound(cfg) == 1


def _agree_worker(rank, size, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_1803_08833_b200.distributed import agree_errors
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        ok = agree_errors(0, 0)
        bad = agree_errors(0x20 if rank == 1 else (0x4 if rank == 2 else 0),
                           {1: 17, 2: 12}.get(rank, 0))
        q.put((rank, ok, bad))
    finally:
        dist.destroy_process_group()


def test_agree_errors_three_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(3))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, bad in res:
        assert ok == (0, -1, -1)
        assert bad == (0x24, 12, 1)          # OR of bits, earliest step, lowest failing rank


def test_merge_pieces_reference_semantics():
    from paper_1803_08833_b200.distributed import merge_pieces
    from paper_1803_08833_b200.engine import raster_checksum
    cfg = tiny_config()
    mk = lambda r, g, t, w: dict(rank=r, g=np.array(g, np.uint64), t=np.array(t), n_spikes=len(g),
                                 rec=10 * (r + 1), ext=5, syn=100, csum=2 ** 63 + r, cons=0.5 + r,
                                 wall=w, steady=900, peak=1000)
    res = merge_pieces(cfg, [mk(1, [7, 3], [2.0, 1.0], 0.2), mk(0, [5, 9], [1.0, 0.5], 0.3)])
    assert res.raster_gids.tolist() == [9, 3, 5, 7]
    assert res.raster_times.tolist() == [0.5, 1.0, 1.0, 2.0]
    assert res.raster_checksum == raster_checksum(res.raster_gids, res.raster_times)
    assert (res.n_spikes, res.recurrent_events, res.external_events) == (4, 30, 10)
    assert res.construction_checksum == (2 ** 64 + 1) % 2 ** 64
    assert res.sim_seconds_wall == 0.3 and res.construction_seconds == 1.5
    assert res.steady_bytes_per_worker == [900, 900] and res.worker_count == 2
    off = merge_pieces(cfg, [mk(0, [1], [1.0], 0.1)], record_raster=False)
    assert len(off.raster_gids) == 0 and off.raster_checksum == 0 and off.n_spikes == 1


def test_run_b200_workers_refuses_cpu_without_hanging():
    """run_b200(config, k > 1) spawns its workers; without a CUDA device they
    fail loudly and the error reaches the caller (no CPU fallback, no hang)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_1803_08833_b200.engine import run_b200
    with pytest.raises(RuntimeError, match="CUDA device"):
        run_b200(tiny_config(), 2)
