"""Multi-process CPU oracle (test / baseline infrastructure only).

Runs the numpy oracle (corticarc_oracle.ShardSim) in k worker processes, one
shard each, tiled like the reference's run_multiprocess (engine.py:494-528)
and exchanging spikes over a gloo process group with the same
counters-then-payload protocol (paper_1803_08833_b200.distributed.SpikeExchange).
Connectivity is the shared CSR (e.g. built by the GPU generator and copied to
host), cut into per-shard incoming stores here, so only the simulation loop
is timed - the reference's normalized-cost convention (metrics.py:114-123).
"""

from __future__ import annotations

import os
import socket
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def shard_net(cfg, row_off, tgt_global, delay, weight, rank, size):
    """Incoming store of one shard from a global CSR keyed by source gid."""
    from oracle import corticarc_oracle as O
    from paper_1803_08833_b200.partition import map_columns_to_workers
    grid = cfg.grid
    n = grid.neurons_per_column
    pm = map_columns_to_workers(grid, size)
    cols = pm.owned_columns(rank)
    col_rank = np.full(grid.n_columns, -1, np.int64)
    col_rank[cols] = np.arange(len(cols))
    # chunked over source rows (the global arrays are memory-mapped; the
    # temporaries of one chunk stay small even for G-synapse stores)
    parts = []
    n_rows = len(row_off) - 1
    r0 = 0
    while r0 < n_rows:
        r1 = min(n_rows, max(r0 + 1, int(np.searchsorted(row_off, row_off[r0] + 32_000_000))))
        a, b = int(row_off[r0]), int(row_off[r1])
        tg = np.asarray(tgt_global[a:b])
        keep = col_rank[tg // n] >= 0
        srcc = np.repeat(np.arange(r0, r1, dtype=np.int64), np.diff(row_off[r0:r1 + 1]))
        parts.append((srcc[keep], tg[keep], np.asarray(delay[a:b])[keep],
                      np.asarray(weight[a:b])[keep]))
        r0 = r1
    src = np.concatenate([q[0] for q in parts]) if parts else np.empty(0, np.int64)
    tg = np.concatenate([q[1] for q in parts]) if parts else np.empty(0, np.int64)
    d = np.concatenate([q[2] for q in parts]) if parts else np.empty(0, np.uint8)
    w = np.concatenate([q[3] for q in parts]) if parts else np.empty(0, np.float32)
    del parts
    sources, starts = np.unique(src, return_index=True)
    offsets = np.concatenate([starts, [len(src)]]).astype(np.int64)
    tl = (col_rank[tg // n] * n + tg % n).astype(np.uint32)
    return O.ShardNet(sources.astype(np.uint64), offsets, tl, d.astype(np.uint16),
                      w.astype(np.float32), 0, 0)


def _worker(rank, size, port, cfg, paths, steps, budget_s, q, raster_path=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), OMP_NUM_THREADS="1")
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle import corticarc_oracle as O
    from paper_1803_08833_b200.distributed import SpikeExchange, dest_masks_from_rows
    torch.set_num_threads(1)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        row_off, tgt, dly, wgt = (np.load(p, mmap_mode="r") for p in paths)
        net = shard_net(cfg, np.asarray(row_off), tgt, dly, wgt, rank, size)
        sim = O.ShardSim(cfg, net, rank, size)
        has = np.zeros(cfg.grid.n_neurons, np.uint8)
        has[net.sources.astype(np.int64)] = 1
        allh = [torch.empty(cfg.grid.n_neurons, dtype=torch.uint8) for _ in range(size)]
        dist.all_gather(allh, torch.from_numpy(has))
        masks = dest_masks_from_rows([h.numpy().astype(bool) for h in allh],
                                     sim.gids.astype(np.int64))
        x = SpikeExchange(rank, size, masks, "cpu")
        dist.barrier()
        t0 = time.perf_counter()
        done = 0
        rg, rt = [], []
        for t in range(steps):
            li = torch.from_numpy(sim.prev_idx.astype(np.int64))
            g = torch.from_numpy(sim.gids[sim.prev_idx].astype(np.int64))
            tm = torch.from_numpy(sim.prev_t.astype(np.float64))
            in_g, in_t = x.exchange(li, g, tm)
            inc = [(in_g.numpy().astype(np.uint64), in_t.numpy())] if in_g.numel() else []
            g_out, t_out = sim.step(t, inc)
            if raster_path is not None:
                rg.append(np.asarray(g_out, np.uint64))
                rt.append(np.asarray(t_out, np.float64))
            done += 1
            # all ranks agree on stopping (bounded sample)
            flag = torch.tensor([1 if time.perf_counter() - t0 > budget_s else 0])
            dist.all_reduce(flag, op=dist.ReduceOp.MAX)
            if flag.item():
                break
        wall = time.perf_counter() - t0
        if raster_path is not None:
            np.save(f"{raster_path}_{rank}_g.npy",
                    np.concatenate(rg) if rg else np.empty(0, np.uint64))
            np.save(f"{raster_path}_{rank}_t.npy", np.concatenate(rt) if rt else np.empty(0))
        q.put((rank, done, wall, sim.rec, sim.ext, x.stats["seconds"]))
    finally:
        dist.destroy_process_group()


def run_oracle_mp(cfg, row_off, tgt_global, delay, weight, workers: int, steps: int,
                  budget_s: float, collect_raster: bool = False):
    """Time the oracle loop on `workers` processes; returns a dict with
    events/s, steps done, wall (max over ranks) and exchange seconds (and with
    collect_raster the merged raster sorted by (time, gid), and the recurrent /
    external event counts)."""
    import multiprocessing as mp
    tmp = tempfile.mkdtemp(prefix="cc_oracle_")
    paths = []
    for name, arr in (("row_off", row_off), ("tgt", tgt_global), ("dly", delay), ("wgt", weight)):
        p = os.path.join(tmp, name + ".npy")
        np.save(p, arr)
        paths.append(p)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    rpath = os.path.join(tmp, "raster") if collect_raster else None
    procs = [ctx.Process(target=_worker,
                         args=(r, workers, port, cfg, paths, steps, budget_s, q, rpath))
             for r in range(workers)]
    for p in procs:
        p.start()
    res = [q.get(timeout=3600) for _ in range(workers)]
    for p in procs:
        p.join(timeout=120)
    out = {}
    if collect_raster:
        gs, ts = [], []
        for r in range(workers):
            for kind, lst in (("g", gs), ("t", ts)):
                f = f"{rpath}_{r}_{kind}.npy"
                lst.append(np.load(f))
                os.unlink(f)
        g, t = np.concatenate(gs), np.concatenate(ts)
        o = np.lexsort((g, t))
        out = dict(raster_gids=g[o], raster_times=t[o],
                   recurrent_events=int(sum(r[3] for r in res)),
                   external_events=int(sum(r[4] for r in res)))
    for p in paths:
        os.unlink(p)
    os.rmdir(tmp)
    steps_done = min(r[1] for r in res)
    wall = max(r[2] for r in res)
    ev = sum(r[3] + r[4] for r in res)
    return dict(value=ev / wall if wall > 0 else 0.0, steps=steps_done, wall_s=wall,
                events=int(ev), exchange_s=max(r[5] for r in res), workers=workers, **out)
