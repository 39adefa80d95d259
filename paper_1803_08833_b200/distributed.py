"""Multi-GPU runs: one process per GPU, columns sharded by contiguous blocks.

Replaces the reference's transport layer for the hot loop:

    construct_network exchange (network.py:229-310)  -> each rank regenerates its
                                                        own incoming synapses
                                                        (network.build_b200); only
                                                        row-presence bitmaps are
                                                        all-gathered once to build
                                                        the destination masks
    deliver_spikes two-phase AER (network.py:325-379) -> SpikeExchange.exchange:
                                                        counts all-to-all, then
                                                        payload all-to-all-v over
                                                        NCCL (gloo on CPU tests)

The exchange logic is plain torch so the same code runs on CUDA tensors with
NCCL and on CPU tensors with gloo (tests/test_distributed_cpu.py drives it
with the CPU oracle as the per-shard compute).
"""

from __future__ import annotations

import ctypes as C
import json
import os
import time
from typing import List, Optional, Tuple

import numpy as np

__all__ = ["SpikeExchange", "dest_masks_from_rows", "DistributedSimulator",
           "run_multi_gpu", "bench_distributed", "ProtocolViolation", "run_local_shards"]


class ProtocolViolation(RuntimeError):
    """Payload does not match its announced counter (network.py:66-67)."""


def dest_masks_from_rows(has_row_by_rank: List[np.ndarray], owned_gids: np.ndarray) -> np.ndarray:
    """Bit d of mask[i] is set iff rank d stores >= 1 synapse of source
    owned_gids[i] (the reference's source_masks, network.py:229-230)."""
    mask = np.zeros(len(owned_gids), dtype=np.int64)
    for d, has in enumerate(has_row_by_rank):
        mask |= (np.asarray(has)[owned_gids].astype(np.int64) << d)
    return mask


class SpikeExchange:
    """Per-step AER exchange between shards over a torch.distributed group.

    Payload per spike: (gid, float64 time bits) as two int64 words.  Counts go
    first (one all_to_all of W integers), then the payload as an
    all_to_all_single with per-pair split sizes - the reference's
    counters-then-payloads protocol.
    """

    def __init__(self, rank: int, size: int, dest_mask_local, device, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.size, self.group = rank, size, group
        self.device = torch.device(device)
        self.mask = torch.as_tensor(np.asarray(dest_mask_local, dtype=np.int64), device=self.device)
        self.bits = torch.arange(size, device=self.device, dtype=torch.int64)
        self.stats = dict(steps=0, spikes_sent=0, payload_bytes=0, seconds=0.0)

    def exchange(self, local_idx, gids, times) -> Tuple[object, object]:
        """local_idx/gids/times: this rank's spikes of one step (any order).
        Returns (gids, times) received from every source rank, concatenated
        in source-rank order."""
        torch, dist = self.torch, self.dist
        t0 = time.perf_counter()
        n = int(local_idx.numel())
        if n:
            m = self.mask[local_idx.long()]                            # [n]
            sel = ((m[:, None] >> self.bits[None, :]) & 1).bool()      # [n, W]
            dest = sel.nonzero(as_tuple=False)                         # (spike, dest) pairs, dest-major after sort
            order = torch.argsort(dest[:, 1], stable=True)
            dest = dest[order]
            send_counts = torch.bincount(dest[:, 1], minlength=self.size)
            payload = torch.stack([gids.long()[dest[:, 0]],
                                   times.double()[dest[:, 0]].view(torch.int64)], dim=1)
        else:
            send_counts = torch.zeros(self.size, dtype=torch.int64, device=self.device)
            payload = torch.zeros((0, 2), dtype=torch.int64, device=self.device)
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        sc = send_counts.tolist()
        rc = recv_counts.tolist()
        recv = torch.empty((sum(rc), 2), dtype=torch.int64, device=self.device)
        dist.all_to_all_single(recv, payload.contiguous(), output_split_sizes=rc,
                               input_split_sizes=sc, group=self.group)
        if recv.shape[0] != sum(rc):
            raise ProtocolViolation(f"rank {self.rank}: announced {sum(rc)} spikes, got {recv.shape[0]}")
        self.stats["steps"] += 1
        self.stats["spikes_sent"] += sum(sc)
        self.stats["payload_bytes"] += 16 * sum(sc)
        self.stats["seconds"] += time.perf_counter() - t0
        return recv[:, 0], recv[:, 1].view(torch.float64)


def _has_row_all_ranks(net, size, group=None):
    import torch
    import torch.distributed as dist
    ln = net.row_off[1:] - net.row_off[:-1]
    has = (ln > 0).to(torch.uint8)
    gathered = [torch.empty_like(has) for _ in range(size)]
    dist.all_gather(gathered, has, group=group)
    return [g.cpu().numpy().astype(bool) for g in gathered]


class DistributedSimulator:
    """One rank's shard: Simulator in exchange mode + SpikeExchange per step."""

    def __init__(self, cfg, rank: int, size: int, device=None, group=None, **sim_kw):
        import torch
        from .engine import Simulator
        from .network import build_b200
        self.torch = torch
        self.rank, self.size = rank, size
        self.dev = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        self.net = build_b200(cfg, rank=rank, size=size, device=self.dev)
        self.sim = Simulator(cfg, self.net, direct_log=False, use_graphs=False, device=self.dev,
                             **sim_kw)
        has = _has_row_all_ranks(self.net, size, group)
        masks = dest_masks_from_rows(has, self.sim.gids)
        self.xchg = SpikeExchange(rank, size, masks, self.dev, group)
        n = cfg.grid.neurons_per_column
        self.local_of_col = np.full(cfg.grid.n_columns, -1, np.int64)
        self.local_of_col[self.net.owned_columns] = np.arange(len(self.net.owned_columns))
        self.lut = torch.as_tensor(self.local_of_col, device=self.dev)
        self.n_col = n
        self.t = 0
        self.timers = dict(exchange=0.0, kernels=0.0)
        self.n_in = torch.zeros(1, dtype=torch.int32, device=self.dev)

    def step(self) -> None:
        torch = self.torch
        L, sim = self.sim.L, self.sim
        from . import _lib
        s = torch.cuda.current_stream(self.dev).cuda_stream
        t0 = time.perf_counter()
        sim._launch_step(s)                      # deliver + plan + stage + update
        torch.cuda.synchronize(self.dev)
        t1 = time.perf_counter()
        ctl = sim.buf["ctl"]
        out_n = int(sim.ctl().out_n)
        g = sim.buf["out_gid"][:out_n].long() & 0xFFFFFFFF
        tm = sim.buf["out_t"][:out_n]
        li = self.lut[g // self.n_col] * self.n_col + g % self.n_col
        rg, rt = self.xchg.exchange(li, g, tm)
        k = int(rg.numel())
        in_g = rg.to(torch.int32).contiguous()
        in_t = rt.contiguous()
        self.n_in.fill_(k)
        _lib.check(L.cc_ingest(C.byref(sim.shard), in_g.data_ptr() if k else 0,
                               in_t.data_ptr() if k else 0, self.n_in.data_ptr(), s), "cc_ingest")
        # reset the out-list fill (ctl.out_n, byte offset of field)
        off = _lib.Ctl.out_n.offset
        ctl.view(torch.uint8)[off:off + 4].zero_()
        torch.cuda.synchronize(self.dev)
        self.timers["kernels"] += t1 - t0
        self.timers["exchange"] += time.perf_counter() - t1
        self.t += 1

    def advance(self, n_steps: int, check_every: int = 100) -> None:
        for i in range(n_steps):
            self.step()
            if (i + 1) % check_every == 0 or i == n_steps - 1:
                self.sim.check()


def run_local_shards(config, size: int, device=None):
    """All `size` shards of a multi-GPU run, stepped in turn on ONE device.

    Same shard code as run_multi_gpu - per-rank generator (build_b200 rank /
    size), exchange-mode neuron step (out-list), cc_ingest - with the AER
    exchange done in-process: destination d receives, in source-rank order,
    the spikes whose source has a row on d (SpikeExchange semantics).  No
    kernel waits on another shard's kernel.  Used to test partition invariance
    of the CUDA path on a single B200 (tests/test_gpu_parity.py)."""
    import torch
    from . import _lib
    from .engine import RunResult, Simulator, raster_checksum
    from .network import build_b200
    dev = torch.device(device or f"cuda:{torch.cuda.current_device()}")
    nets = [build_b200(config, rank=r, size=size, device=dev) for r in range(size)]
    sims = [Simulator(config, nets[r], direct_log=False, use_graphs=False, device=dev)
            for r in range(size)]
    has = [((n.row_off[1:] - n.row_off[:-1]) > 0).cpu().numpy() for n in nets]
    n_col = config.grid.neurons_per_column
    masks, luts = [], []
    for r in range(size):
        masks.append(torch.as_tensor(dest_masks_from_rows(has, sims[r].gids), device=dev))
        lut = np.full(config.grid.n_columns, -1, np.int64)
        lut[nets[r].owned_columns] = np.arange(len(nets[r].owned_columns))
        luts.append(torch.as_tensor(lut, device=dev))
    n_in = torch.zeros(1, dtype=torch.int32, device=dev)
    off = _lib.Ctl.out_n.offset
    stream = torch.cuda.current_stream(dev)
    t0 = time.perf_counter()
    for step in range(config.n_steps):
        out = []
        for r, sim in enumerate(sims):
            sim._launch_step(stream.cuda_stream)
        torch.cuda.synchronize(dev)
        for r, sim in enumerate(sims):
            k = int(sim.ctl().out_n)
            g = sim.buf["out_gid"][:k].long() & 0xFFFFFFFF
            li = luts[r][g // n_col] * n_col + g % n_col
            out.append((g, sim.buf["out_t"][:k].clone(), masks[r][li] if k else g))
            sim.buf["ctl"].view(torch.uint8)[off:off + 4].zero_()
        for d, sim in enumerate(sims):
            gs, ts = [], []
            for g, tm, m in out:
                if g.numel():
                    sel = ((m >> d) & 1).bool()
                    gs.append(g[sel])
                    ts.append(tm[sel])
            in_g = torch.cat(gs).to(torch.int32) if gs else torch.zeros(0, dtype=torch.int32,
                                                                        device=dev)
            in_t = torch.cat(ts) if ts else torch.zeros(0, dtype=torch.float64, device=dev)
            n_in.fill_(int(in_g.numel()))
            _lib.check(sim.L.cc_ingest(C.byref(sim.shard), in_g.data_ptr() if in_g.numel() else 0,
                                       in_t.data_ptr() if in_t.numel() else 0, n_in.data_ptr(),
                                       stream.cuda_stream), "cc_ingest")
            torch.cuda.synchronize(dev)
        if (step + 1) % 100 == 0 or step == config.n_steps - 1:
            for sim in sims:
                sim.check()
    wall = time.perf_counter() - t0
    ctls = [sim.ctl() for sim in sims]
    parts = [sim.raster() for sim in sims]
    g = np.concatenate([p[0] for p in parts]) if parts else np.empty(0, np.uint64)
    t = np.concatenate([p[1] for p in parts]) if parts else np.empty(0)
    o = np.lexsort((g, t))
    g, t = g[o], t[o]
    return RunResult(
        config=config, worker_count=size, raster_gids=g, raster_times=t,
        n_spikes=sum(int(c.n_spikes) for c in ctls),
        recurrent_events=sum(int(c.rec_events) for c in ctls),
        external_events=sum(int(c.ext_events) for c in ctls),
        recurrent_synapses=sum(n.n_synapses for n in nets),
        construction_checksum=sum(n.checksum for n in nets) % 2 ** 64,
        raster_checksum=raster_checksum(g, t),
        construction_seconds=max(n.construction_seconds for n in nets),
        sim_seconds_wall=wall,
        substep_seconds={"deliver": 0.0, "expand": 0.0, "external": 0.0, "integrate": wall},
        steady_bytes_per_worker=[n.steady_bytes for n in nets],
        peak_bytes_per_worker=[n.peak_bytes for n in nets])


def _init_dist():
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        dist.init_process_group(backend="nccl" if torch.cuda.is_available() else "gloo")
    rank, size = dist.get_rank(), dist.get_world_size()
    if torch.cuda.is_available():
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    return rank, size


def run_multi_gpu(config, workers: int):
    """Run under torchrun (WORLD_SIZE == workers): every rank simulates its
    shard; rank 0 returns the merged RunResult (engine._merge_results
    semantics, engine.py:414-446), other ranks return None."""
    import torch
    import torch.distributed as dist
    from .engine import RunResult, raster_checksum
    if int(os.environ.get("WORLD_SIZE", "1")) != workers:
        raise RuntimeError(f"run_b200(workers={workers}) must be launched with torchrun "
                           f"--nproc-per-node {workers} (one process per GPU)")
    rank, size = _init_dist()
    ds = DistributedSimulator(config, rank, size)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ds.advance(config.n_steps)
    wall = time.perf_counter() - t0
    c = ds.sim.ctl()
    g, t = ds.sim.raster()
    mine = dict(g=g, t=t, n_spikes=int(c.n_spikes), rec=int(c.rec_events), ext=int(c.ext_events),
                syn=ds.net.n_synapses, csum=ds.net.checksum, cons=ds.net.construction_seconds,
                wall=wall, steady=ds.net.steady_bytes, peak=ds.net.peak_bytes,
                xchg=ds.timers["exchange"], kern=ds.timers["kernels"])
    allr = [None] * size
    dist.all_gather_object(allr, mine)
    if rank != 0:
        return None
    g = np.concatenate([r["g"] for r in allr])
    t = np.concatenate([r["t"] for r in allr])
    o = np.lexsort((g, t))
    g, t = g[o], t[o]
    return RunResult(
        config=config, worker_count=size, raster_gids=g, raster_times=t,
        n_spikes=sum(r["n_spikes"] for r in allr), recurrent_events=sum(r["rec"] for r in allr),
        external_events=sum(r["ext"] for r in allr), recurrent_synapses=sum(r["syn"] for r in allr),
        construction_checksum=sum(r["csum"] for r in allr) % 2 ** 64,
        raster_checksum=raster_checksum(g, t),
        construction_seconds=max(r["cons"] for r in allr),
        sim_seconds_wall=max(r["wall"] for r in allr),
        substep_seconds={"deliver": max(r["xchg"] for r in allr),
                         "expand": 0.0, "external": 0.0,
                         "integrate": max(r["kern"] for r in allr)},
        steady_bytes_per_worker=[r["steady"] for r in allr],
        peak_bytes_per_worker=[r["peak"] for r in allr])


def bench_distributed(args, cfg) -> None:
    """bench.py for N > 1 (launched by torchrun): device-timed K steps, max
    over ranks, rank 0 prints the JSON line."""
    import torch
    import torch.distributed as dist
    rank, size = _init_dist()
    ds = DistributedSimulator(cfg, rank, size)
    ds.advance(args.warmup)
    c0 = ds.sim.ctl()
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    x0 = ds.timers["exchange"]
    ds.advance(args.steps)
    ev1.record()
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([ev0.elapsed_time(ev1)], device=ds.dev)
    xs = torch.tensor([ds.timers["exchange"] - x0], device=ds.dev, dtype=torch.float64)
    c1 = ds.sim.ctl()
    ev = torch.tensor([(c1.rec_events + c1.ext_events) - (c0.rec_events + c0.ext_events)],
                      device=ds.dev, dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    dist.all_reduce(xs, op=dist.ReduceOp.MAX)
    dist.all_reduce(ev, op=dist.ReduceOp.SUM)
    if rank == 0:
        ms_v = float(ms.item())
        line = {
            "metric": "synaptic events/s (recurrent + external)",
            "value": float(ev.item()) / (ms_v / 1e3), "unit": "events/s", "n_gpus": size,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_v / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded counter-based RNG, bit-exact with the reference streams",
            "config": {"workload": f"BASELINE config {args.config}", "grid":
                       f"{cfg.grid.nx}x{cfg.grid.ny}", "parallelism": f"column blocks x{size}"},
            "wall_s_per_sim_s": (ms_v / 1e3) / (args.steps * cfg.timestep_ms / 1e3),
            "exchange_fraction": float(xs.item()) * 1e3 / ms_v,
            "gpu_launches": 5 * args.steps,
        }
        print(json.dumps(line))
    dist.destroy_process_group()
