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


def _aer_cap(sim) -> int:
    """Spikes one shard can emit in a step: every owned neuron at most the
    engine's per-step bound (refractoriness >= dt gives 1)."""
    from .engine import _spikes_per_step_bound
    return max(1, sim.n_local * _spikes_per_step_bound(sim.cfg))


class DistributedSimulator:
    """One rank's shard: Simulator in exchange mode plus a device-driven AER
    exchange per step - cc_pack_aer (fixed-size slot per destination), one
    equal-split all_to_all_single (NCCL), cc_ingest_aer - so whole chunks of
    steps are captured into a CUDA graph with no host synchronisation."""

    def __init__(self, cfg, rank: int, size: int, device=None, group=None, chunk: int = 100,
                 use_graphs: bool = True, force_exchange: bool = False, **sim_kw):
        import torch
        from .engine import Simulator
        from .network import build_b200
        self.torch = torch
        self.rank, self.size, self.group = rank, size, group
        self.dev = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        self.net = build_b200(cfg, rank=rank, size=size, device=self.dev)
        has = _has_row_all_ranks(self.net, size, group)
        n = cfg.grid.neurons_per_column
        gids = (self.net.owned_columns[:, None].astype(np.int64) * n + np.arange(n)[None, :]).ravel()
        # own spikes are logged locally by the neuron kernel; only neurons with
        # rows on other shards go through the exchange (self bit cleared)
        masks = dest_masks_from_rows(has, gids) & ~np.int64(1 << rank)
        self.has_remote = bool(masks.any())
        self.sim = Simulator(cfg, self.net, direct_log=True, remote=masks != 0, use_graphs=False,
                             device=self.dev, **sim_kw)
        self.mask = torch.as_tensor(masks.astype(np.uint32).view(np.int32), device=self.dev)
        n = cfg.grid.neurons_per_column
        self.local_of_col = np.full(cfg.grid.n_columns, -1, np.int64)
        self.local_of_col[self.net.owned_columns] = np.arange(len(self.net.owned_columns))
        self.lut = torch.as_tensor(self.local_of_col.astype(np.int32), device=self.dev)
        self.n_col = n
        self.cap = _aer_cap(self.sim)
        # one rank: nothing to exchange (force_exchange keeps the pack / NCCL /
        # ingest kernels in the step, to measure or test that path on one GPU)
        self.exchange_needed = size > 1 or force_exchange
        self.send = torch.zeros((size, 1 + 2 * self.cap), dtype=torch.int64, device=self.dev)
        self.recv = torch.zeros_like(self.send)
        self.chunk = max(1, int(chunk))
        self.use_graphs = use_graphs
        self._graph = None
        self.t = 0
        self.timers = dict(exchange=0.0, kernels=0.0)

    def _launch(self, stream) -> None:
        """One step on `stream` (torch stream): deliver, neuron step, pack,
        all-to-all, ingest - no host synchronisation."""
        from . import _lib
        L, sim, s = self.sim.L, self.sim, stream.cuda_stream
        sim._launch_step(s)
        if not self.exchange_needed:
            return
        _lib.check(L.cc_pack_aer(C.byref(sim.shard), self.mask.data_ptr(), self.size, self.cap,
                                 self.send.data_ptr(), self.lut.data_ptr(), s), "cc_pack_aer")
        self.dist_a2a()
        _lib.check(L.cc_ingest_aer(C.byref(sim.shard), self.recv.data_ptr(), self.size, self.cap,
                                   s), "cc_ingest_aer")

    def measure_exchange(self, n_steps: int):
        """(exchange ms, step ms) summed over n eager steps, CUDA events on the
        stream: exchange = pack + all-to-all + ingest."""
        from . import _lib
        torch = self.torch
        st = torch.cuda.current_stream(self.dev)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n_steps)]
        L, sim, s = self.sim.L, self.sim, st.cuda_stream
        for e in ev:
            e[0].record(st)
            sim._launch_step(s)
            e[1].record(st)
            if self.exchange_needed:
                _lib.check(L.cc_pack_aer(C.byref(sim.shard), self.mask.data_ptr(), self.size,
                                         self.cap, self.send.data_ptr(), self.lut.data_ptr(), s))
                self.dist_a2a()
                _lib.check(L.cc_ingest_aer(C.byref(sim.shard), self.recv.data_ptr(), self.size,
                                           self.cap, s))
            e[2].record(st)
        torch.cuda.synchronize(self.dev)
        self.t += n_steps
        self.sim.t = self.t
        self.sim.check()
        return (sum(e[1].elapsed_time(e[2]) for e in ev), sum(e[0].elapsed_time(e[2]) for e in ev))

    def dist_a2a(self) -> None:
        import torch.distributed as dist
        dist.all_to_all_single(self.recv, self.send, group=self.group)

    def step(self) -> None:
        self._launch(self.torch.cuda.current_stream(self.dev))
        self.t += 1

    def _capture(self) -> None:
        torch = self.torch
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=torch.cuda.Stream(self.dev)):
            st = torch.cuda.current_stream(self.dev)
            for _ in range(self.chunk):
                self._launch(st)
        self._graph = g

    def advance(self, n_steps: int) -> None:
        """Steps in chunks (CUDA graph replays once the communicator is warm),
        with the device counters checked and the raster drained per chunk."""
        done = 0
        while done < n_steps:
            k = min(self.chunk, n_steps - done)
            if self.use_graphs and k == self.chunk and self.t > 0:
                if self._graph is None:
                    self._capture()
                self._graph.replay()
                self.t += k
            else:
                for _ in range(k):
                    self.step()
            done += k
            self.sim.t = self.t
            self.sim.check()


def run_local_shards(config, size: int, device=None, flat_ingest: bool = False,
                     local_direct: bool = True):
    """All `size` shards of a multi-GPU run, stepped in turn on ONE device.

    Same shard code as run_multi_gpu - per-rank generator (build_b200 rank /
    size), exchange-mode neuron step (out-list), cc_pack_aer, cc_ingest_aer -
    with the all-to-all done by device copies of the packed slots.  No kernel
    waits on another shard's kernel.  Used to test partition invariance of
    the CUDA path on a single B200 (tests/test_gpu_parity.py).  flat_ingest:
    receive through cc_ingest (one flat AER list per shard, the entry for
    hosts with their own transport) instead of cc_ingest_aer."""
    import torch
    from . import _lib
    from .engine import RunResult, Simulator, raster_checksum
    from .network import build_b200
    dev = torch.device(device or f"cuda:{torch.cuda.current_device()}")
    nets = [build_b200(config, rank=r, size=size, device=dev) for r in range(size)]
    has = [((n.row_off[1:] - n.row_off[:-1]) > 0).cpu().numpy() for n in nets]
    n = config.grid.neurons_per_column
    mk = []
    for r in range(size):
        gids = (nets[r].owned_columns[:, None].astype(np.int64) * n + np.arange(n)[None, :]).ravel()
        m = dest_masks_from_rows(has, gids)
        mk.append(m & ~np.int64(1 << r) if local_direct else m)
    # local_direct: own spikes logged by the neuron kernel, the exchange carries
    # only spikes with rows on other shards (DistributedSimulator's mode);
    # otherwise every spike goes out-list -> pack -> exchange -> ingest
    sims = [Simulator(config, nets[r], direct_log=local_direct,
                      remote=(mk[r] != 0) if local_direct else None, use_graphs=False, device=dev)
            for r in range(size)]
    cap = max(_aer_cap(sm) for sm in sims)
    masks, luts, sends = [], [], []
    for r in range(size):
        masks.append(torch.as_tensor(mk[r].astype(np.uint32).view(np.int32), device=dev))
        lut = np.full(config.grid.n_columns, -1, np.int32)
        lut[nets[r].owned_columns] = np.arange(len(nets[r].owned_columns))
        luts.append(torch.as_tensor(lut, device=dev))
        sends.append(torch.zeros((size, 1 + 2 * cap), dtype=torch.int64, device=dev))
    recv = torch.zeros((size, 1 + 2 * cap), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    s = stream.cuda_stream
    t0 = time.perf_counter()
    for step in range(config.n_steps):
        for r, sim in enumerate(sims):
            sim._launch_step(s)
            _lib.check(sim.L.cc_pack_aer(C.byref(sim.shard), masks[r].data_ptr(), size, cap,
                                         sends[r].data_ptr(), luts[r].data_ptr(), s),
                       "cc_pack_aer")
        for d, sim in enumerate(sims):
            for r in range(size):                       # recv[r] = slot d of source r
                recv[r].copy_(sends[r][d])
            if flat_ingest:
                cnt = recv[:, 0].tolist()
                ev = torch.cat([recv[r, 1:1 + 2 * c].view(-1, 2) for r, c in enumerate(cnt)])
                g32 = ev[:, 0].to(torch.int32).contiguous()
                tf = ev[:, 1].contiguous().view(torch.float64)
                n_in = torch.tensor([g32.numel()], dtype=torch.int32, device=dev)
                _lib.check(sim.L.cc_ingest(C.byref(sim.shard), g32.data_ptr(), tf.data_ptr(),
                                           n_in.data_ptr(), s), "cc_ingest")
                torch.cuda.synchronize(dev)             # the temporaries die here
            else:
                _lib.check(sim.L.cc_ingest_aer(C.byref(sim.shard), recv.data_ptr(), size, cap,
                                               s), "cc_ingest_aer")
        if (step + 1) % 100 == 0 or step == config.n_steps - 1:
            for sim in sims:
                sim.check()
    torch.cuda.synchronize(dev)
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
                wall=wall, steady=ds.net.steady_bytes, peak=ds.net.peak_bytes)
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
        # the exchange runs inside the same CUDA graphs as the kernels
        substep_seconds={"deliver": 0.0, "expand": 0.0, "external": 0.0,
                         "integrate": max(r["wall"] for r in allr)},
        steady_bytes_per_worker=[r["steady"] for r in allr],
        peak_bytes_per_worker=[r["peak"] for r in allr])


def bench_distributed(args, cfg) -> None:
    """bench.py for N > 1 (launched by torchrun): K steps timed with CUDA
    events on every rank (max over ranks); returns the JSON line on rank 0.  The
    step loop is host-driven (exchange per step), so the same timed region is
    also the end-to-end number (host loop, NCCL exchange, raster copies)."""
    import torch
    import torch.distributed as dist
    rank, size = _init_dist()
    ds = DistributedSimulator(cfg, rank, size, force_exchange=getattr(args, "exchange", False))
    ds.advance(args.warmup)
    c0 = ds.sim.ctl()
    clocks = None
    if rank == 0:
        import bench as _b                               # the repo-root bench module
        clocks = _b.Clocks(torch.cuda.current_device())
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    ev0.record()
    ds.advance(args.steps)
    ev1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    dist.barrier()
    clk = clocks.stop() if clocks is not None else None
    ms = torch.tensor([ev0.elapsed_time(ev1)], device=ds.dev)
    wl = torch.tensor([wall], device=ds.dev, dtype=torch.float64)
    c1 = ds.sim.ctl()
    ev = torch.tensor([(c1.rec_events + c1.ext_events) - (c0.rec_events + c0.ext_events),
                       c1.rec_events - c0.rec_events, c1.n_spikes - c0.n_spikes],
                      device=ds.dev, dtype=torch.float64)
    # exchange share from a short eager sample after the timed region
    xm, sm = ds.measure_exchange(20)
    xs = torch.tensor([xm / max(sm, 1e-9)], device=ds.dev, dtype=torch.float64)
    a2a_bytes = float(ds.send.numel() * 8)
    for x in (ms, xs, wl):
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
    dist.all_reduce(ev, op=dist.ReduceOp.SUM)
    if rank == 0:
        ms_v = float(ms.item())
        total, rec = float(ev[0].item()), float(ev[1].item())
        try:
            hbm = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(
                os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"])
        except Exception:
            hbm = 6650.0
        ach = rec / (ms_v / 1e3) * 17 / 1e9 / size          # per GPU
        line = {
            "metric": "synaptic events/s (recurrent + external)",
            "value": total / (ms_v / 1e3), "unit": "events/s", "n_gpus": size,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_v / args.steps,
            "higher_is_better": True,
            "scaling": "weak" if (size > 1 and getattr(args, "scaling", "strong") == "weak")
            else "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded counter-based RNG (connectivity, Poisson drive), "
                    "bit-exact with the reference streams",
            "config": {"workload": (f"BASELINE config {args.config}"
                                    + (" grid once per GPU (weak scaling)"
                                       if size > 1 and getattr(args, "scaling", "") == "weak"
                                       else "")
                                    + f": {cfg.grid.nx}x{cfg.grid.ny} columns x "
                                      f"{cfg.grid.neurons_per_column} neurons, "
                                      f"{cfg.kernel.kind} lateral decay, calibrated drive"),
                       "grid": f"{cfg.grid.nx}x{cfg.grid.ny}", "neurons": cfg.grid.n_neurons,
                       "parallelism": f"column blocks x{size} (one process per GPU, NCCL)",
                       "l2": "no flush between steps (per-step working set > 126 MB L2)"},
            "wall_s_per_sim_s": (ms_v / 1e3) / (args.steps * cfg.timestep_ms / 1e3),
            "exchange_fraction": float(xs.item()),
            "exchange": "device-driven: cc_pack_aer + equal-split NCCL all_to_all_single "
                        f"({a2a_bytes / 1e6:.2f} MB per rank per step) + cc_ingest_aer, "
                        "captured in CUDA graphs of 100 steps",
            "roofline": {"bound": "hbm", "kernel": "whole step, per GPU (exchange mode)",
                         "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                         "traffic": None, "bytes_per_event": 17},
            "e2e": {"value": total / float(wl.item()), "unit": "events/s",
                    "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 12.0 * float(ev[2].item()) / args.steps,
                    "api": "DistributedSimulator.advance wall (graph replays, per-chunk "
                           "counter checks and raster copies)"},
            "gpu_launches": 5 * args.steps,       # deliver, plan, stage, pack, ingest per step
            "clocks": clk,
        }
        dist.destroy_process_group()
        return line
    dist.destroy_process_group()
