"""Multi-GPU runs: one process per GPU, columns sharded by contiguous blocks.

Replaces the reference's transport layer for the hot loop:

    construct_network exchange (network.py:229-310)  -> each rank regenerates its
                                                        own incoming synapses
                                                        (network.build_b200); only
                                                        row-presence bitmaps are
                                                        all-gathered once to build
                                                        the destination masks
    deliver_spikes two-phase AER (network.py:325-379) -> the per-step spike
                                                        exchange, one of three
                                                        transports (below)
    run / run_multiprocess (engine.py:449-528)       -> run_spawned (one process
                                                        per worker, started here)
                                                        and run_multi_gpu (under
                                                        torchrun)

Transports of the per-step exchange (DistributedSimulator):

  "p2p"   the product path.  Every rank owns a receive window (CUDA IPC) with one
          region per source rank and step parity, sized for the exact worst case
          (the source's neurons that have >= 1 synapse here), plus a flag word
          per source.  k_stage pushes each spike of a neuron with remote rows into
          the destination's region as it is emitted (NVLink stores, overlapped
          with the integration of the rest of the step), its last block publishes
          the counts with a system-scope release, and cc_exchange_ingest waits for
          every source's flag and logs the received spikes.  Only the spikes
          actually emitted cross NVLink; no NCCL call is on the step.  Chunks of
          steps run as CUDA graphs when the ranks own distinct GPUs ("device"
          sync).  When ranks share a GPU (tests, run_spawned on a one-GPU host)
          the same kernels run eagerly with a host barrier between the push and
          the ingest ("host" sync), so no kernel ever waits on another process's.
  "nccl"  baseline: cc_pack_aer into one fixed-size slot per destination, an
          NCCL all-to-all of the slots (equal splits; the self slot is empty and
          copied locally) captured in the chunk graphs, cc_ingest_aer.  Slots are sized for the largest exact per-pair
          worst case, agreed by all ranks.
  "gloo"  the slots transport with the all-to-all on the host over gloo (eager;
          ranks may share a GPU): tests the pack / ingest kernels across real
          processes.

SpikeExchange is the host-side statement of the reference protocol (counts,
then payloads of those sizes) used by the CPU tests and the CPU oracle.
"""

from __future__ import annotations

import ctypes as C
import json
import os
import socket
import time
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = ["SpikeExchange", "dest_masks_from_rows", "send_caps", "window_layout", "WindowLayout",
           "DistributedSimulator", "run_multi_gpu", "run_spawned", "bench_distributed",
           "ProtocolViolation", "run_local_shards", "merge_pieces", "agree_errors",
           "TRANSPORTS"]

TRANSPORTS = ("p2p", "nccl", "gloo")
XWAIT_NS = int(30e9)          # a source's step flag not in after 30 s: CC_ERR_XWAIT
FLAG_SLOTS = 32               # flag words per parity (one per possible source rank)
REC_BYTES = 16                # AER record {gid, t lo, t hi, 0}


class ProtocolViolation(RuntimeError):
    """Payload does not match its announced counter (network.py:66-67)."""


def dest_masks_from_rows(has_row_by_rank: List[np.ndarray], owned_gids: np.ndarray) -> np.ndarray:
    """Bit d of mask[i] is set iff rank d stores >= 1 synapse of source
    owned_gids[i] (the reference's source_masks, network.py:229-230)."""
    mask = np.zeros(len(owned_gids), dtype=np.int64)
    for d, has in enumerate(has_row_by_rank):
        mask |= (np.asarray(has)[owned_gids].astype(np.int64) << d)
    return mask


def send_caps(masks: np.ndarray, size: int) -> np.ndarray:
    """caps[d] = the owned neurons with destination bit d: the most spikes this
    rank can send to rank d in one step (a neuron spikes at most once per step
    since tau_arp >= dt, engine._spikes_per_step_bound)."""
    m = np.asarray(masks, np.int64)
    return np.array([int(((m >> d) & 1).sum()) for d in range(size)], np.int64)


@dataclass(frozen=True)
class WindowLayout:
    """Byte layout of one rank's receive window: flag words [2][FLAG_SLOTS]
    (u64), then per parity one region per source rank."""
    rec_off: Tuple[Tuple[int, ...], Tuple[int, ...]]    # [parity][src] byte offset
    cap: Tuple[int, ...]                               # [src] records
    nbytes: int

    def flag_off(self, parity: int, src: int) -> int:
        return (parity * FLAG_SLOTS + src) * 8


def window_layout(caps_to_me: Sequence[int]) -> WindowLayout:
    """Layout of a receive window given the per-source capacities (records)."""
    caps = tuple(int(c) for c in caps_to_me)
    if len(caps) > FLAG_SLOTS:
        raise ValueError(f"at most {FLAG_SLOTS} ranks")
    off = 2 * FLAG_SLOTS * 8
    rec = []
    for _ in range(2):
        row = []
        for c in caps:
            row.append(off)
            off += c * REC_BYTES
        rec.append(tuple(row))
    return WindowLayout(rec_off=(rec[0], rec[1]), cap=caps, nbytes=max(off, 2 * FLAG_SLOTS * 8))


def agree_errors(bits: int, step: int, group=None) -> Tuple[int, int, int]:
    """All ranks learn whether any rank failed: (OR of the error bits, the
    earliest failing step, the lowest failing rank or -1).  Host collective
    over the (gloo) group; called after every chunk so that no rank steps on
    while another has stopped (its peers would wait for its exchange)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    big = (1 << 62)
    v = torch.tensor([1 if bits else 0, step if bits else big, rank if bits else big],
                     dtype=torch.int64)
    anyf = v[:1].clone()
    dist.all_reduce(anyf, op=dist.ReduceOp.MAX, group=group)
    if not int(anyf.item()):
        return 0, -1, -1
    b = torch.tensor([int(bits)], dtype=torch.int64)
    dist.all_reduce(b, op=dist.ReduceOp.BOR if hasattr(dist.ReduceOp, "BOR") else dist.ReduceOp.MAX,
                    group=group)
    mn = v[1:].clone()
    dist.all_reduce(mn, op=dist.ReduceOp.MIN, group=group)
    return int(b.item()), int(mn[0].item()), int(mn[1].item())


class SpikeExchange:
    """Per-step AER exchange between shards over a torch.distributed group
    (host-side statement of the reference protocol).

    Payload per spike: (gid, float64 time bits) as two int64 words.  Counts go
    first (one all_to_all of W integers), then the payload as an
    all_to_all_single with per-pair split sizes - the reference's
    counters-then-payloads protocol (network.py:325-379).
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
            dest = sel.nonzero(as_tuple=False)                         # (spike, dest) pairs
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


def _owned_gids(net, n_col: int) -> np.ndarray:
    return (net.owned_columns[:, None].astype(np.int64) * n_col + np.arange(n_col)[None, :]).ravel()


def _has_row(net) -> np.ndarray:
    return ((net.row_off[1:] - net.row_off[:-1]) > 0).cpu().numpy()


def _xpeer_table(entries: List[Tuple[int, int, int, int, int]], device):
    """cc_xpeer array on the device from (rec0, rec1, flag0, flag1, cap) tuples."""
    import torch
    from . import _lib
    arr = (_lib.XPeer * max(1, len(entries)))()
    for i, (r0, r1, f0, f1, cap) in enumerate(entries):
        arr[i].rec[0], arr[i].rec[1] = r0, r1
        arr[i].flag[0], arr[i].flag[1] = f0, f1
        arr[i].cap = cap
    raw = np.frombuffer(bytes(arr), dtype=np.uint8).copy()
    return torch.from_numpy(raw).to(device)


class PeerExchange:
    """The p2p transport's buffers for one shard: its own receive window, the
    peers' windows as mapped here, and the device tables cc_xpeer xdst / xsrc.

    `windows[r]` is rank r's window base address in this process; caps is the
    [src][dst] capacity matrix (records).  loopback: a one-rank run routes its
    own spikes through its window (measures the exchange on one GPU)."""

    def __init__(self, sim, rank: int, size: int, masks: np.ndarray, caps: np.ndarray,
                 windows: List[int], loopback: bool = False, keep=()):
        import torch
        self.sim, self.rank, self.size = sim, rank, size
        self.caps = np.asarray(caps, np.int64)
        self.windows = list(windows)
        self.keep = list(keep)                   # objects owning the window memory
        self.loopback = loopback
        lay = [window_layout(self.caps[:, d]) for d in range(size)]
        self.layouts = lay

        def linked(a, b):
            return a != b or loopback

        dst, src = [], []
        for d in range(size):
            if linked(rank, d):
                L, base = lay[d], self.windows[d]
                dst.append((base + L.rec_off[0][rank], base + L.rec_off[1][rank],
                            base + L.flag_off(0, rank), base + L.flag_off(1, rank),
                            int(self.caps[rank, d])))
            else:
                dst.append((0, 0, 0, 0, 0))
        me, base = lay[rank], self.windows[rank]
        for s in range(size):
            if linked(s, rank):
                src.append((base + me.rec_off[0][s], base + me.rec_off[1][s],
                            base + me.flag_off(0, s), base + me.flag_off(1, s),
                            int(self.caps[s, rank])))
            else:
                src.append((0, 0, 0, 0, 0))
        dev = sim.dev
        self.xdst = _xpeer_table(dst, dev)
        self.xsrc = _xpeer_table(src, dev)
        self.xcnt = torch.zeros(32, dtype=torch.int32, device=dev)
        self.xmask = torch.as_tensor(np.asarray(masks, np.int64).astype(np.uint32).view(np.int32),
                                     device=dev)
        sh = sim.shard
        sh.n_ranks, sh.rank = size, rank
        sh.xmask = self.xmask.data_ptr()
        sh.xdst, sh.xsrc = self.xdst.data_ptr(), self.xsrc.data_ptr()
        sh.xcnt = self.xcnt.data_ptr()
        sh.xwait_ns = XWAIT_NS
        if loopback:
            sh.direct_log = 0                    # own spikes come back through the window

    @property
    def window_bytes(self) -> int:
        return self.layouts[self.rank].nbytes


class _IpcWindow:
    """A receive window allocated with cc_xwin_alloc; peers' windows opened
    with cc_xwin_open (closed / freed on release)."""

    def __init__(self, L, nbytes: int):
        self.L = L
        self.ptr = C.c_void_p()
        self.handle = C.create_string_buffer(64)
        from . import _lib
        _lib.check(L.cc_xwin_alloc(int(nbytes), C.byref(self.ptr), self.handle), "cc_xwin_alloc")
        self.opened: List[int] = []

    def open(self, handle: bytes) -> int:
        from . import _lib
        p = C.c_void_p()
        _lib.check(self.L.cc_xwin_open(handle, C.byref(p)), "cc_xwin_open")
        self.opened.append(p.value)
        return p.value

    def release(self):
        for p in self.opened:
            self.L.cc_xwin_close(p)
        self.opened = []
        if self.ptr.value:
            self.L.cc_xwin_free(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def _exchange_plan(net, rank: int, size: int, group, n_col: int):
    """Destination masks of this rank's neurons (own bit clear) and the
    [src][dst] capacity matrix, all-gathered (host collectives on `group`)."""
    import torch
    import torch.distributed as dist
    has = torch.from_numpy(_has_row(net).astype(np.uint8))
    gathered = [torch.empty_like(has) for _ in range(size)]
    dist.all_gather(gathered, has, group=group)
    hs = [g.numpy().astype(bool) for g in gathered]
    masks = dest_masks_from_rows(hs, _owned_gids(net, n_col)) & ~np.int64(1 << rank)
    mine = torch.from_numpy(send_caps(masks, size))
    rows = [torch.empty_like(mine) for _ in range(size)]
    dist.all_gather(rows, mine, group=group)
    caps = np.stack([r.numpy() for r in rows])           # caps[s][d]
    return masks, caps


class DistributedSimulator:
    """One rank's shard: Simulator plus the per-step spike exchange.

    transport "p2p" (default), "nccl" or "gloo" (module docstring); sync
    "device" (chunks of steps as CUDA graphs; ranks own distinct GPUs) or
    "host" (eager steps, host barrier between the push and the ingest: ranks
    may share a GPU).  `group` is a gloo (CPU) group for setup, barriers and
    the per-chunk error agreement; nccl_group the NCCL group of the "nccl"
    transport.  loopback (one rank, p2p): the rank's own spikes go through its
    window, to measure the exchange on one GPU."""

    def __init__(self, cfg, rank: int, size: int, device=None, group=None, chunk: int = 100,
                 transport: str = "p2p", sync: str = "device", nccl_group=None,
                 loopback: bool = False, **sim_kw):
        import torch
        from .engine import Simulator
        from .network import build_b200
        if transport not in TRANSPORTS:
            raise ValueError(f"transport must be one of {TRANSPORTS}")
        if sync not in ("device", "host"):
            raise ValueError("sync must be 'device' or 'host'")
        if transport == "nccl" and sync == "host":
            raise ValueError("the nccl transport needs one GPU per rank (sync='device')")
        if transport == "gloo":
            sync = "host"
        self.torch = torch
        self.cfg = cfg
        self.rank, self.size, self.group, self.nccl_group = rank, size, group, nccl_group
        self.transport, self.sync = transport, sync
        self.dev = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        self.net = build_b200(cfg, rank=rank, size=size, device=self.dev)
        n = cfg.grid.neurons_per_column
        self.n_col = n
        masks, caps = _exchange_plan(self.net, rank, size, group, n)
        self.masks, self.caps = masks, caps
        self.loopback = bool(loopback and size == 1)
        if self.loopback:
            has = _has_row(self.net)[_owned_gids(self.net, n)]
            masks = has.astype(np.int64)                 # bit 0: rows on this (own) shard
            caps = send_caps(masks, 1)[None, :]
            self.masks, self.caps = masks, caps
        self.exchange_needed = size > 1 or self.loopback
        self.x = None
        self._win = None
        if transport == "p2p":
            self.sim = Simulator(cfg, self.net, direct_log=True, use_graphs=False, device=self.dev,
                                 **sim_kw)
            if self.exchange_needed:
                self._setup_p2p(masks, caps)
        else:
            # (loopback: every spike goes out-list -> slot 0 -> back in)
            self.sim = Simulator(cfg, self.net, direct_log=not self.loopback,
                                 remote=None if self.loopback else masks != 0,
                                 use_graphs=False, device=self.dev, **sim_kw)
            # one slot size for every pair (the largest exact per-pair worst case):
            # every rank derives the same cap from the gathered matrix
            self.cap = max(1, int(caps.max()) if caps.size else 1)
            self.mask_dev = torch.as_tensor(np.asarray(masks, np.int64).astype(np.uint32)
                                            .view(np.int32), device=self.dev)
            lut = np.full(cfg.grid.n_columns, -1, np.int32)
            lut[self.net.owned_columns] = np.arange(len(self.net.owned_columns))
            self.lut = torch.as_tensor(lut, device=self.dev)
            self.send = torch.zeros((size, 1 + 2 * self.cap), dtype=torch.int64, device=self.dev)
            self.recv = torch.zeros_like(self.send)
            if transport == "gloo":
                self._send_h = torch.zeros(self.send.shape, dtype=torch.int64, pin_memory=True)
                self._recv_h = torch.zeros(self.send.shape, dtype=torch.int64)
        self.chunk = max(1, int(chunk))
        self._graph = None
        self.t = 0
        self.error = None
        self._barrier()

    # ------------------------------------------------------------ setup
    def _barrier(self):
        import torch.distributed as dist
        if self.size > 1:
            dist.barrier(group=self.group)

    def _setup_p2p(self, masks, caps):
        import torch.distributed as dist
        L = self.sim.L
        lay = window_layout(caps[:, self.rank])
        if self.loopback:
            self._win = _IpcWindow(L, lay.nbytes)
            windows = [self._win.ptr.value]
        else:
            self._win = _IpcWindow(L, lay.nbytes)
            handles = [None] * self.size
            dist.all_gather_object(handles, bytes(self._win.handle.raw), group=self.group)
            windows = [self._win.ptr.value if r == self.rank else self._win.open(handles[r])
                       for r in range(self.size)]
        self.x = PeerExchange(self.sim, self.rank, self.size, masks, caps, windows,
                              loopback=self.loopback, keep=[self._win])

    # ------------------------------------------------------------ steps
    def _a2a(self) -> None:
        """The slots transports' all-to-all (self slot not sent)."""
        import torch
        import torch.distributed as dist
        skip = -1 if self.loopback else self.rank

        def parts(buf):
            return [buf[d] if d != skip else buf[d][:0] for d in range(self.size)]
        if self.transport == "nccl":
            # equal splits over all slots (capturable); the self slot is empty
            # unless loopback, and NCCL copies it locally
            dist.all_to_all_single(self.recv, self.send, group=self.nccl_group)
            return
        # gloo: host staging (eager); gloo has all_to_all_single only
        self._send_h.copy_(self.send)
        rows = [d for d in range(self.size) if d != skip]
        w = self._send_h.shape[1]
        inp = self._send_h[rows].reshape(-1)
        out = torch.empty_like(inp)
        split = [w if d != skip else 0 for d in range(self.size)]
        dist.all_to_all_single(out, inp, output_split_sizes=split, input_split_sizes=split,
                               group=self.group)
        self._recv_h[rows] = out.view(len(rows), w)
        if skip >= 0:
            self._recv_h[skip, 0] = 0
        self.recv.copy_(self._recv_h)

    def _launch(self, stream) -> None:
        """One step on `stream`: deliver, neuron step (p2p: with the pushes and
        the flag publication), then the receive half."""
        from . import _lib
        L, sim, s = self.sim.L, self.sim, stream.cuda_stream
        sim._launch_step(s)
        if not self.exchange_needed:
            return
        if self.transport == "p2p":
            if self.sync == "host":
                self.torch.cuda.synchronize(self.dev)      # my pushes are complete
                self._barrier()                            # ... and every other rank's
            _lib.check(L.cc_exchange_ingest(C.byref(sim.shard), s), "cc_exchange_ingest")
            return
        _lib.check(L.cc_pack_aer(C.byref(sim.shard), self.mask_dev.data_ptr(), self.size,
                                 self.cap, self.send.data_ptr(), self.lut.data_ptr(), s),
                   "cc_pack_aer")
        if self.transport == "gloo":
            self.torch.cuda.synchronize(self.dev)
        self._a2a()
        _lib.check(L.cc_ingest_aer(C.byref(sim.shard), self.recv.data_ptr(), self.size, self.cap,
                                   s), "cc_ingest_aer")

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

    def _check_all(self, collect_raster: bool = True) -> None:
        """Drain this rank's chunk and agree with every other rank on errors:
        all ranks raise together (the failing one with its own message)."""
        from . import _lib
        self.torch.cuda.synchronize(self.dev)
        c = self.sim.ctl()
        bits, step = int(c.error_bits), int(c.error_step)
        if self.size > 1:
            abits, astep, arank = agree_errors(bits, step, self.group)
        else:
            abits, astep, arank = bits, step, (0 if bits else -1)
        if abits:
            if bits:
                msg = f"rank {self.rank}, step {step}: {_lib.decode_errors(bits)}"
            else:
                msg = (f"rank {arank} failed at step {astep} "
                       f"({_lib.decode_errors(abits)}); rank {self.rank} stopped with it")
            self.error = msg
            raise _lib.EngineError(msg, abits)
        self.sim.check(collect_raster)

    def advance(self, n_steps: int, collect_raster: bool = True) -> None:
        """Steps in chunks (device sync: CUDA graph replays once the first
        chunk ran eagerly), with the counters checked, errors agreed across
        ranks and the raster drained per chunk."""
        done = 0
        graphs = self.sync == "device"
        while done < n_steps:
            k = min(self.chunk, n_steps - done)
            if graphs and k == self.chunk and self.t > 0:
                if self._graph is None:
                    self._capture()
                self._graph.replay()
                self.t += k
            else:
                for _ in range(k):
                    self.step()
            done += k
            self.sim.t = self.t
            self._check_all(collect_raster)

    def exchange_stats(self) -> dict:
        c = self.sim.ctl()
        if self.transport == "p2p":
            per_step_bytes = None
            return dict(transport="p2p", sync=self.sync, records_sent=int(c.x_sent),
                        records_received=int(c.x_recv),
                        window_bytes=self.x.window_bytes if self.x else 0,
                        flag_bytes_per_step=8 * (self.size - 1 if self.size > 1 else 1),
                        bytes_per_record=REC_BYTES, per_step_bytes=per_step_bytes)
        slot = (1 + 2 * self.cap) * 8
        return dict(transport=self.transport, sync=self.sync, slot_bytes=slot,
                    per_step_bytes=slot * max(0, self.size - 1))

    def measure_exchange(self, n_steps: int):
        """(exchange ms, step ms) summed over n eager steps, CUDA events on the
        stream: the exchange is the receive half (p2p: the ingest, including
        the wait for the slowest source) or pack + all-to-all + ingest."""
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
                if self.transport == "p2p":
                    if self.sync == "host":
                        torch.cuda.synchronize(self.dev)
                        self._barrier()
                    _lib.check(L.cc_exchange_ingest(C.byref(sim.shard), s))
                else:
                    _lib.check(L.cc_pack_aer(C.byref(sim.shard), self.mask_dev.data_ptr(),
                                             self.size, self.cap, self.send.data_ptr(),
                                             self.lut.data_ptr(), s))
                    if self.transport == "gloo":
                        torch.cuda.synchronize(self.dev)
                    self._a2a()
                    _lib.check(L.cc_ingest_aer(C.byref(sim.shard), self.recv.data_ptr(),
                                               self.size, self.cap, s))
            e[2].record(st)
        torch.cuda.synchronize(self.dev)
        self.t += n_steps
        self.sim.t = self.t
        self._check_all()
        return (sum(e[1].elapsed_time(e[2]) for e in ev), sum(e[0].elapsed_time(e[2]) for e in ev))

    def piece(self, wall: float) -> dict:
        """This rank's share of the RunResult (engine._merge_results inputs)."""
        c = self.sim.ctl()
        g, t = self.sim.raster()
        return dict(rank=self.rank, g=g, t=t, n_spikes=int(c.n_spikes), rec=int(c.rec_events),
                    ext=int(c.ext_events), syn=self.net.n_synapses, csum=self.net.checksum,
                    cons=self.net.construction_seconds, wall=wall,
                    steady=self.net.steady_bytes, peak=self.net.peak_bytes,
                    device_bytes=self.sim.device_bytes + (self.x.window_bytes if self.x else 0),
                    exchange=self.exchange_stats())

    def close(self):
        if self._win is not None:
            self.torch.cuda.synchronize(self.dev)
            self._barrier()                       # nobody writes into a window being freed
            self._win.release()
            self._win = None


def merge_pieces(config, pieces: List[dict], record_raster: bool = True):
    """engine._merge_results (engine.py:414-446) over the ranks' pieces."""
    from .engine import RunResult, raster_checksum
    pieces = sorted(pieces, key=lambda p: p["rank"])
    if record_raster:
        g = np.concatenate([p["g"] for p in pieces]) if pieces else np.empty(0, np.uint64)
        t = np.concatenate([p["t"] for p in pieces]) if pieces else np.empty(0)
        o = np.lexsort((g, t))
        g, t = g[o].astype(np.uint64), t[o]
    else:
        g, t = np.empty(0, np.uint64), np.empty(0)
    wall = max((p["wall"] for p in pieces), default=0.0)
    return RunResult(
        config=config, worker_count=len(pieces), raster_gids=g, raster_times=t,
        n_spikes=sum(p["n_spikes"] for p in pieces),
        recurrent_events=sum(p["rec"] for p in pieces),
        external_events=sum(p["ext"] for p in pieces),
        recurrent_synapses=sum(p["syn"] for p in pieces),
        construction_checksum=sum(p["csum"] for p in pieces) % 2 ** 64,
        raster_checksum=raster_checksum(g, t),
        construction_seconds=max((p["cons"] for p in pieces), default=0.0),
        sim_seconds_wall=wall,
        substep_seconds={"deliver": 0.0, "expand": 0.0, "external": 0.0, "integrate": wall},
        steady_bytes_per_worker=[p["steady"] for p in pieces],
        peak_bytes_per_worker=[p["peak"] for p in pieces],
        workers=[{k: v for k, v in p.items() if k not in ("g", "t")} for p in pieces],
        device_stats=dict(exchange=[p.get("exchange") for p in pieces],
                          device_bytes=[p.get("device_bytes") for p in pieces]))


def run_local_shards(config, size: int, device=None, flat_ingest: bool = False,
                     local_direct: bool = True, transport: str = "slots"):
    """All `size` shards of a multi-GPU run, stepped in turn on ONE device, in
    one process.  No kernel waits on another shard's kernel.  Used to test
    partition invariance of the CUDA path on a single B200.

    transport "slots": exchange-mode neuron step (out-list), cc_pack_aer, the
    all-to-all as device copies of the packed slots, cc_ingest_aer (or, with
    flat_ingest, cc_ingest of one flat AER list per shard); local_direct=False
    sends every spike through the exchange.  transport "p2p": the peer-store
    kernels with the windows as plain device buffers: every shard's neuron
    step pushes into the others' windows, then every shard ingests."""
    import torch
    from . import _lib
    from .engine import Simulator
    from .network import build_b200
    dev = torch.device(device or f"cuda:{torch.cuda.current_device()}")
    nets = [build_b200(config, rank=r, size=size, device=dev) for r in range(size)]
    has = [_has_row(n) for n in nets]
    n = config.grid.neurons_per_column
    mk = []
    for r in range(size):
        m = dest_masks_from_rows(has, _owned_gids(nets[r], n))
        mk.append(m & ~np.int64(1 << r) if (local_direct or transport == "p2p") else m)
    stream = torch.cuda.current_stream(dev)
    s = stream.cuda_stream
    if transport == "p2p":
        sims = [Simulator(config, nets[r], direct_log=True, use_graphs=False, device=dev)
                for r in range(size)]
        caps = np.stack([send_caps(mk[r], size) for r in range(size)])
        wins = [torch.zeros(window_layout(caps[:, d]).nbytes, dtype=torch.uint8, device=dev)
                for d in range(size)]
        xs = [PeerExchange(sims[r], r, size, mk[r], caps, [w.data_ptr() for w in wins])
              for r in range(size)]
        t0 = time.perf_counter()
        for step in range(config.n_steps):
            for sim in sims:
                sim._launch_step(s)
            for sim in sims:
                _lib.check(sim.L.cc_exchange_ingest(C.byref(sim.shard), s), "cc_exchange_ingest")
            if (step + 1) % 100 == 0 or step == config.n_steps - 1:
                for sim in sims:
                    sim.check()
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - t0
        del xs
    else:
        sims = [Simulator(config, nets[r], direct_log=local_direct,
                          remote=(mk[r] != 0) if local_direct else None, use_graphs=False,
                          device=dev)
                for r in range(size)]
        caps = np.stack([send_caps(mk[r], size) for r in range(size)])
        cap = max(1, int(caps.max()))
        masks, luts, sends = [], [], []
        for r in range(size):
            masks.append(torch.as_tensor(mk[r].astype(np.uint32).view(np.int32), device=dev))
            lut = np.full(config.grid.n_columns, -1, np.int32)
            lut[nets[r].owned_columns] = np.arange(len(nets[r].owned_columns))
            luts.append(torch.as_tensor(lut, device=dev))
            sends.append(torch.zeros((size, 1 + 2 * cap), dtype=torch.int64, device=dev))
        recv = torch.zeros((size, 1 + 2 * cap), dtype=torch.int64, device=dev)
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
    pieces = []
    for r, sim in enumerate(sims):
        c = sim.ctl()
        g, t = sim.raster()
        pieces.append(dict(rank=r, g=g, t=t, n_spikes=int(c.n_spikes), rec=int(c.rec_events),
                           ext=int(c.ext_events), syn=nets[r].n_synapses, csum=nets[r].checksum,
                           cons=nets[r].construction_seconds, wall=wall,
                           steady=nets[r].steady_bytes, peak=nets[r].peak_bytes,
                           x_sent=int(c.x_sent), x_recv=int(c.x_recv)))
    res = merge_pieces(config, pieces)
    res.device_stats["x_sent"] = sum(p["x_sent"] for p in pieces)
    res.device_stats["x_recv"] = sum(p["x_recv"] for p in pieces)
    return res


# ------------------------------------------------------------------ runners
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pick_device(rank: int, size: int):
    """(cuda device index, sync mode): one GPU per rank when there are enough,
    else ranks share GPUs and the exchange is host-synchronised."""
    import torch
    n_dev = torch.cuda.device_count()
    if n_dev <= 0:
        raise RuntimeError("paper_1803_08833_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    return rank % n_dev, ("device" if n_dev >= size else "host")


def _rank_run(config, rank: int, size: int, transport: str, group, nccl_group=None,
              chunk: int = 100, sync: Optional[str] = None) -> dict:
    """Body of one worker: build, step the whole run, return its piece."""
    import torch
    import torch.distributed as dist
    dev_idx, auto_sync = _pick_device(rank, size)
    torch.cuda.set_device(dev_idx)
    sync = sync or auto_sync
    if transport == "nccl" and sync == "host":
        raise RuntimeError("transport 'nccl' needs one GPU per rank")
    ds = DistributedSimulator(config, rank, size, device=f"cuda:{dev_idx}", group=group,
                              nccl_group=nccl_group, transport=transport, sync=sync, chunk=chunk)
    fault = os.environ.get("CC_TEST_FAULT")          # tests: "rank:raster_cap" fails that rank
    if fault and int(fault.split(":")[0]) == rank:
        ds.sim.shard.raster_cap = int(fault.split(":")[1])
    try:
        dist.barrier(group=group)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ds.advance(config.n_steps, collect_raster=config.record_raster)
        wall = time.perf_counter() - t0
        return ds.piece(wall)
    finally:
        ds.close()


def _spawn_worker(rank: int, size: int, port: int, config, transport: str, chunk: int, q):
    import torch
    import torch.distributed as dist
    # own rendezvous: a parent started by torchrun hands down
    # TORCHELASTIC_USE_AGENT_STORE, with which rank 0 would connect to the
    # agent's store instead of starting this one
    os.environ.pop("TORCHELASTIC_USE_AGENT_STORE", None)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=size)
    try:
        nccl_group = None
        if transport == "nccl":
            nccl_group = dist.new_group(backend="nccl")
        q.put(("ok", rank, _rank_run(config, rank, size, transport, None, nccl_group, chunk)))
    except BaseException as err:                      # noqa: BLE001 - forwarded to the parent
        q.put(("err", rank, err))
    finally:
        try:
            dist.destroy_process_group()
        except Exception:
            pass
        torch.cuda.synchronize() if torch.cuda.is_available() else None


def run_spawned(config, workers: int, transport: str = "p2p", chunk: int = 100,
                timeout: float = 3600.0):
    """run_multiprocess (engine.py:494-528) for the B200 engine: start one
    process per worker (GPU rank % device_count; ranks share GPUs, host-
    synchronised, when there are fewer GPUs than workers), run, and merge the
    results (engine._merge_results semantics).  The first worker error is
    re-raised here."""
    import multiprocessing as mp
    import queue as _queue
    if transport not in TRANSPORTS:
        raise ValueError(f"transport must be one of {TRANSPORTS}")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_spawn_worker, args=(r, workers, port, config, transport, chunk, q),
                         daemon=True)
             for r in range(workers)]
    for p in procs:
        p.start()
    pieces, err, err_at, errs = [], None, 0.0, []
    deadline = time.time() + timeout
    received = 0
    try:
        while received < workers:
            try:
                kind, r, val = q.get(timeout=1.0)
            except _queue.Empty:
                now = time.time()
                if err is not None and now > err_at + 15.0:
                    break                       # the others are stuck behind the failed rank
                dead = [i for i, p in enumerate(procs) if p.exitcode not in (None, 0)]
                if dead and err is None:
                    raise RuntimeError(f"worker(s) {dead} died (exit codes "
                                       f"{[procs[i].exitcode for i in dead]})")
                if now > deadline:
                    raise TimeoutError(f"run_spawned: {len(pieces)} of {workers} workers "
                                       f"finished in {timeout:.0f} s")
                continue
            received += 1
            if kind == "ok":
                pieces.append(val)
            else:
                errs.append((r, val))
                if err is None:
                    err, err_at = val, time.time()
        if err is not None:
            # the failing rank's own error over the ones of the ranks that
            # stopped with it (agree_errors)
            own = [e for _, e in errs if "stopped with it" not in str(e)]
            raise (own or [err])[0]
    finally:
        for p in procs:
            p.join(timeout=0.5 if err is not None else 30)
            if p.is_alive():
                p.terminate()
                p.join(timeout=10)
    return merge_pieces(config, pieces, record_raster=config.record_raster)


def _init_dist():
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        if "MASTER_ADDR" not in os.environ:           # one process, no launcher
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()),
                              RANK="0", WORLD_SIZE="1")
        dist.init_process_group(backend="gloo")
    rank, size = dist.get_rank(), dist.get_world_size()
    return rank, size


def run_multi_gpu(config, workers: int, transport: str = "p2p"):
    """Run under torchrun (WORLD_SIZE == workers): every rank simulates its
    shard; rank 0 returns the merged RunResult, other ranks return None."""
    import torch.distributed as dist
    if int(os.environ.get("WORLD_SIZE", "1")) != workers:
        raise RuntimeError(f"run_multi_gpu(workers={workers}) must run under torchrun "
                           f"--nproc-per-node {workers}; use run_b200 / run_spawned otherwise")
    rank, size = _init_dist()
    group = dist.new_group(backend="gloo")
    nccl_group = dist.new_group(backend="nccl") if transport == "nccl" else None
    piece = _rank_run(config, rank, size, transport, group, nccl_group)
    allp = [None] * size
    dist.all_gather_object(allp, piece, group=group)
    if rank != 0:
        return None
    return merge_pieces(config, allp, record_raster=config.record_raster)


def bench_distributed(args, cfg) -> Optional[dict]:
    """bench.py under torchrun (N > 1) or with --exchange on one GPU (loopback):
    K steps timed with CUDA events on every rank (max over ranks); rank 0
    returns the JSON line."""
    import sys
    import torch
    import torch.distributed as dist
    from . import _lib
    rank, size = _init_dist()
    group = dist.new_group(backend="gloo")
    transport = getattr(args, "transport", "p2p")
    dev_idx, sync = _pick_device(rank, size)
    torch.cuda.set_device(dev_idx)
    loop = size == 1

    def start(tr):
        """Shard + exchange over transport `tr`, warmed up; None (on every
        rank) if any rank's exchange failed during the warm-up."""
        nccl_group = dist.new_group(backend="nccl") if tr == "nccl" else None
        d, ok = None, 1
        try:
            d = DistributedSimulator(cfg, rank, size, device=f"cuda:{dev_idx}", group=group,
                                     nccl_group=nccl_group, transport=tr, sync=sync,
                                     loopback=loop, raster_steps=args.steps + 100)
            settle = int(getattr(args, "settle", 0) or 0)
            if settle:
                d.advance(settle, collect_raster=False)    # onset -> steady operating point
            d.advance(args.warmup)
            if tr == "p2p" and os.environ.get("CC_TEST_P2P_FAIL"):      # tests
                raise _lib.EngineError("step 0: injected peer-exchange failure", 0x400)
        except _lib.EngineError as err:
            if not (err.bits & (0x400 | 0x800)):                         # not the exchange
                raise
            print(f"[bench] rank {rank}: {tr} exchange failed ({err})", file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int64)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if int(flag.item()):
            return d
        if d is not None:
            d.close()
        return None

    # the peer-store exchange is the product path; if its flags do not cross
    # between the GPUs of this box (CC_ERR_XWAIT on some rank during the
    # warm-up) the run falls back to the NCCL slots transport and says so
    ds = start(transport)
    if ds is None and transport == "p2p" and sync == "device":
        transport = "nccl"
        ds = start(transport)
    if ds is None:
        raise RuntimeError("bench: the spike exchange failed on every transport")
    # one warm replay of the chunk graph outside the timed region
    if sync == "device" and args.steps >= ds.chunk:
        ds.advance(ds.chunk)
    c0 = ds.sim.ctl()
    clocks = None
    if rank == 0:
        import bench as _b                               # the repo-root bench module
        clocks = _b.Clocks(dev_idx)
    dist.barrier(group=group)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    ev0.record()
    ds.advance(args.steps, collect_raster=True)
    ev1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    dist.barrier(group=group)
    clk = clocks.stop() if clocks is not None else None
    c1 = ds.sim.ctl()
    xm, sm = ds.measure_exchange(20)
    xs = ds.exchange_stats()
    sent = float(c1.x_sent - c0.x_sent)
    vals = torch.tensor([ev0.elapsed_time(ev1), wall, xm / max(sm, 1e-9),
                         16.0 * sent / args.steps + 8 * max(1, size - 1)], dtype=torch.float64)
    evs = torch.tensor([(c1.rec_events + c1.ext_events) - (c0.rec_events + c0.ext_events),
                        c1.rec_events - c0.rec_events, c1.n_spikes - c0.n_spikes],
                       dtype=torch.float64)
    dist.all_reduce(vals, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(evs, op=dist.ReduceOp.SUM, group=group)
    ds.close()
    line = None
    if rank == 0:
        ms_v, wl = float(vals[0]), float(vals[1])
        total, rec = float(evs[0]), float(evs[1])
        try:
            hbm = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(
                os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"])
        except Exception:
            hbm = 6650.0
        ach = rec / (ms_v / 1e3) * 17 / 1e9 / size          # per GPU
        per_step_bytes = (float(vals[3]) if transport == "p2p"
                          else float(xs.get("per_step_bytes") or 0.0))
        line = {
            "metric": "synaptic events/s (recurrent + external)",
            "value": total / (ms_v / 1e3), "unit": "events/s", "n_gpus": size,
            "steps": args.steps, "warmup": args.warmup,
            "settle_steps": int(getattr(args, "settle", 0) or 0),
            "ms_per_step": ms_v / args.steps,
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
                                      f"{cfg.kernel.kind} lateral decay, "
                                      f"drive {cfg.external.rate_per_synapse_hz} Hz"),
                       "grid": f"{cfg.grid.nx}x{cfg.grid.ny}", "neurons": cfg.grid.n_neurons,
                       "parallelism": (f"column blocks x{size}, one process per GPU, "
                                       f"{transport} exchange ({sync} sync)"
                                       + (", loopback (own spikes through the exchange)"
                                          if loop else "")),
                       "l2": "no flush between steps (per-step working set > 126 MB L2)"},
            "wall_s_per_sim_s": (ms_v / 1e3) / (args.steps * cfg.timestep_ms / 1e3),
            "exchange_fraction": float(vals[2]),
            "exchange": dict(xs, per_rank_bytes_per_step_max=per_step_bytes,
                             what=("p2p: spikes pushed by k_stage into the destinations' "
                                   "windows (16 B each) + one flag word per pair; the "
                                   "fraction is the ingest kernel (wait + log) over the step"
                                   if transport == "p2p" else
                                   "pack + all-to-all of fixed slots + ingest")),
            "roofline": {"bound": "hbm", "kernel": "whole step, per GPU (exchange mode)",
                         "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                         "traffic": None, "bytes_per_event": 17},
            "e2e": {"value": total / wl, "unit": "events/s",
                    "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 12.0 * float(evs[2]) / args.steps,
                    "api": "DistributedSimulator.advance wall (graph replays, per-chunk "
                           "counter checks, cross-rank error agreement and raster copies)"},
            "gpu_launches": (int(ds.sim.L.cc_kernels_per_step(C.byref(ds.sim.shard))) + 1)
            * args.steps,
            "clocks": clk,
        }
    dist.destroy_process_group()
    return line
