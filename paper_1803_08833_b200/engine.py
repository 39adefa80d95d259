"""B200 simulation engine: device buffers, CUDA-graph step loop, RunResult.

Drop-in for the reference's simulate entry points (corticarc/engine.py):

    run_b200(config, workers=1) -> RunResult      ~ engine.run / run_multiprocess
    Simulator(config, net).run(n_steps)           ~ run_worker's step loop (:318-394)

Per step two kernels run on one stream (k_deliver, k_neuron; see
csrc/sim_kernels.cu); chunks of steps are captured once into a CUDA graph and
replayed, with a host check of the device counters between chunks (errors are
raised with the step they occurred at, the raster is copied out).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import _lib
from .geometry import grid_totals
from .network import DeviceNetwork, build_b200
from .spec import MemoryBudgetError

__all__ = ["RunResult", "Simulator", "run_b200", "raster_checksum", "estimate_worker_bytes",
           "write_raster"]

MASK64 = (1 << 64) - 1
DOMAIN = 0x636F727469636172
# shards of at least this many neurons deliver with 16 lanes per spike (see Shard setup)
DEL_WIDE_NEURONS = 2_000_000
ROUTED_DEFAULT = True          # routed delivery in the high-rate regime (Simulator)
L1_TARGET_REGIONS = 1024       # routed delivery: regions grow from 1024 neurons to stay below this
P_INIT_STATE, P_EXTERNAL, P_EXTERNAL_TIME = 4, 5, 7


def _sm(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def _h2(seed: int, purpose: int) -> int:
    """First two links of counter_uniforms' splitmix chain (rng.py:85-86)."""
    return _sm(_sm((seed & MASK64) ^ DOMAIN) ^ purpose)


def raster_checksum(gids, times) -> int:
    """network.py:91-97 (order independent)."""
    if len(gids) == 0:
        return 0
    u = np.uint64
    lo = np.asarray(gids, dtype=u)
    hi = np.asarray(times, dtype=np.float64).view(u)
    with np.errstate(over="ignore"):
        def sm(x):
            z = x + u(0x9E3779B97F4A7C15)
            z = (z ^ (z >> u(30))) * u(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> u(27))) * u(0x94D049BB133111EB)
            return z ^ (z >> u(31))
        return int(np.sum(sm(lo ^ sm(hi)), dtype=u))


def write_raster(path, gids, times_ms) -> None:
    """`time_ms<TAB>neuron_gid` lines in ascending (time, gid) order - the
    reference's raster file format (engine.py:531-536), byte for byte."""
    gids = np.asarray(gids)
    times_ms = np.asarray(times_ms, dtype=np.float64)
    order = np.lexsort((gids, times_ms))
    with open(path, "w") as fh:
        fh.writelines(f"{t:.9f}\t{int(g)}\n" for t, g in zip(times_ms[order], gids[order]))


def estimate_worker_bytes(config, workers: int) -> int:
    """The reference's pre-allocation estimate (engine.py:278-283)."""
    local, remote = grid_totals(config.kernel, config.grid)
    syn = (local + remote) / workers
    state = config.grid.n_neurons / workers * 13 * 8
    return int(syn * 32 + state)


@dataclass
class RunResult:
    """Same fields and meanings as the reference RunResult (engine.py:251-275)."""
    config: object
    worker_count: int
    raster_gids: np.ndarray
    raster_times: np.ndarray
    n_spikes: int
    recurrent_events: int
    external_events: int
    recurrent_synapses: int
    construction_checksum: int
    raster_checksum: int
    construction_seconds: float
    sim_seconds_wall: float
    substep_seconds: Dict[str, float]
    steady_bytes_per_worker: List[int]
    peak_bytes_per_worker: List[int]
    workers: list = field(default_factory=list)
    probe_state: Optional[np.ndarray] = None      # [steps, P, 4]
    probe_v_end: Optional[np.ndarray] = None      # [steps, P]
    device_stats: dict = field(default_factory=dict)

    @property
    def mean_rate_hz(self) -> float:
        denom = self.config.grid.n_neurons * self.config.duration_s
        return self.n_spikes / denom if denom else 0.0


def _pop(p) -> _lib.Pop:
    q = _lib.Pop()
    q.tau_m, q.tau_c, q.E = p.tau_m, p.tau_c, p.E
    q.V_theta, q.V_r, q.tau_arp, q.alpha_c = p.V_theta, p.V_r, p.tau_arp, p.alpha_c
    q.sfa = p.g_c / p.C_m
    q.k1 = p.tau_c - p.tau_m
    q.k2 = p.tau_m * p.tau_c
    q.r_tau_m, q.r_tau_c, q.r_k2 = 1.0 / q.tau_m, 1.0 / q.tau_c, 1.0 / q.k2
    return q


def default_bin_cap(cfg) -> int:
    """Records per (slot, 32-neuron group) list: 32 x (~3x the inputs an
    interior neuron receives per step at 20 Hz plus headroom), a power of two
    in [2048, 16384]; rarer bursts go through the grouped overflow list."""
    from .geometry import expected_fanout
    want = 32 * (3.0 * expected_fanout(cfg.kernel, cfg.grid) * 0.02 * cfg.timestep_ms + 32)
    return int(min(16384, max(2048, 1 << int(math.ceil(math.log2(want))))))


def _spikes_per_step_bound(cfg) -> int:
    taus = [cfg.exc_params.tau_arp, cfg.inh_params.tau_arp]
    if min(taus) <= 0:
        return 8
    return int(math.floor(cfg.timestep_ms / min(taus))) + 1


class Simulator:
    """One shard's device state and step loop."""

    TIMED_STEPS = 10          # steps of the sampled chunk carrying event-record nodes

    def __init__(self, cfg, net: DeviceNetwork, *, probes=None, probe_steps: int = 0,
                 bin_cap: Optional[int] = None, chunk: int = 100,
                 use_graphs: bool = True, direct_log: Optional[bool] = None,
                 remote=None,
                 raster_steps: Optional[int] = None, substeps: bool = False, device=None,
                 capacity=None, sublists: Optional[int] = None,
                 routed: Optional[bool] = None):
        import torch
        self.L = _lib.lib()
        self.torch = torch
        self.cfg, self.net = cfg, net
        self.dev = torch.device(device or net.row_off.device)
        dev = self.dev
        grid = cfg.grid
        n = grid.neurons_per_column
        owned = net.owned_columns
        gids = (owned[:, None].astype(np.int64) * n + np.arange(n)[None, :]).ravel()
        self.gids = gids
        n_local = len(gids)
        D = cfg.d_max
        bound = _spikes_per_step_bound(cfg)
        step_cap = default_bin_cap(cfg)        # records per group and step
        # Input sub-lists per group (by target lane range).  One list per group
        # has the fewest reservation atomics and is best while a group's inputs
        # fit two or three work items; at high rates (a group takes ten and
        # more items, each of which would read the whole list) 8 sub-lists let
        # an item read only its own lanes' records: -19 % per step at the 37 Hz
        # stress point, +7 % / +18 % at configs 1 / 3.  The rate is not known
        # before the run: a drive of >= 10 external events per neuron and step
        # is taken as the mark of the high-rate regime (CC_SUBLISTS overrides).
        if sublists is None:
            sublists = int(os.environ.get("CC_SUBLISTS", "0")) or \
                (8 if cfg.external.mean_per_step(cfg.timestep_ms) >= 10.0 else 1)
        n_sub = int(sublists)
        cnt_stride = _lib.cnt_stride(n_sub)
        self.n_sub = n_sub
        if bin_cap is None:                    # per sub-list: 2x an even share
            bin_cap = max(256, 2 * step_cap // n_sub)
        n_groups = (n_local + 31) // 32
        # list stride bin_cap + bin_pad records: with a power-of-two stride the
        # appends of one step (same small offsets in thousands of lists) land in
        # few L2 slices / DRAM channels
        bin_pad = int(os.environ.get("CC_BIN_PAD", "0"))
        self.chunk = max(1, int(chunk))
        self.use_graphs = use_graphs
        direct = (net.size == 1) if direct_log is None else direct_log
        T = torch
        i32, i64, f64 = T.int32, T.int64, T.float64
        spk_cap = max(1, min(net.nonempty_rows(), grid.n_neurons) * bound)
        spk_cap = 1 << (spk_cap - 1).bit_length()     # power of two: ref -> slot is a shift
        if spk_cap * (D + 1) >= 2 ** 32:
            raise MemoryBudgetError("spike log references exceed 32 bits")
        # capacity = {"ovf", "scratch", "evrec"} multipliers of the buffers sized
        # by expectation rather than by a hard bound (overflow list, spill staging,
        # ordered-input records): run_b200 re-runs from t = 0 with the one that
        # overflowed doubled (onset bursts fail within the first steps)
        self.capacity = cap = {"ovf": 1, "scratch": 1, "evrec": 1, **(capacity or {})}
        ovf_cap = max(4096, n_local * 8) * cap["ovf"]
        if spk_cap * (D + 1) >= 2 ** 27:
            raise MemoryBudgetError("spike log references exceed the 27 bits of a ring record")
        seg_stride = (D + 1 + 7) // 8 * 8
        dseg = net.delay_segments(D, seg_stride)
        raster_cap = max(1024, n_local * bound * max(self.chunk, raster_steps or 0))
        # spill staging (neuron-steps with > NEURON_WCAP inputs, all of one step)
        per_neuron = int(os.environ.get("CC_SCRATCH_PER_NEURON", "64"))
        scratch_cap = max(1 << 16, n_local * per_neuron) * cap["scratch"]
        # ordered-input records of one step: the expected list capacity of a step,
        # the overflow list and every neuron's Poisson budget (beyond it the
        # step fails with "event staging scratch exhausted")
        lam = cfg.external.mean_per_step(cfg.timestep_ms)
        ext_m = int(math.ceil(lam + 12.0 * math.sqrt(lam))) + 20 if lam > 0 else 0
        evrec_cap = (n_groups * step_cap + n_local * ext_m) * cap["evrec"] + ovf_cap
        self.buf = dict(
            gid=T.from_numpy(gids.astype(np.uint32).view(np.int32)).to(dev),
            state=T.zeros((n_local, 4), dtype=f64, device=dev),
            bin_cnt=T.zeros(2 * n_groups * n_sub * cnt_stride, dtype=i32,
                            device=dev),
            bin_rec=T.empty((2, n_groups, n_sub, bin_cap + bin_pad), dtype=i64,
                            device=dev),
            grp_n=T.zeros(n_groups, dtype=i32, device=dev),
            grp_sub=T.zeros((n_groups, n_sub), dtype=i32, device=dev),
            ovf_rec=T.empty((2, ovf_cap, 4), dtype=i32, device=dev),
            ovf_cnt=T.zeros(2, dtype=i32, device=dev),
            ovf_sorted=T.empty((ovf_cap, 4), dtype=i32, device=dev),
            ovf_off=T.zeros(n_groups, dtype=i32, device=dev),
            ovf_fill=T.zeros(n_groups, dtype=i32, device=dev),
            log_t=T.empty((D + 1, spk_cap), dtype=f64, device=dev),
            log_gid=T.empty((D + 1, spk_cap), dtype=i32, device=dev),
            log_ctr=T.zeros(D + 1, dtype=i64, device=dev),
            log_len=T.zeros(D + 1, dtype=i64, device=dev),
            log_r0=T.empty((D + 1, spk_cap), dtype=i64, device=dev),
            log_dseg=T.empty((D + 1, spk_cap, seg_stride), dtype=T.int16, device=dev),
            raster_gid=T.empty(raster_cap, dtype=i32, device=dev),
            raster_t=T.empty(raster_cap, dtype=f64, device=dev),
            out_gid=T.empty(max(1, n_local * bound), dtype=i32, device=dev),
            out_t=T.empty(max(1, n_local * bound), dtype=f64, device=dev),
            scratch=T.empty((scratch_cap, 14), dtype=T.float32, device=dev),   # 56 B/event
            probe_map=T.full((n_local,), -1, dtype=i32, device=dev),
            ev_n=T.zeros(n_local, dtype=i32, device=dev),
            ev_nr=T.zeros(n_local, dtype=i32, device=dev),
            evrec=T.empty((evrec_cap, 6), dtype=f64, device=dev),          # 48 B/input
            ev_off=T.zeros(n_local, dtype=i32, device=dev),
            grp_items=T.zeros(n_groups, dtype=i32, device=dev),
            grp_done=T.zeros(n_groups, dtype=i32, device=dev),
            rounds=T.zeros(_lib.ITEM_CLASSES * ((n_local + 31) // 32) * 32 * 2, dtype=i32,
                           device=dev),

            ctl=T.zeros(C.sizeof(_lib.Ctl) // 8, dtype=i64, device=dev),
            tailc=T.zeros(256, dtype=i32, device=dev),
        )
        # Routed (two-pass) delivery (csrc/route_kernels.cuh): the step's arrivals
        # go first to one record array per region of 2^rb consecutive neurons,
        # then from there to the input lists, both passes sorting tiles in shared
        # memory and copying whole runs instead of one scattered store per event.
        # It pays at the paper's event volumes (the high-rate regime, where the
        # sub-lists are on as well); below, k_deliver's single pass is faster.
        # CC_ROUTED=0/1 overrides.
        if routed is None:
            env = os.environ.get("CC_ROUTED", "")
            routed = bool(int(env)) if env else ROUTED_DEFAULT and n_sub > 1
        self.routed = bool(routed)
        if self.routed:
            rb_max = 15 - (n_sub.bit_length() - 1)       # lists per region <= CC_L1_MAX_LISTS
            rb = int(os.environ.get("CC_L1_RB", "0")) or 11
            while rb < rb_max and -(-n_local // (1 << rb)) > L1_TARGET_REGIONS:
                rb += 1
            n_regions = -(-n_local // (1 << rb))
            if rb > rb_max or n_regions > _lib.L1_MAX_REGIONS:
                raise MemoryBudgetError(f"routed delivery: {n_local} neurons need more than "
                                        f"{_lib.L1_MAX_REGIONS} regions")
            # records per region and step: half the list capacity of its groups
            l1_cap = (int(os.environ.get("CC_L1_CAP", "0")) or
                      max(4096, (1 << (rb - 5)) * step_cap // 2)) * cap["ovf"]
            self.buf.update(
                l1_cnt=T.zeros(2 * n_regions * _lib.L1_STRIDE, dtype=i32, device=dev),
                l1_ref=T.empty((n_regions, l1_cap), dtype=i32, device=dev),
                l1_w=T.empty((n_regions, l1_cap), dtype=i32, device=dev),
                l1_tgt=T.empty((n_regions, l1_cap), dtype=T.int16, device=dev))
            # per-neuron record counts from k_bin: the planning pass then does
            # not read the lists' records (CC_L1_NCNT=0: it counts them itself)
            if rb <= _lib.L1_NCNT_MAX_RB and int(os.environ.get("CC_L1_NCNT", "1")):
                self.buf["l1_ncnt"] = T.zeros(2 * n_groups * 32, dtype=i32, device=dev)
        self.probes = None if probes is None else np.asarray(probes, np.int64)
        n_probe = 0 if self.probes is None else len(self.probes)
        if n_probe:
            self.buf["probe_map"][T.from_numpy(self.probes).to(dev)] = \
                T.arange(n_probe, dtype=i32, device=dev)
        self.buf["probe_out"] = T.zeros((max(1, probe_steps), max(1, n_probe), 5), dtype=f64,
                                        device=dev)
        self.buf["ctl"][6] = (1 << 63) - 1          # error_step = LLONG_MAX
        b = self.buf
        sh = _lib.Shard()
        sh.n_local, sh.n_col, sh.n_exc_col = n_local, n, grid.n_excitatory_per_column
        sh.d_max, sh.bin_cap, sh.log_slots = D, bin_cap, D + 1
        sh.n_groups, sh.bin_pad = n_groups, bin_pad
        sh.n_sub = n_sub
        sh.flags = int(os.environ.get("CC_FLAGS", "0"))    # CC_FLAG_* (measurement / tests)
        if self.routed:
            sh.l1_rb, sh.n_regions, sh.l1_cap = rb, n_regions, l1_cap
            for k in ("l1_cnt", "l1_ref", "l1_w", "l1_tgt"):
                setattr(sh, k, b[k].data_ptr())
            if "l1_ncnt" in b:
                sh.l1_ncnt = b["l1_ncnt"].data_ptr()
            # the tail delivery's scattered deposits are what this mode avoids
            sh.flags |= _lib.FLAG_NO_TAIL_DELIVERY
        sh.spk_cap, sh.seg_stride = spk_cap, seg_stride
        # delivery lanes per spike: 16 on shards of >= 2 M neurons (config 3 gaussian: k_deliver
        # 448 -> 367 us, step -3.3 %), 8 below (configs 1, 2 and the config-4 GPU block: 16 lanes are ~1 % slower);
        # CC_DEL_LPS overrides for experiments (profiles/r01l_delivery_sweep.md)
        # (k_route, whose tile staging is indifferent to the run structure: 16 lanes
        # - config 2 stress point, delivery 779 -> 752 us)
        lps = int(os.environ.get("CC_DEL_LPS", "0")) or (
            16 if n_local >= DEL_WIDE_NEURONS or self.routed else 8)
        if lps not in (8, 16):
            raise ValueError(f"CC_DEL_LPS must be 8 or 16, got {lps}")
        sh.del_lps_log2 = lps.bit_length() - 1
        sh.ovf_cap, sh.raster_cap = ovf_cap, raster_cap
        sh.scratch_cap, sh.n_rows = scratch_cap, grid.n_neurons
        sh.evrec_cap = evrec_cap
        sh.round_cap = ((n_local + 31) // 32) * 32
        sh.out_cap = b["out_gid"].numel()
        lam = cfg.external.mean_per_step(cfg.timestep_ms)
        if lam > 0:
            sh.ext_budget = int(math.ceil(lam + 12.0 * math.sqrt(lam))) + 20
            sh.ext_thresh = math.exp(-lam)
        else:
            sh.ext_budget, sh.ext_thresh = 0, 1.0
        sh.n_probe = n_probe
        sh.direct_log = 1 if direct else 0
        # exchange with local logging: neurons that also have rows on other
        # shards go to the out-list as well (uint8 tensor, one entry per neuron)
        self.remote = None if remote is None else \
            torch.as_tensor(np.asarray(remote, dtype=np.uint8), device=dev)
        sh.remote = self.remote.data_ptr() if self.remote is not None else None
        sh.h2_ext = _h2(cfg.seed, P_EXTERNAL)
        sh.h2_time = _h2(cfg.seed, P_EXTERNAL_TIME)
        sh.h2_init = _h2(cfg.seed, P_INIT_STATE)
        sh.dt = cfg.timestep_ms
        sh.ext_weight = cfg.external.weight_mv
        sh.pop[0] = _pop(cfg.exc_params)
        sh.pop[1] = _pop(cfg.inh_params)
        sh.gid, sh.state = b["gid"].data_ptr(), b["state"].data_ptr()
        sh.row_off, sh.syn_tgt = net.row_off.data_ptr(), net.syn_tgt.data_ptr()
        sh.dseg = dseg.data_ptr()
        sh.syn_w, sh.syn_d = net.syn_w.data_ptr(), net.syn_d.data_ptr()
        for k in ("bin_cnt", "bin_rec", "grp_n", "grp_sub", "ovf_rec", "ovf_cnt", "ovf_sorted", "ovf_off",
                  "ovf_fill", "log_t", "log_gid", "log_ctr", "log_len", "log_r0", "log_dseg",
                  "raster_gid", "raster_t", "out_gid", "out_t", "scratch",
                  "ev_n", "ev_nr", "rounds", "evrec", "ev_off", "grp_items", "grp_done",
                  "probe_map", "probe_out", "ctl", "tailc"):
            setattr(sh, k, b[k].data_ptr())
        sh.probe_steps = b["probe_out"].shape[0] if n_probe else 0
        self.shard = sh
        self.n_local = n_local
        # per-kernel device time of graph-replayed chunks (RunResult.substep_seconds)
        self.substeps = substeps
        self._timer = None
        self.kernel_ms = dict(deliver=0.0, neuron=0.0, steps=0)
        self.t = 0
        self.raster_g: List[np.ndarray] = []
        self.raster_t: List[np.ndarray] = []
        self.device_bytes = sum(x.numel() * x.element_size() for x in b.values())
        stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(self.L.cc_init_state(C.byref(sh), stream), "cc_init_state")
        _lib.check(self.L.cc_prepare(), "cc_prepare")
        self._graph_t = None
        self._graphs = [None, None]
        if use_graphs:
            # Pipelined chunks (advance): two graphs alternate between two raster
            # buffers; each ends by snapshotting the counters and emptying the
            # raster, so the host drains chunk k while chunk k+1 runs.
            rc2 = max(1024, n_local * bound * self.chunk)
            b["raster_gid2"] = T.empty(rc2, dtype=i32, device=dev)
            b["raster_t2"] = T.empty(rc2, dtype=f64, device=dev)
            b["snap"] = T.zeros((2, b["ctl"].numel()), dtype=i64, device=dev)
            sh2 = _lib.Shard.from_buffer_copy(sh)
            sh2.raster_gid, sh2.raster_t = b["raster_gid2"].data_ptr(), b["raster_t2"].data_ptr()
            sh2.raster_cap = rc2
            self.shards = [sh, sh2]
            self._rasters = [(b["raster_gid"], b["raster_t"]), (b["raster_gid2"], b["raster_t2"])]
            self._snap_host = T.empty((2, b["ctl"].numel()), dtype=i64, pin_memory=True)
            self._copy_stream = T.cuda.Stream(dev)
            self._copied = [None, None]
            self.device_bytes = sum(x.numel() * x.element_size() for x in b.values())
            # capture once, outside any timed region
            for i in range(2):
                self._capture(self.chunk, torch.cuda.Stream(dev), slot=i)
            if substeps:
                self._capture(self.chunk, torch.cuda.Stream(dev), timed=True, slot=0)

    # ------------------------------------------------------------------ steps
    def _launch_step(self, stream) -> None:
        _lib.check(self.L.cc_deliver(C.byref(self.shard), stream), "cc_deliver")
        _lib.check(self.L.cc_neuron_step(C.byref(self.shard), stream), "cc_neuron_step")

    def kernels_per_step(self) -> int:
        """Kernels cc_deliver + cc_neuron_step launch per step for this shard."""
        return int(self.L.cc_kernels_per_step(C.byref(self.shard)))

    def ctl(self) -> _lib.Ctl:
        raw = self.buf["ctl"].cpu().numpy().tobytes()
        return _lib.Ctl.from_buffer_copy(raw)

    def check(self, collect_raster: bool = True) -> _lib.Ctl:
        """Synchronise, raise on device errors, drain the raster buffer."""
        self.torch.cuda.synchronize(self.dev)
        c = self.ctl()
        if c.error_bits:
            raise _lib.EngineError(f"step {c.error_step}: {_lib.decode_errors(c.error_bits)}",
                                   int(c.error_bits))
        if c.raster_n:
            n = int(c.raster_n)
            if collect_raster:
                self.raster_g.append(self.buf["raster_gid"][:n].cpu().numpy().view(np.uint32)
                                     .astype(np.uint64))
                self.raster_t.append(self.buf["raster_t"][:n].cpu().numpy())
            self.buf["ctl"][4] = 0
        return c

    def _capture(self, steps: int, stream_obj, timed: bool = False, slot: int = 0):
        """The chunk graph of pipeline slot `slot` (its raster buffer), ending
        with the counter snapshot and the raster reset; timed: event-record
        nodes before and after each step's delivery (2 per step + 1 at the
        end) on its first TIMED_STEPS steps - one sampled chunk only, since the
        nodes cost ~9 % of a timed step."""
        torch = self.torch
        if timed and self._timer is None:
            self._timer = C.c_void_p()
            _lib.check(self.L.cc_timer_create(2 * steps + 1, C.byref(self._timer)))
        tm = self._timer if timed else None
        sh = self.shards[slot]
        g = torch.cuda.CUDAGraph()
        n_timed = min(steps, self.TIMED_STEPS)
        with torch.cuda.graph(g, stream=stream_obj):
            s = torch.cuda.current_stream(self.dev).cuda_stream
            for i in range(steps):
                if tm is not None and i < n_timed:
                    _lib.check(self.L.cc_timer_record(tm, 2 * i, s))
                _lib.check(self.L.cc_deliver(C.byref(sh), s), "cc_deliver")
                if tm is not None and i < n_timed:
                    _lib.check(self.L.cc_timer_record(tm, 2 * i + 1, s))
                _lib.check(self.L.cc_neuron_step(C.byref(sh), s), "cc_neuron_step")
                if tm is not None and i == n_timed - 1:
                    _lib.check(self.L.cc_timer_record(tm, 2 * n_timed, s))
            self.buf["snap"][slot].copy_(self.buf["ctl"])
            self.buf["ctl"][4].zero_()                       # raster_n
        if timed:
            self._graph_t = g
        else:
            self._graphs[slot] = g
        return g

    def _read_substeps(self, steps: int) -> None:
        steps = min(steps, self.TIMED_STEPS)
        el = self.L.cc_timer_elapsed_ms
        d = sum(el(self._timer, 2 * i, 2 * i + 1) for i in range(steps))
        n = sum(el(self._timer, 2 * i + 1, 2 * i + 2) for i in range(steps))
        self.kernel_ms["deliver"] += d
        self.kernel_ms["neuron"] += n
        self.kernel_ms["steps"] += steps

    def __del__(self):
        try:
            if self._timer is not None:
                self.L.cc_timer_destroy(self._timer)
        except Exception:
            pass

    def capture(self, steps: int, timer=None, timer_base: int = 0):
        """A CUDA graph of `steps` steps; with a timer (cc_timer_create handle)
        event-record nodes bracket every kernel: events timer_base + 3*i,
        +1, +2 around k_deliver / k_neuron of step i."""
        torch = self.torch
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=torch.cuda.Stream(self.dev)):
            s = torch.cuda.current_stream(self.dev).cuda_stream
            for i in range(steps):
                if timer is not None:
                    _lib.check(self.L.cc_timer_record(timer, timer_base + 3 * i, s))
                _lib.check(self.L.cc_deliver(C.byref(self.shard), s), "cc_deliver")
                if timer is not None:
                    _lib.check(self.L.cc_timer_record(timer, timer_base + 3 * i + 1, s))
                _lib.check(self.L.cc_neuron_step(C.byref(self.shard), s), "cc_neuron_step")
                if timer is not None:
                    _lib.check(self.L.cc_timer_record(timer, timer_base + 3 * i + 2, s))
        return g

    def advance(self, n_steps: int, collect_raster: bool = True) -> None:
        """Run n_steps more steps: full chunks as pipelined graph replays, the
        remainder eagerly."""
        full = n_steps // self.chunk if self.use_graphs else 0
        if full:
            self._advance_graphs(full, collect_raster)
        rest = n_steps - full * self.chunk
        s = self.torch.cuda.current_stream(self.dev).cuda_stream
        while rest > 0:
            k = min(self.chunk, rest)
            for _ in range(k):
                self._launch_step(s)
            self.t += k
            rest -= k
            self.check(collect_raster)

    def _advance_graphs(self, n_chunks: int, collect_raster: bool) -> None:
        """Chunk k runs graph k % 2; the host drains chunk k (counters, errors,
        raster) on a copy stream while chunk k + 1 runs, and chunk k + 2 waits
        for that drain before reusing the raster buffer."""
        torch = self.torch
        main = torch.cuda.current_stream(self.dev)
        pend = []
        for k in range(n_chunks):
            i = k & 1
            timed = k == 0 and self._graph_t is not None and not self.kernel_ms["steps"]
            if self._copied[i] is not None:
                main.wait_event(self._copied[i])
            (self._graph_t if timed else self._graphs[i]).replay()
            ev = torch.cuda.Event()
            ev.record(main)
            self.t += self.chunk
            pend.append((i, ev, timed))
            if len(pend) == 2:
                self._drain(*pend.pop(0), collect_raster)
        while pend:
            self._drain(*pend.pop(0), collect_raster)

    def _drain(self, i: int, ev, timed: bool, collect_raster: bool) -> None:
        torch = self.torch
        cs = self._copy_stream
        cs.wait_event(ev)
        with torch.cuda.stream(cs):
            self._snap_host[i].copy_(self.buf["snap"][i], non_blocking=True)
        cs.synchronize()
        c = _lib.Ctl.from_buffer_copy(self._snap_host[i].numpy().tobytes())
        if c.error_bits:
            raise _lib.EngineError(f"step {c.error_step}: {_lib.decode_errors(c.error_bits)}",
                                   int(c.error_bits))
        n = int(c.raster_n)
        if n and collect_raster:
            rg, rt = self._rasters[i]
            with torch.cuda.stream(cs):
                self.raster_g.append(rg[:n].cpu().numpy().view(np.uint32).astype(np.uint64))
                self.raster_t.append(rt[:n].cpu().numpy())
        done = torch.cuda.Event()
        done.record(cs)
        self._copied[i] = done
        if timed:
            self._read_substeps(self.chunk)

    def raster(self):
        g = np.concatenate(self.raster_g) if self.raster_g else np.empty(0, np.uint64)
        t = np.concatenate(self.raster_t) if self.raster_t else np.empty(0)
        o = np.lexsort((g, t))
        return g[o], t[o]

    def probe_results(self, steps: int):
        if self.probes is None:
            return None, None
        p = self.buf["probe_out"][:steps].cpu().numpy()
        return p[:, :, :4].copy(), p[:, :, 4].copy()


def _substeps(sim, n_steps: int, wall: float) -> dict:
    """RunResult.substep_seconds (engine.py:251-275 keys): expand = delivery
    kernel, integrate = neuron step (Poisson drive, sort and update are one
    kernel pair, so external is folded into it), deliver = spike exchange
    (none on one GPU).  The simulation wall is apportioned by the kernel-time
    shares measured with CUDA event nodes on one graph chunk; without a timed
    chunk, the wall goes to integrate."""
    km = sim.kernel_ms
    tot = km["deliver"] + km["neuron"]
    if not km["steps"] or tot <= 0:
        return {"deliver": 0.0, "expand": 0.0, "external": 0.0, "integrate": wall}
    return {"deliver": 0.0, "expand": wall * km["deliver"] / tot, "external": 0.0,
            "integrate": wall * km["neuron"] / tot}


def run_b200(config, workers: int = 1, *, net: Optional[DeviceNetwork] = None, probes=None,
             steps: Optional[int] = None, bin_cap: Optional[int] = None, chunk: int = 100,
             use_graphs: bool = True, device=None) -> RunResult:
    """Build (unless `net` is given) and simulate on one B200; same result
    contract as corticarc.engine.run (engine.py:449-480).  workers > 1 runs
    one process per GPU (see paper_1803_08833_b200.distributed)."""
    import torch
    if workers != 1:
        from .distributed import run_multi_gpu, run_spawned
        est = estimate_worker_bytes(config, workers)
        if est > config.memory_budget_bytes:
            raise MemoryBudgetError(
                f"estimated {est / 1e9:.2f} GB per worker exceeds the "
                f"{config.memory_budget_bytes / 1e9:.2f} GB budget")
        transport = os.environ.get("CC_TRANSPORT", "p2p")
        if int(os.environ.get("WORLD_SIZE", "1")) == workers:      # under torchrun
            return run_multi_gpu(config, workers, transport=transport)
        return run_spawned(config, workers, transport=transport, chunk=chunk)
    est = estimate_worker_bytes(config, workers)
    if est > config.memory_budget_bytes:
        raise MemoryBudgetError(
            f"estimated {est / 1e9:.2f} GB per worker exceeds the "
            f"{config.memory_budget_bytes / 1e9:.2f} GB budget")
    _lib.lib()
    if net is None:
        net = build_b200(config, device=device)
    n_steps = config.n_steps if steps is None else steps
    capacity = None
    while True:
        sim = Simulator(config, net, probes=probes, probe_steps=n_steps, bin_cap=bin_cap,
                        chunk=chunk, use_graphs=use_graphs, substeps=True, device=device,
                        capacity=capacity)
        torch.cuda.synchronize(sim.dev)
        t0 = time.perf_counter()
        try:
            sim.advance(n_steps, collect_raster=getattr(config, "record_raster", True))
        except _lib.EngineError as err:
            # an expectation-sized buffer overflowed (e.g. a synchronous onset
            # burst): the run is deterministic, so re-run it from t = 0 with that
            # buffer doubled (up to 32x); hard bounds and protocol errors raise
            capacity = _lib.grow_capacity(err, sim.capacity)
            if capacity is None:
                raise
            del sim
            torch.cuda.empty_cache()
            continue
        break
    wall = time.perf_counter() - t0
    c = sim.ctl()
    g, t = sim.raster()
    ps, pv = sim.probe_results(n_steps)
    return RunResult(
        config=config, worker_count=1, raster_gids=g, raster_times=t,
        n_spikes=int(c.n_spikes), recurrent_events=int(c.rec_events),
        external_events=int(c.ext_events), recurrent_synapses=net.n_synapses,
        construction_checksum=net.checksum, raster_checksum=raster_checksum(g, t),
        construction_seconds=net.construction_seconds, sim_seconds_wall=wall,
        substep_seconds=_substeps(sim, n_steps, wall),
        steady_bytes_per_worker=[net.steady_bytes], peak_bytes_per_worker=[net.peak_bytes],
        probe_state=ps, probe_v_end=pv,
        device_stats=dict(max_bin=int(c.max_bin), max_events=int(c.max_events),
                          spilled=int(c.spilled_total), overflow=int(c.ovf_total),
                          bin_cap=sim.shard.bin_cap, device_bytes=sim.device_bytes,
                          capacity=dict(sim.capacity)))
