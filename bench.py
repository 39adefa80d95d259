"""Benchmark: synaptic events/s of the per-millisecond DPSNN loop on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A "step" is one simulated 1 ms step of the whole network (k_deliver + k_neuron
for every shard).  Workload: N = 1, BASELINE config 1 - 8x8 grid of
1240-neuron columns (79,360 LIF+SFA neurons, ~95 M synapses), Gaussian
lateral decay, calibrated operating point (presets.py); N > 1 (torchrun),
BASELINE config 2 (24x24 exponential, 1.39 G synapses) split over the GPUs
(strong scaling; --scaling weak tiles config 1 once per GPU).  Connectivity and
drive are generated on the device from the seed (bit-exact with the
reference's streams); timing excludes construction like the reference's
normalized cost (metrics.py:114-123).

settle     = the metric is defined at the calibrated steady operating point
             (~7.5 Hz; its CPU side-by-side times a window after
             the onset, "e.g. steps 100-149").  A run starts from V0 ~ U[V_r,
             V_theta) with a synchronous onset burst, so when W < 200 both arms
             first step the network S = 200 - W untimed steps (`settle_steps` in
             the line), then do the W warm-up steps and time exactly K steps.
             With the default W = 200, S = 0.  --settle overrides.
value      = (recurrent + external events in steps S+W .. S+W+K-1) / device time of
             those K steps (CUDA events around warm CUDA-graph replays, one sync).
e2e        = same metric, same steps, through the public step API: wall clock of
             Simulator.advance(K) after advance(W) (the loop run_b200 runs:
             pipelined chunk graphs, per-chunk counter / error checks, raster
             device->host copies).  Recurrent events count at expansion
             (engine.py:366), so a window that includes the onset's first steps
             counts the burst's whole fan-out early; both numbers exclude them.
roofline   = k_deliver against measured HBM bandwidth, 17 B per recurrent
             event; per-kernel times from event-record nodes
             in instrumented graph replays of the same workload: one as timed
             (kernel shares), one with k_stage's tail delivery switched off so
             that k_deliver deposits every arrival (the roofline line).
cpu_baseline = the CPU oracle (numpy port of the reference loop) on the same
             connectivity, 1 core, bounded sample.
--impl reference = the oracle on all host cores (oracle/mp_runner.py), steps
             W .. W+K-1 of a run from t = 0 timed; imports nothing from the
             product package.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SETTLE_MIN = 200              # untimed steps before the timed window (settle + warm-up)
BYTES_PER_EVENT = 17          # 9 B CSR record + 8 B deposit
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def peaks():
    try:
        with open(PEAKS_PATH) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler during the timed region."""

    def __init__(self, gpu: int):
        self.path = tempfile.mktemp(suffix=".csv")
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8 and parts[0].replace(".", "").isdigit():
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


def n_ranks(args) -> int:
    return max(int(os.environ.get("WORLD_SIZE", "1")), args.gpus)


def weak_tiling(n: int):
    """Column blocks of the weak-scaling series: n GPUs -> (a, b) copies of the
    single-GPU grid along x and y, a >= b, a * b = n (1, 2x1, 2x2, 4x2)."""
    b = int(math.isqrt(n))
    while n % b:
        b -= 1
    return n // b, b


def resolve_defaults(args) -> None:
    """N = 1: BASELINE config 1 (the single-B200 config); N > 1: BASELINE
    config 2 split over the GPUs (the config BASELINE states at 1/2/4/8)."""
    if args.config is None:
        args.config = 1 if n_ranks(args) == 1 else 2
    if getattr(args, "settle", None) is None:
        args.settle = max(0, SETTLE_MIN - max(args.warmup, 3))


def workload_grid(args, nx: int, ny: int):
    if getattr(args, "grid", None):
        nx, ny = (int(v) for v in args.grid.lower().split("x"))
    n = n_ranks(args)
    if n > 1 and args.scaling == "weak":
        # per-GPU work fixed: the BASELINE grid once per GPU, tiled (the column
        # partition hands each rank one block of about the single-GPU size)
        a, b = weak_tiling(n)
        nx, ny = nx * a, ny * b
    return nx, ny


def workload(args):
    from dataclasses import replace
    from paper_1803_08833_b200.presets import baseline_config
    cfg = baseline_config(args.config, args.regime, kernel=args.kernel,
                          duration_s=(args.settle + args.warmup + args.steps) / 1000.0,
                          seed=args.seed, drive_hz=args.drive)
    nx, ny = workload_grid(args, cfg.grid.nx, cfg.grid.ny)
    return replace(cfg, grid=replace(cfg.grid, nx=nx, ny=ny))


def scaling_of(args) -> str:
    return "weak" if n_ranks(args) > 1 and args.scaling == "weak" else "strong"


def oracle_net(net):
    """DeviceNetwork -> the oracle's ShardNet (host copy of the same CSR)."""
    from oracle import corticarc_oracle as O
    row_off, tgt, w, d = net.host_csr()
    ln = np.diff(row_off)
    src = np.flatnonzero(ln).astype(np.uint64)
    offs = np.concatenate([row_off[src.astype(np.int64)], [row_off[-1]]]).astype(np.int64)
    return O.ShardNet(src, offs, tgt.astype(np.uint32), d.astype(np.uint16), w, net.checksum,
                      net.n_synapses)


def cpu_oracle_sample(cfg, net, budget_s: float, max_steps: int):
    """Time the numpy oracle (1 core) on the same connectivity from t=0."""
    from oracle import corticarc_oracle as O
    onet = oracle_net(net)
    sim = O.ShardSim(cfg, onet)
    t0 = time.perf_counter()
    steps = 0
    while steps < max_steps and time.perf_counter() - t0 < budget_s:
        inc = [sim.outgoing()] if len(sim.prev_idx) else []
        sim.step(steps, inc)
        steps += 1
    wall = time.perf_counter() - t0
    ev = sim.rec + sim.ext
    return dict(value=ev / wall if wall > 0 else 0.0, unit="events/s", cores=1, kind="port",
                sample=f"oracle/corticarc_oracle.py ShardSim, config {cfg.grid.nx}x{cfg.grid.ny}, "
                       f"steps 0..{steps - 1} from t=0 ({ev} events, {wall:.1f} s, 1 thread)",
                steps=steps, events=int(ev), wall_s=wall)


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference_arm(args):
    """The reference's CPU implementation of the path, timed on the host's
    cores: the numpy oracle of the reference loop (a restatement pinned to the
    reference's own outputs, tests/golden) on k processes with the
    reference's counters-then-payloads exchange over gloo, on connectivity the
    oracle generates on the same k processes.  This process imports nothing
    from the product package (no CUDA library is loaded).  W + K steps from
    t = 0 are run and the last K are timed, like the GPU arm."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.configs import baseline_config as oracle_config
    from oracle.mp_runner import build_global_csr, run_oracle_mp, tiles
    W, K, S = args.warmup, args.steps, args.settle
    probe = oracle_config(args.config, args.regime, kernel=args.kernel)
    nx, ny = workload_grid(args, probe.grid.nx, probe.grid.ny)
    cfg = oracle_config(args.config, args.regime, kernel=args.kernel,
                        duration_s=(S + W + K) / 1000.0, seed=args.seed, drive_hz=args.drive,
                        grid=f"{nx}x{ny}")
    k = next(k for k in range(min(host_threads(), cfg.grid.n_columns), 0, -1)
             if tiles(cfg.grid, k))
    budget = float(os.environ.get("CC_REF_BUDGET_S", "150"))
    row_off, tgt, dly, wgt, gen_s = build_global_csr(cfg, k)
    r = run_oracle_mp(cfg, row_off, tgt, dly, wgt, k, S + W + K, budget, warmup=S + W)
    steps_t = max(1, r["timed_steps"])
    ms = r["timed_wall_s"] * 1000.0 / steps_t
    sample = (f"oracle/mp_runner.py: numpy oracle of the reference loop on {k} processes "
              f"(gloo exchange, counters then payloads), config {cfg.grid.nx}x{cfg.grid.ny}, "
              f"connectivity generated by the oracle on {k} processes ({len(wgt)} synapses, "
              f"{gen_s:.0f} s); steps 0..{r['steps'] - 1} from t=0 run, the last {steps_t} "
              f"timed ({r['timed_events']} events in {r['timed_wall_s']:.1f} s)"
              + ("; stopped by the time budget" if r["steps"] < S + W + K else ""))
    line = {
        "metric": "synaptic events/s (recurrent + external)", "value": r["value"],
        "unit": "events/s", "n_gpus": args.gpus, "steps": steps_t, "warmup": W,
        "settle_steps": S,
        "ms_per_step": ms, "higher_is_better": True, "scaling": scaling_of(args),
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded counter-based RNG; connectivity and drive bit-exact with "
                "the reference streams)",
        "config": config_block(cfg, None, args) | {"synapses": int(len(wgt))},
        "impl": "reference",
        "cpu_baseline": {"value": r["value"], "unit": "events/s", "cores": k, "kind": "port",
                         "sample": sample},
        "e2e": {"value": r["value"], "unit": "events/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s_per_sim_s": ms,
        "exchange_s": r["exchange_s"],
    }
    emit(line)


def config_block(cfg, net, args):
    return {"workload": f"BASELINE config {args.config}: {cfg.grid.nx}x{cfg.grid.ny} columns x "
                        f"{cfg.grid.neurons_per_column} LIF+SFA neurons, {cfg.kernel.kind} "
                        f"lateral decay, {args.regime} operating point",
            "regime": args.regime,
            "grid": f"{cfg.grid.nx}x{cfg.grid.ny}", "neurons": cfg.grid.n_neurons,
            "synapses": int(net.n_synapses) if net is not None else None,
            "kernel": cfg.kernel.kind, "drive_hz": cfg.external.rate_per_synapse_hz,
            "j_inh_mv": cfg.genspec.j_inh_exc, "j_inh_inh_mv": cfg.genspec.j_inh_inh,
            "dt_ms": cfg.timestep_ms, "seed": cfg.seed,
            "l2": "no flush between steps: the per-step working set (CSR rows of the "
                  "spiking sources, delay ring, spike log; 0.86 GB CSR at config 1) is "
                  "scattered over more than the 126 MB L2",
            "parallelism": f"column blocks over {args.gpus} GPU(s)"}


_JSON_OUT = None


def emit(line: dict) -> None:
    """The one JSON line on the real stdout (fd 1 is pointed at stderr while
    the bench runs, so library banners - e.g. NCCL's version line - cannot mix
    into the result stream)."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def _isolate_stdout() -> None:
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def main():
    _isolate_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--settle", type=int, default=None,
                    help="untimed steps from t = 0 before the warm-up (default: what is "
                         "missing to 200 untimed steps, so that the timed window is the "
                         "steady operating point and not the onset burst)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=None,
                    help="BASELINE config (default: 1 on one GPU, 2 on N > 1 GPUs)")
    ap.add_argument("--regime", default="calibrated", choices=["calibrated", "literal", "stress"])
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1: spike exchange (peer stores, or the NCCL slots baseline)")
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--drive", type=float, default=None)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--chunk", type=int, default=100)
    ap.add_argument("--bin-cap", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--instrument-steps", type=int, default=200)
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N > 1: strong = the config's grid split over the GPUs (default), "
                         "weak = the config's grid once per GPU")
    ap.add_argument("--grid", default=None,
                    help="override the config's grid, e.g. 48x24 (one GPU's block of config 4)")
    ap.add_argument("--exchange", action="store_true",
                    help="one GPU, own spikes routed through the peer exchange (loopback)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    resolve_defaults(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1 or args.exchange:
        from paper_1803_08833_b200.distributed import bench_distributed
        line = bench_distributed(args, workload(args))
        if line is not None:
            emit(line)
        return None
    return bench_single(args)


def bench_single(args):
    import torch
    from paper_1803_08833_b200 import _lib
    from paper_1803_08833_b200.network import build_b200
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    cfg = workload(args)
    net = build_b200(cfg)
    capacity = {}
    while True:
        try:
            return _bench_single(args, cfg, net, capacity)
        except _lib.EngineError as err:
            # an expectation-sized buffer overflowed (onset burst of a strongly
            # driven config): measure again from t = 0 with it doubled
            capacity = _lib.grow_capacity(err, {**dict(ovf=1, scratch=1, evrec=1), **capacity})
            if capacity is None:
                raise
            torch.cuda.empty_cache()


def _bench_single(args, cfg, net, capacity):
    import torch
    from paper_1803_08833_b200 import _lib
    from paper_1803_08833_b200.engine import Simulator
    L = _lib.lib()
    dev = torch.device("cuda:0")
    K, W = args.steps, args.warmup
    # timed: steps W .. W+K-1 (like the reference arm), as K / CH replays of a
    # CH-step graph; CH divides K and fits in the warm-up, whose last CH steps
    # are one untimed replay of that same graph (graph upload and first-launch
    # costs stay outside the timed region)
    CH = max(d for d in range(1, min(args.chunk, W, K) + 1) if K % d == 0)
    sim = Simulator(cfg, net, chunk=CH, raster_steps=K + CH, bin_cap=args.bin_cap,
                    capacity=capacity)
    if args.settle:
        sim.advance(args.settle, collect_raster=False)     # onset -> steady operating point
    sim.advance(W - CH)                                    # warm-up (eager + graphs)
    sim.check()
    g_main = sim.capture(CH)
    # the clock sampler starts (and settles) before the warm replay, so that
    # nothing but graph replays sits between the warm-up and the timed region
    clocks = Clocks(0)
    time.sleep(0.3)
    g_main.replay()
    torch.cuda.synchronize(dev)
    sim.t += CH
    c0 = sim.check(collect_raster=False)
    stream = torch.cuda.current_stream(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(K // CH):
        g_main.replay()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    sim.t += K
    c1 = sim.check(collect_raster=False)
    events = (c1.rec_events + c1.ext_events) - (c0.rec_events + c0.ext_events)
    rec = c1.rec_events - c0.rec_events
    spikes = c1.n_spikes - c0.n_spikes
    value = events / (ms / 1e3)

    # instrumented replays: per-kernel durations from event-record nodes.
    # (a) as timed (k_stage's idle warps deliver most of the next step's
    #     delay>=2 events): kernel shares;
    # (b) with that tail delivery switched off (flags 4096), so k_deliver
    #     deposits every arrival: the delivery kernel's roofline.
    NI = min(args.instrument_steps, 1000)

    def instrumented(debug: int):
        timer = C.c_void_p()
        _lib.check(L.cc_timer_create(3 * NI, C.byref(timer)))
        base_flags = sim.shard.flags                   # (routed delivery: no tail delivery)
        sim.shard.flags = base_flags | debug
        g_t = sim.capture(NI, timer=timer)
        sim.shard.flags = base_flags
        ca = sim.check(collect_raster=False)
        g_t.replay()
        torch.cuda.synchronize(dev)
        sim.t += NI
        cb = sim.check(collect_raster=False)
        d_ms = float(np.sum([L.cc_timer_elapsed_ms(timer, 3 * i, 3 * i + 1) for i in range(NI)]))
        n_ms = float(np.sum([L.cc_timer_elapsed_ms(timer, 3 * i + 1, 3 * i + 2)
                             for i in range(NI)]))
        L.cc_timer_destroy(timer)
        return dict(del_ms=d_ms, neu_ms=n_ms, rec=cb.rec_events - ca.rec_events,
                    ev=(cb.rec_events + cb.ext_events) - (ca.rec_events + ca.ext_events),
                    dep=cb.del_events - ca.del_events, tail=cb.tail_events - ca.tail_events)

    run_a = instrumented(0)
    run_b = instrumented(4096)
    del_ms, neu_ms = run_a["del_ms"], run_a["neu_ms"]
    del_i, tail_i = run_a["dep"], run_a["tail"]
    hbm, peak_src = peaks()
    achieved = (run_b["dep"] * BYTES_PER_EVENT / (run_b["del_ms"] / 1e3) / 1e9
                if run_b["del_ms"] > 0 else 0.0)
    traffic = None
    stage_ncu = {}
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            key = f"config{args.config}" + ("" if args.regime == "calibrated" else f"_{args.regime}")
            prof_d = json.load(open(prof)).get(key, {})
            # the roofline kernel is replay (b)'s k_deliver: its ncu DRAM bytes
            traffic = prof_d.get("k_deliver_b", {}).get("dram_bytes_per_launch")
            if traffic is None and "k_route_b" in prof_d:         # routed delivery: both passes
                traffic = (prof_d["k_route_b"]["dram_bytes_per_launch"]
                           + prof_d.get("k_bin_b", {}).get("dram_bytes_per_launch", 0.0))
            stage_ncu = prof_d.get("k_stage", {})
        except Exception:
            traffic = None
    kernels = {
        "k_deliver": {"avg_us": 1e3 * del_ms / NI, "share": del_ms / (del_ms + neu_ms),
                      "events_per_launch": del_i / NI,
                      "bytes_per_launch": del_i * BYTES_PER_EVENT / NI},
        "tail_delivery": {"events_per_step": tail_i / NI,
                          "share_of_arrivals": tail_i / max(1, tail_i + del_i),
                          "what": "step t+1's delay>=2 events deposited by k_stage(t)'s "
                                  "idle warps (inside the k_neuron time)"},
        "k_neuron": {"avg_us": 1e3 * neu_ms / NI, "share": neu_ms / (del_ms + neu_ms),
                     "neuron_events_per_launch": run_a["ev"] / NI},
        "k_deliver_all_arrivals": {"avg_us": 1e3 * run_b["del_ms"] / NI,
                                   "events_per_launch": run_b["dep"] / NI,
                                   "k_neuron_avg_us": 1e3 * run_b["neu_ms"] / NI,
                                   "what": "replay (b): tail delivery off, k_deliver deposits "
                                           "every arrival (roofline kernel)"},
        "instrumented_steps": NI,
        "instrumented_ms_per_step": (del_ms + neu_ms) / NI,
    }
    dsegb = int(sum(x.numel() * x.element_size() for x in net.dseg_cache.values()))
    line = {
        "metric": "synaptic events/s (recurrent + external)",
        "value": value, "unit": "events/s", "n_gpus": 1, "steps": K, "warmup": W,
        "settle_steps": args.settle,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded counter-based RNG (connectivity, Poisson drive), "
                "bit-exact with the reference streams",
        "config": config_block(cfg, net, args),
        "wall_s_per_sim_s": (ms / 1e3) / (K * cfg.timestep_ms / 1e3),
        "recurrent_events_per_s": rec / (ms / 1e3),
        "mean_rate_hz": spikes / (cfg.grid.n_neurons * K * cfg.timestep_ms / 1e3),
        "roofline": {"bound": "hbm", "kernel": "k_deliver", "achieved": achieved, "peak": hbm,
                     "units": "events k_deliver deposited x 17 B / its average launch time, "
                              "replay (b) with every arrival delivered by k_deliver",
                     "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                     "traffic_source": "profiles/ncu_summary.json: dram__bytes_read.sum + "
                                       "dram__bytes_write.sum of one replay-(b) k_deliver "
                                       "launch (ncu --set full)",
                     "peak_source": peak_src,
                     "bytes_per_event": BYTES_PER_EVENT},
        "dominant_kernel": {
            "kernel": "k_plan + k_stage (k_neuron)", "share": neu_ms / (del_ms + neu_ms),
            "inputs_per_s": run_a["ev"] / NI / (neu_ms / NI / 1e3),
            "bound": "fp64 latency / issue: per input 2 exp, 1 expm1, 4 divides, the "
                     "exact ordering and a serial in-order update; 24 resident warps/SM",
            "k_stage_ncu": {k: stage_ncu[k] for k in ("warp_instructions", "ipc_per_sm",
                                                        "warps_active_per_sm",
                                                        "dram_bytes_per_launch", "source")
                            if k in stage_ncu},
            "why_not_the_roofline_kernel": "neither HBM- nor tensor-bound (IPC ~1.5 of 4, "
                                           "DRAM ~0.3 TB/s); the HBM roofline is reported "
                                           "for the delivery kernel (north star)"},
        "step_roofline": {"achieved": rec / (ms / 1e3) * BYTES_PER_EVENT / 1e9, "peak": hbm,
                          "unit": "GB/s",
                          "frac": rec / (ms / 1e3) * BYTES_PER_EVENT / 1e9 / hbm,
                          "definition": "recurrent events/s x 17 B over the whole step "
                                        "(BASELINE.md roofline formula)"},
        "kernels": kernels,
        "gpu_launches": int(L.cc_kernels_per_step(C.byref(sim.shard))) * K,
        "stage_grid": {"warps": int(L.cc_stage_warps(C.byref(sim.shard))),
                       "sublists_per_group": int(sim.shard.n_sub),
                       "what": "k_stage's persistent grid (resident warps, 4 per block)"},
        "clocks": clk,
        "construction_s": net.construction_seconds,
        "bytes_per_synapse_steady": net.steady_bytes / max(1, net.n_synapses),
        "capacity": dict(sim.capacity),
        "memory": {"csr_bytes": int(net.steady_bytes),
                   "delay_segment_table_bytes": int(sum(x.numel() * x.element_size()
                                                        for x in net.dseg_cache.values())),
                   "simulation_buffer_bytes": int(sim.device_bytes),
                   "device_bytes_total": int(net.steady_bytes + sim.device_bytes + dsegb),
                   "bytes_per_synapse_total": (net.steady_bytes + sim.device_bytes + dsegb)
                   / max(1, net.n_synapses),
                   "torch_max_allocated_bytes": int(torch.cuda.max_memory_allocated(dev)),
                   "what": "CSR (9 B/synapse + row index) and every simulation buffer of the "
                           "shard (input lists, ordered-input records, spill staging, spike "
                           "log, state), as allocated; paper's memory study: PAPER.md:698-710"},
        "device_stats": {"max_bin": int(c1.max_bin), "max_events": int(c1.max_events),
                         "overflow_records": int(c1.ovf_total),
                         "spilled_neuron_steps": int(c1.spilled_total),
                         "bin_cap": sim.shard.bin_cap},
    }
    del sim, g_main
    torch.cuda.empty_cache()
    if not args.no_e2e:
        # end to end through the public step API over the same steps as value:
        # a fresh Simulator (run_b200's), W untimed steps, then the wall clock of
        # advance(K) - pipelined chunk graphs, per-chunk counter checks, error
        # checks and the raster's device->host copies (the expansion-time event
        # count of the onset's first steps stays out of both numbers)
        # ... on connectivity uploaded from the host in the reference's own store
        # layout (import_csr: the "given the reference-generated connectivity"
        # entry), when the host copy is small enough to make here: a one-time
        # host->device copy, reported beside the per-step figures
        net2, conn = net, {"source": "generated on the device from the seed (build_b200)",
                           "h2d_bytes_once": 0}
        if net.n_synapses <= int(os.environ.get("CC_E2E_IMPORT_MAX", "300000000")):
            from paper_1803_08833_b200.network import export_csr, import_csr
            store = export_csr(net)
            torch.cuda.synchronize(dev)
            i0 = time.perf_counter()
            net2 = import_csr(cfg, store["sources"], store["offsets"], store["target_local"],
                              store["delay"], store["weight"])
            torch.cuda.synchronize(dev)
            imp_s = time.perf_counter() - i0
            if net2.checksum != net.checksum:
                raise RuntimeError("import_csr: construction checksum differs from the generator's")
            conn = {"source": "import_csr(host store in the reference's IncomingSynapses layout, "
                              "network.py:114-152); checksum equal to the device generator's",
                    "h2d_bytes_once": int(8 * (cfg.grid.n_neurons + 1) + 13 * net.n_synapses
                                          + 4 * len(store["sources"])),
                    "import_seconds": imp_s}
            del store
        sim2 = Simulator(cfg, net2, chunk=min(args.chunk, K), raster_steps=K, capacity=capacity)
        if args.settle:
            sim2.advance(args.settle, collect_raster=False)
        sim2.advance(W)
        ca = sim2.check()
        torch.cuda.synchronize(dev)
        w0 = time.perf_counter()
        sim2.advance(K)
        wall = time.perf_counter() - w0
        cb = sim2.ctl()
        ev = (cb.rec_events + cb.ext_events) - (ca.rec_events + ca.ext_events)
        n_sp = cb.n_spikes - ca.n_spikes
        n_chunks = math.ceil(K / sim2.chunk)
        line["e2e"] = {"value": ev / wall, "unit": "events/s",
                       "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": (12 * n_sp + C.sizeof(_lib.Ctl) * n_chunks) / K,
                       "api": "paper_1803_08833_b200.Simulator.advance(K) wall after advance(W) "
                              "(the step loop of run_b200)",
                       "steps": K, "warmup": W, "connectivity": conn}
        if "import_seconds" in conn:
            line["e2e"]["value_including_import"] = ev / (wall + conn["import_seconds"])
        del sim2, net2
    if not args.no_cpu:
        cb = cpu_oracle_sample(cfg, net, float(os.environ.get("CC_CPU_BUDGET_S", "20")), 10 ** 9)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    emit(line)


if __name__ == "__main__":
    main()
