"""Full-length parity at a BASELINE config: the CUDA engine against the CPU
oracle (numpy port of the reference loop, pinned to the reference's own
fixtures) on the same connectivity, over the config's whole duration.

    python tools/long_parity.py [CONFIG] [DURATION_S] [SHARDS] [REGIME] [GRID]

GRID (e.g. 48x24: one GPU's block of config 4) replaces the config's grid.

SHARDS > 1 runs the multi-shard path (distributed.run_local_shards: W column
blocks with their own generator, spike exchange by device copies) on one GPU.

Writes gpurun_out/long_parity_config<N>.json (committed under profiles/)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1803_08833_b200.engine import run_b200  # noqa: E402
from paper_1803_08833_b200.network import build_b200  # noqa: E402
from paper_1803_08833_b200.presets import baseline_config  # noqa: E402
from oracle.mp_runner import run_oracle_mp  # noqa: E402


def main():
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    dur = float(sys.argv[2]) if len(sys.argv) > 2 and float(sys.argv[2]) > 0 else None
    shards = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    regime = sys.argv[4] if len(sys.argv) > 4 else "calibrated"
    cfg = baseline_config(idx, regime, duration_s=dur)
    grid = sys.argv[5] if len(sys.argv) > 5 else ""
    if grid:
        from dataclasses import replace
        nx, ny = (int(v) for v in grid.lower().split("x"))
        cfg = replace(cfg, grid=replace(cfg.grid, nx=nx, ny=ny))
    net = build_b200(cfg)
    t0 = time.perf_counter()
    if shards > 1:
        from paper_1803_08833_b200.distributed import run_local_shards
        res = run_local_shards(cfg, shards)
    else:
        res = run_b200(cfg, 1, net=net)
    gpu_s = time.perf_counter() - t0
    row_off, tgt, w, d = net.host_csr()
    del net
    import torch
    torch.cuda.empty_cache()
    k = min(len(os.sched_getaffinity(0)), 16)
    from paper_1803_08833_b200.partition import map_columns_to_workers
    while k > 1:
        try:
            map_columns_to_workers(cfg.grid, k)
            break
        except ValueError:
            k -= 1
    t1 = time.perf_counter()
    ref = run_oracle_mp(cfg, row_off, np.asarray(tgt, dtype=np.int32), d, w, k, cfg.n_steps, 1e9,
                        collect_raster=True)
    cpu_s = time.perf_counter() - t1
    same_g = bool(np.array_equal(res.raster_gids, ref["raster_gids"]))
    same_t = bool(np.array_equal(res.raster_times.view(np.uint64),
                                 ref["raster_times"].view(np.uint64)))
    out = dict(config=idx, grid=f"{cfg.grid.nx}x{cfg.grid.ny}", steps=cfg.n_steps, gpu_shards=shards,
               synapses=int(res.recurrent_synapses), spikes_gpu=int(res.n_spikes),
               spikes_oracle=int(len(ref["raster_gids"])), raster_gids_equal=same_g,
               raster_times_bit_equal=same_t,
               recurrent_events=[int(res.recurrent_events), ref["recurrent_events"]],
               external_events=[int(res.external_events), ref["external_events"]],
               raster_checksum=f"0x{res.raster_checksum:016x}", gpu_wall_s=gpu_s,
               oracle_wall_s=cpu_s, oracle_processes=k,
               mean_rate_hz=res.mean_rate_hz, regime=regime,
               device_stats={k_: v for k_, v in (res.device_stats or {}).items()
                             if not isinstance(v, dict)},
               delivery=("routed (k_route + k_bin), 8 sub-lists"
                         if os.environ.get("CC_ROUTED", "") != "0" and regime == "stress"
                         else "k_deliver"))
    print(json.dumps(out))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    name = (f"long_parity_config{idx}" + (f"_{shards}shards" if shards > 1 else "")
            + ("" if regime == "calibrated" else f"_{regime}") + (f"_{grid}" if grid else ""))
    with open(os.path.join(ROOT, "gpurun_out", name + ".json"), "w") as fh:
        json.dump(out, fh, indent=1)
    ok = same_g and same_t and out["recurrent_events"][0] == out["recurrent_events"][1] \
        and out["external_events"][0] == out["external_events"][1]
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
