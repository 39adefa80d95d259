"""Bytes per synapse stored and on-device generation throughput, Gaussian vs
exponential (the paper's memory study), for BASELINE configs
1-4, plus the simulation buffers a Simulator allocates on top.  Config 4
(96x96) is built as rank 0 of an 8-GPU tiling (one GPU's shard)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1803_08833_b200.geometry import grid_totals  # noqa: E402
from paper_1803_08833_b200.network import build_b200  # noqa: E402
from paper_1803_08833_b200.presets import baseline_config  # noqa: E402

cases = [(1, "gaussian", 1), (2, "exponential", 1), (3, "gaussian", 1), (3, "exponential", 1),
         (4, "exponential", 8)]
only = sys.argv[1:]
out = []
for idx, kern, size in cases:
    if only and f"{idx}{kern[0]}" not in only:
        continue
    cfg = baseline_config(idx, "calibrated", kernel=kern)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    net = build_b200(cfg, rank=0, size=size)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    local, remote = grid_totals(cfg.kernel, cfg.grid)
    row = dict(config=idx, kernel=kern, grid=f"{cfg.grid.nx}x{cfg.grid.ny}", shard=f"0/{size}",
               neurons_local=net.n_local, synapses=net.n_synapses,
               forecast_total=local + remote, build_s=dt,
               synapses_per_s=net.n_synapses / dt,
               csr_bytes=9 * net.n_synapses, index_bytes=8 * (cfg.grid.n_neurons + 1),
               bytes_per_synapse_steady=net.steady_bytes / net.n_synapses,
               bytes_per_synapse_peak=net.peak_bytes / net.n_synapses,
               reference_bytes_per_synapse_steady=12.0, reference_peak_floor=24.0,
               max_row=net.row_len_max, halo_sources=len(net.src_gids),
               checksum=f"0x{net.checksum:016x}", gpu_mem_peak_gb=torch.cuda.max_memory_allocated() / 1e9)
    # the simulation's own device buffers on top (input lists, spike log,
    # ordered-input records, spill staging, raster, delay-segment table)
    from paper_1803_08833_b200.engine import Simulator
    sim = Simulator(cfg, net, use_graphs=False)
    torch.cuda.synchronize()
    row.update(sim_buffer_bytes=sim.device_bytes,
               dseg_bytes=sum(v.numel() * v.element_size() for v in net.dseg_cache.values()),
               device_allocated_gb=torch.cuda.memory_allocated() / 1e9)
    del sim
    print(json.dumps(row), flush=True)
    out.append(row)
    del net
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/memory_study.json", "w"), indent=1)
