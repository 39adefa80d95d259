"""Steps for ncu captures: warm up W steps (graphs), then run S eager steps
between cudaProfilerStart/Stop (use ncu --profile-from-start off).

    python tools/prof_steps.py --config 1 --warmup 400 --steps 2 [--flags 4096]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_08833_b200.engine import Simulator  # noqa: E402
from paper_1803_08833_b200.network import build_b200  # noqa: E402
from paper_1803_08833_b200.presets import baseline_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--regime", default="calibrated")
ap.add_argument("--grid", default=None)
ap.add_argument("--warmup", type=int, default=400)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--flags", type=int, default=0)
a = ap.parse_args()
cfg = baseline_config(a.config, a.regime, duration_s=(a.warmup + a.steps) / 1000.0)
if a.grid:
    from dataclasses import replace
    nx, ny = (int(v) for v in a.grid.split("x"))
    cfg = replace(cfg, grid=replace(cfg.grid, nx=nx, ny=ny))
net = build_b200(cfg)
from paper_1803_08833_b200 import _lib  # noqa: E402
capacity = None
while True:                      # onset bursts: grow the overflowed buffer (run_b200's policy)
    sim = Simulator(cfg, net, chunk=100, capacity=capacity)
    try:
        sim.advance(a.warmup)
        break
    except _lib.EngineError as err:
        capacity = _lib.grow_capacity(err, sim.capacity)
        if capacity is None:
            raise
        del sim
        torch.cuda.empty_cache()
sim.shard.flags |= a.flags          # (keeps the routed mode's no-tail-delivery flag)
s = torch.cuda.current_stream().cuda_stream
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.steps):
    sim._launch_step(s)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
sim.t += a.steps
c = sim.check(collect_raster=False)
print("ok", c.n_spikes, c.rec_events)
