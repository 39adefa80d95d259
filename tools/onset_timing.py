"""Per-step device time of the first steps (onset) of BASELINE config 1:
graph replays vs eager launches vs run_b200's wall (diagnostic)."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_08833_b200 import _lib  # noqa: E402
from paper_1803_08833_b200.engine import Simulator, run_b200  # noqa: E402
from paper_1803_08833_b200.network import build_b200  # noqa: E402
from paper_1803_08833_b200.presets import baseline_config  # noqa: E402

L = _lib.lib()
cfg = baseline_config(1, "calibrated", duration_s=0.025)
net = build_b200(cfg)
for mode in ("eager", "graph", "eager"):
    sim = Simulator(cfg, net, chunk=5, raster_steps=30, use_graphs=False)
    timer = C.c_void_p()
    L.cc_timer_create(3 * 25, C.byref(timer))
    s = torch.cuda.current_stream().cuda_stream
    if mode == "graph":
        gs = [sim.capture(5, timer=timer, timer_base=15 * k) for k in range(5)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for g in gs:
            g.replay()
    else:
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(25)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(25):
            evs[i][0].record()
            L.cc_deliver(C.byref(sim.shard), s)
            evs[i][1].record()
            L.cc_neuron_step(C.byref(sim.shard), s)
            evs[i][2].record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if mode == "graph":
        d = [L.cc_timer_elapsed_ms(timer, 3 * i, 3 * i + 1) for i in range(25)]
        n = [L.cc_timer_elapsed_ms(timer, 3 * i + 1, 3 * i + 2) for i in range(25)]
    else:
        d = [e[0].elapsed_time(e[1]) for e in evs]
        n = [e[1].elapsed_time(e[2]) for e in evs]
    c = sim.ctl()
    print(mode, f"wall {wall*1e3:.2f} ms, spikes {c.n_spikes}, events {c.rec_events + c.ext_events}")
    print("  deliver us", np.round(np.array(d) * 1e3, 1).tolist())
    print("  neuron  us", np.round(np.array(n) * 1e3, 1).tolist())
    L.cc_timer_destroy(timer)
    del sim
res = run_b200(cfg, 1, net=net)
print("run_b200 wall ms", res.sim_seconds_wall * 1e3, "events", res.recurrent_events + res.external_events)
