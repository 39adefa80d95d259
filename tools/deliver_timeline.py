"""[needs a library built with -DCC_TIMING_PROBES=1, selected with CC_LIB_PATH]
Per-warp timeline of k_deliver (flags bit 256)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1803_08833_b200 import _lib  # noqa: E402
from paper_1803_08833_b200.engine import Simulator  # noqa: E402
from paper_1803_08833_b200.network import build_b200  # noqa: E402
from paper_1803_08833_b200.presets import baseline_config  # noqa: E402

cfg = baseline_config(1, "calibrated")
net = build_b200(cfg)
sim = Simulator(cfg, net, chunk=100)
sim.advance(400)
L = sim.L
st = torch.cuda.current_stream().cuda_stream
nw = 148 * 2 * 8
extra = int(os.environ.get("DBG", "0"))
for rep in range(3):
    sim.shard.flags = 256 | extra
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(L.cc_deliver(C.byref(sim.shard), st))
    e1.record()
    sim.shard.flags = 0
    _lib.check(L.cc_neuron_step(C.byref(sim.shard), st))
    torch.cuda.synchronize()
    raw = sim.buf["scratch"].view(torch.int64).reshape(-1)
    base = raw.numel() - 65536 * 8
    tail = raw[base - nw * 4: base].cpu().numpy().reshape(nw, 4)[::-1].astype(np.int64)
    t0 = tail[:, 0].min()
    start = (tail[:, 0] - t0) / 1e3
    setup = (tail[:, 1] - tail[:, 0]) / 1e3
    loop = (tail[:, 2] - tail[:, 1]) / 1e3
    nunits = tail[0, 3] >> 32          # work units (delay, 4 spikes)
    busy = np.arange(nw) < nunits
    print(f"rep {rep}: event-timed {e0.elapsed_time(e1)*1e3:.1f} us, units {nunits}, span {((tail[:,2]-t0)/1e3).max():.1f} us")
    print(f"  warp start: p50 {np.median(start):.2f} max {start.max():.2f}; setup p50 {np.median(setup):.2f} max {setup.max():.2f}")
    print(f"  loop (busy warps): p50 {np.median(loop[busy]):.2f} p90 {np.percentile(loop[busy],90):.2f} max {loop[busy].max():.2f}")
    nb = 148 * 2
    ends = raw[base - 65536 * 4 - nb: base - 65536 * 4].cpu().numpy().astype(np.int64)
    print(f"  block ends after loop: max {(ends.max()-t0)/1e3:.2f} us; last loop end {(tail[:,2].max()-t0)/1e3:.2f} us")
