"""[needs a library built with -DCC_TIMING_PROBES=1, selected with CC_LIB_PATH]
Per-group timeline of k_plan (flags bit 512): start, records counted,
Poisson done, items split, items queued."""
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
ng = sim.shard.n_groups
for rep in range(3):
    _lib.check(L.cc_deliver(C.byref(sim.shard), st))
    sim.shard.flags = 512
    _lib.check(L.cc_neuron_step(C.byref(sim.shard), st))
    sim.shard.flags = 0
    torch.cuda.synchronize()
    raw = sim.buf["scratch"].view(torch.int64).reshape(-1)
    tail = raw[raw.numel() - ng * 8:].cpu().numpy().reshape(ng, 8)[::-1].astype(np.int64)
    t0 = tail[:, 0].min()
    rel = (tail[:, :5] - t0) / 1e3
    print(f"rep {rep}: groups {ng}, span {rel[:, 4].max():.1f} us")
    print("  start   quantiles:", [round(float(np.percentile(rel[:, 0], q)), 2) for q in (0, 50, 90, 100)])
    for k, name in enumerate(["records", "poisson", "split", "queue"]):
        d = rel[:, k + 1] - rel[:, k]
        print(f"  {name:8s} p50 {np.median(d):6.2f} p90 {np.percentile(d, 90):6.2f} max {d.max():6.2f}")
    print("  end     quantiles:", [round(float(np.percentile(rel[:, 4], q)), 2) for q in (0, 50, 90, 100)])
    heavy = tail[:, 6] > np.percentile(tail[:, 6], 90)
    print(f"  heavy groups (c_all p90+ = {np.percentile(tail[:, 6], 90):.0f}): end p50 {np.median(rel[heavy, 4]):.2f}")
