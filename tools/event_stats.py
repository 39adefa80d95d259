"""Distribution of inputs per neuron-step at steady state (design diagnostics).
Recurrent counts are read from the delay ring after k_deliver; external counts
from the same counter-based Poisson draw (host copy)."""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1803_08833_b200 import _lib  # noqa: E402
from paper_1803_08833_b200.engine import Simulator  # noqa: E402
from paper_1803_08833_b200.network import build_b200  # noqa: E402
from paper_1803_08833_b200.presets import baseline_config  # noqa: E402
from oracle.corticarc_oracle import poisson_counts  # noqa: E402

cfg = baseline_config(int(sys.argv[1]) if len(sys.argv) > 1 else 1, "calibrated")
net = build_b200(cfg)
sim = Simulator(cfg, net, chunk=100)
sim.advance(400)
L = sim.L
st = torch.cuda.current_stream().cuda_stream
lam = cfg.external.mean_per_step(cfg.timestep_ms)
stats = []
for t in range(400, 440):
    _lib.check(L.cc_deliver(C.byref(sim.shard), st))
    _lib.check(L.cc_neuron_step(C.byref(sim.shard), st))
    torch.cuda.synchronize()
    n = sim.buf["ev_n"].cpu().numpy().astype(np.int64)      # inputs per neuron (ring + drive)
    w = n[: len(n) // 32 * 32].reshape(-1, 32)
    stats.append(dict(t=t, mean=float(n.mean()), max=int(n.max()), e2e=float((n * n).sum() / max(1, n.sum())),
                      warp_max_sum=int(w.max(1).sum()), warp_sum=int(w.sum()),
                      frac_events_n_gt32=float(n[n > 32].sum() / max(1, n.sum()))))
for s in stats:
    print(json.dumps(s))
ws = sum(s["warp_max_sum"] for s in stats) * 32 / sum(s["warp_sum"] for s in stats)
print("imbalance (sum of warp max * 32 / total)", ws)
