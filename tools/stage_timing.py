"""[needs a library built with -DCC_TIMING_PROBES=1, selected with CC_LIB_PATH]
Per-stage cost of k_neuron: time one step from an identical restored
snapshot with stages masked out (flags), averaged over several steps."""
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

cfg = baseline_config(int(os.environ.get("CFG", "1")), "calibrated")
net = build_b200(cfg)
sim = Simulator(cfg, net, chunk=100)
sim.advance(int(os.environ.get("T0", "400")))
L = sim.L
st = torch.cuda.current_stream().cuda_stream
snap = {k: v.clone() for k, v in sim.buf.items()}
variants = {"full": 0, "deliver: loads only": 64, "deliver: loads+store": 64 | 128}
# neuron = k_stage + k_update (two launches) timed together
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
res = {k: [] for k in variants}
for rep in range(5):
    for name, mask in variants.items():
        for k, v in snap.items():
            sim.buf[k].copy_(v)
        sim.shard.flags = mask
        torch.cuda.synchronize()
        e0.record()
        _lib.check(L.cc_deliver(C.byref(sim.shard), st))
        e1.record()
        _lib.check(L.cc_neuron_step(C.byref(sim.shard), st))
        e2.record()
        torch.cuda.synchronize()
        res[name].append((e0.elapsed_time(e1) * 1e3, e1.elapsed_time(e2) * 1e3))
for name, v in res.items():
    v = np.array(v[1:])
    print(f"{name:28s} deliver {v[:,0].mean():7.1f} us   neuron {v[:,1].mean():7.1f} us")
