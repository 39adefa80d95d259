"""[needs a library built with -DCC_TIMING_PROBES=1, selected with CC_LIB_PATH]
Cost split of k_deliver: one step from an identical restored snapshot with
parts of the deposit masked out (flags 1024: no reservation atomics, 2048: no
record stores), k_stage's tail delivery off so that k_deliver delivers every
arrival.

    CC_LIB_PATH=build_variants/lib_probes.so python tools/stage_timing.py [config] [regime]
"""
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

cfg = baseline_config(int(sys.argv[1]) if len(sys.argv) > 1 else 1,
                      sys.argv[2] if len(sys.argv) > 2 else "calibrated")
net = build_b200(cfg)
capacity = None
while True:
    sim = Simulator(cfg, net, chunk=100, use_graphs=False, capacity=capacity)
    sim.shard.flags = 4096
    try:
        sim.advance(int(os.environ.get("T0", "300")))
        break
    except _lib.EngineError as err:
        capacity = _lib.grow_capacity(err, sim.capacity)
        if capacity is None:
            raise
        del sim
        torch.cuda.empty_cache()
L = sim.L
st = torch.cuda.current_stream().cuda_stream
snap = {k: v.clone() for k, v in sim.buf.items() if k not in ("raster_gid", "raster_t")}
variants = {"full": 0, "no reservation atomics": 1024, "no record stores": 2048,
            "loads only": 1024 | 2048}
e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
res = {k: [] for k in variants}
for rep in range(4):
    for name, mask in variants.items():
        for k, v in snap.items():
            sim.buf[k].copy_(v)
        sim.shard.flags = 4096 | mask
        torch.cuda.synchronize()
        e0.record()
        _lib.check(L.cc_deliver(C.byref(sim.shard), st))
        e1.record()
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1) * 1e3)
ev = int(sim.ctl().del_events)
for name, v in res.items():
    print(f"{name:26s} k_deliver {np.mean(v[1:]):8.1f} us")
