"""[needs a library built with -DCC_TIMING_PROBES=1, selected with CC_LIB_PATH]
Dump k_stage's per-work-item timestamps (flags bit 32) of a few steady-state
steps to an .npz for offline analysis (tools/item_timeline.py prints a summary).

    CC_LIB_PATH=build_variants/lib_probes.so python tools/item_dump.py out.npz [config] [regime]
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

out = sys.argv[1]
cfg = baseline_config(int(sys.argv[2]) if len(sys.argv) > 2 else 1,
                      sys.argv[3] if len(sys.argv) > 3 else "calibrated")
net = build_b200(cfg)
sim = Simulator(cfg, net, chunk=100, capacity=dict(scratch=int(os.environ.get('CC_SCRATCH_X', '1'))))
sim.advance(400)
L = sim.L
st = torch.cuda.current_stream().cuda_stream
res = {}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    _lib.check(L.cc_deliver(C.byref(sim.shard), st))
    sim.shard.flags = 32
    e0.record()
    _lib.check(L.cc_neuron_step(C.byref(sim.shard), st))
    e1.record()
    sim.shard.flags = 0
    torch.cuda.synchronize()
    ni = int(sim.ctl().n_rounds)
    raw = sim.buf["scratch"].view(torch.int64).reshape(-1)
    tail = raw[raw.numel() - ni * 8:].cpu().numpy().reshape(ni, 8)[::-1].astype(np.int64)
    res[f"items{rep}"] = tail
    res[f"ms{rep}"] = np.array(e0.elapsed_time(e1))
    # queue entries (group, lane range) in claim order, for joining with ev_n
    res[f"rounds{rep}"] = sim.buf["rounds"].cpu().numpy()
    res[f"cls{rep}"] = np.array([int(x) for x in sim.ctl().cls_n])
    res[f"ev_n{rep}"] = sim.buf["ev_n"].cpu().numpy()
    print(rep, ni, float(res[f"ms{rep}"]))
np.savez_compressed(out, **res)
