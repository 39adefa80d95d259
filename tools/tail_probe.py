"""[needs a library built with -DCC_TIMING_PROBES=1, selected with CC_LIB_PATH]
The last work items of k_stage to finish: when they were claimed, how long
staging and the group update took, and the update's slow steps (flags bit 32)."""
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
sim.advance(400)
L = sim.L
st = torch.cuda.current_stream().cuda_stream
for rep in range(3):
    _lib.check(L.cc_deliver(C.byref(sim.shard), st))
    base = sim.shard.flags
    sim.shard.flags = base | 32
    _lib.check(L.cc_neuron_step(C.byref(sim.shard), st))
    sim.shard.flags = base
    torch.cuda.synchronize()
    ni = int(sim.ctl().n_rounds)
    raw = sim.buf["scratch"].view(torch.int64).reshape(-1)
    tail = raw[raw.numel() - ni * 8:].cpu().numpy().reshape(ni, 8)[::-1].astype(np.uint64)
    t0 = tail[:, 0].min()
    claim = (tail[:, 0] - t0).astype(np.int64) / 1e3
    end = (tail[:, 4] - t0).astype(np.int64) / 1e3
    upd = tail[:, 5] > 0
    ustart = np.where(upd, (tail[:, 5].astype(np.int64) - int(t0)) / 1e3, np.nan)
    info = np.where(upd, tail[:, 1], 0)
    nmax = (info & 0xffff).astype(np.int64)
    slow = ((info >> 16) & 0xffff).astype(np.int64)
    spk = ((info >> 48) & 0x7fff).astype(np.int64)
    order = np.argsort(-end)[:16]
    print(f"rep {rep}: items {ni}, kernel end {end.max():.1f} us; p90 {np.percentile(end, 90):.1f}")
    print("  item   claim  staged(upd start)  end   upd_us nmax slow spk  rtot  queue_pos")
    for i in order:
        print(f"  {i:5d} {claim[i]:6.1f} {ustart[i]:8.1f} {end[i]:10.1f} {end[i]-ustart[i]:6.1f} "
              f"{nmax[i]:4d} {slow[i]:4d} {spk[i]:3d} {int(tail[i,6]):5d}  {i}")
    # how many updates started after the median warp went idle
    late = upd & (ustart > np.percentile(end, 50))
    print(f"  updates starting after the median completion: {late.sum()} of {upd.sum()}, "
          f"mean {np.nanmean(end[late]-ustart[late]):.1f} us")
