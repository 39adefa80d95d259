"""[needs a library built with -DCC_TIMING_PROBES=1, selected with CC_LIB_PATH]
Per-work-item timeline of k_stage (flags bit 32)."""
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
for rep in range(2):
    _lib.check(L.cc_deliver(C.byref(sim.shard), st))
    sim.shard.flags = 32
    _lib.check(L.cc_neuron_step(C.byref(sim.shard), st))
    sim.shard.flags = 0
    torch.cuda.synchronize()
    ni = int(sim.ctl().n_rounds)
    raw = sim.buf["scratch"].view(torch.int64).reshape(-1)
    nz = torch.nonzero(raw).flatten()
    print("nonzero words in scratch:", nz.numel(), "last idx", int(nz[-1]) if nz.numel() else None, "size", raw.numel())
    tail = raw[raw.numel() - ni * 8:].cpu().numpy().reshape(ni, 8)[::-1].astype(np.int64)
    t0 = tail[:, 0].min()
    rel = (tail[:, :5] - t0) / 1e3
    dur = rel[:, 4] - rel[:, 0]
    print(f"rep {rep}: items {ni}, span {rel[:,4].max():.1f} us, first claim spread {np.sort(rel[:,0])[:2000].max():.1f} us")
    print(f"  item us: mean {dur.mean():.1f} p50 {np.median(dur):.1f} p90 {np.percentile(dur,90):.1f} max {dur.max():.1f}")
    for k, name in enumerate(["gather+drive", "sort", "factors", "publish+update"]):
        d = rel[:, k + 1] - rel[:, k]
        print(f"  {name:14s} mean {d.mean():6.2f} p90 {np.percentile(d,90):6.2f} max {d.max():6.2f}")
    warps = tail[:, 7]
    per_warp = np.bincount(warps)
    print(f"  warps used {np.count_nonzero(per_warp)}, items per warp mean {per_warp[per_warp>0].mean():.2f} max {per_warp.max()}")
    print(f"  rtot mean {tail[:,6].mean():.1f} max {tail[:,6].max()}")
    ends = np.sort(rel[:, 4])
    print("  completion quantiles (us):", [round(float(np.percentile(ends, q)), 1) for q in (10, 50, 90, 99, 100)])
    upd = tail[:, 5] > 0                      # slot 5: update start (0: the item ran no update)
    ud = (tail[upd, 4] - tail[upd, 5]) / 1e3
    print(f"  group updates {upd.sum()}: us mean {ud.mean():.2f} p90 {np.percentile(ud, 90):.2f} max {ud.max():.2f}")
    # tail: when does each warp finish its last item, and how big were late items
    last = {}
    for w_, e_ in zip(warps, rel[:, 4]):
        last[w_] = max(last.get(w_, 0.0), e_)
    lw = np.sort(np.array(list(last.values())))
    print("  warp finish quantiles (us):", [round(float(np.percentile(lw, q)), 1) for q in (0, 10, 50, 90, 100)])
    late = rel[:, 0] > np.percentile(rel[:, 0], 90)
    print(f"  items claimed in the last 10% of claim times: mean rtot {tail[late, 6].mean():.1f}, "
          f"mean dur {dur[late].mean():.1f} us (all: {tail[:, 6].mean():.1f}, {dur.mean():.1f})")
    idle = (rel[:, 4].max() - lw).sum() / (len(lw) * rel[:, 4].max())
    print(f"  warp-time idle after own last item: {100 * idle:.1f}%")
    # the last 5 % of claims: phase durations
    lastk = np.argsort(rel[:, 0])[-max(1, len(rel) // 20):]
    ph = np.diff(rel[lastk][:, [0, 1, 2, 3, 4]], axis=1)
    print(f"  last 5% claims: rtot {tail[lastk, 6].mean():.0f}, gather+drive {ph[:, 0].mean():.1f}, "
          f"sort {ph[:, 1].mean():.1f}, factors {ph[:, 2].mean():.1f}, "
          f"publish+update {ph[:, 3].mean():.1f} us; "
          f"end at {rel[lastk, 4].mean():.1f} (kernel end {rel[:, 4].max():.1f})")
