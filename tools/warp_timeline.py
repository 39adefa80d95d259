"""[needs a library built with -DCC_TIMING_PROBES=1, selected with CC_LIB_PATH]
Per-warp timeline of k_stage (flags bit 32): where does a warp spend time?"""
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
nw = (sim.n_local + 31) // 32
for rep in range(3):
    _lib.check(L.cc_deliver(C.byref(sim.shard), st))
    sim.shard.flags = 32 | 8
    _lib.check(L.cc_neuron_step(C.byref(sim.shard), st))
    sim.shard.flags = 0
    torch.cuda.synchronize()
    raw = sim.buf["scratch"].view(torch.int64).view(-1)
    tail = raw[raw.numel() - nw * 16:].cpu().numpy().reshape(nw, 16)[::-1]
    t0 = tail[:, 0].min()
    s = tail[:, :9].astype(np.float64) - t0
    rounds = tail[:, 9]
    print(f"rep {rep}: kernel span {(tail[:,8].max()-t0)/1e3:.1f} us; warp start spread {(tail[:,0].max()-t0)/1e3:.1f} us")
    dur = (tail[:, 8] - tail[:, 0]) / 1e3
    print(f"  warp duration us: mean {dur.mean():.1f} p50 {np.median(dur):.1f} p90 {np.percentile(dur,90):.1f} max {dur.max():.1f}")
    print(f"  rounds: mean {rounds.mean():.2f} max {rounds.max()}  nmax mean {tail[:,11].mean():.1f}")
    setup = (tail[:, 1] - tail[:, 0]) / 1e3
    g1 = (tail[:, 2] - tail[:, 1]) / 1e3
    s1 = (tail[:, 3] - tail[:, 2]) / 1e3
    f1 = (tail[:, 4] - tail[:, 3]) / 1e3
    print(f"  setup {setup.mean():.1f}  round1: gather+admit {g1.mean():.1f} ext+sort {s1.mean():.1f} factors {f1.mean():.1f}")
    two = rounds >= 2
    if two.any():
        g2 = (tail[two, 5] - tail[two, 4]) / 1e3
        s2 = (tail[two, 6] - tail[two, 5]) / 1e3
        f2 = (tail[two, 7] - tail[two, 6]) / 1e3
        print(f"  round2 ({two.sum()} warps): gather {g2.mean():.1f} sort {s2.mean():.1f} factors {f2.mean():.1f}")
    end = (tail[:, 8] - np.where(two, tail[:, 7], tail[:, 4])) / 1e3
    print(f"  after last round -> end {end.mean():.1f}")
    # per SM occupancy over time
    starts = (tail[:, 0] - t0) / 1e3
    print("  warps started after 10us:", int((starts > 10).sum()), " after 30us:", int((starts > 30).sum()))
order = np.argsort(-dur)
print("slowest warps: idx sm rounds nmax dur setup r1(g,s,f) r2(g,s,f)")
for w in order[:12]:
    r = tail[w]
    print(w, r[10], r[9], r[11], f"{dur[w]:.1f}", f"{(r[1]-r[0])/1e3:.1f}",
          [f"{(r[k]-r[k-1])/1e3:.1f}" for k in range(2, 8)])
# per-SM total warp time
sm = tail[:, 10]
tot = np.bincount(sm, weights=dur)
cnt = np.bincount(sm)
print("per-SM warps min/max", cnt[cnt>0].min(), cnt.max(), " per-SM summed warp-us min/max", tot[cnt>0].min(), tot.max())
nev = sim.buf["ev_n"].cpu().numpy()
nw_ev = np.add.reduceat(nev, np.arange(0, len(nev), 32))
print("events of slowest warps:", [int(nw_ev[w]) for w in order[:12]], " median warp events", np.median(nw_ev))
print("corr(duration, warp events) =", np.corrcoef(dur, nw_ev[:len(dur)])[0,1])
