"""[needs a library built with -DCC_TIMING_PROBES=1, selected with CC_LIB_PATH]
Group-update durations of k_stage against the update's iteration count, slow
steps (refractory / after a spike) and spikes: where the in-order update's
time goes (flags bit 32; slot 1 carries the update's counters)."""
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
rows = []
for rep in range(5):
    _lib.check(L.cc_deliver(C.byref(sim.shard), st))
    base = sim.shard.flags
    sim.shard.flags = base | 32
    _lib.check(L.cc_neuron_step(C.byref(sim.shard), st))
    sim.shard.flags = base
    torch.cuda.synchronize()
    ni = int(sim.ctl().n_rounds)
    raw = sim.buf["scratch"].view(torch.int64).reshape(-1)
    tail = raw[raw.numel() - ni * 8:].cpu().numpy().reshape(ni, 8)[::-1].astype(np.uint64)
    upd = tail[:, 5] > 0
    info = tail[upd, 1]
    dur = (tail[upd, 4].astype(np.int64) - tail[upd, 5].astype(np.int64)) / 1e3
    nmax = (info & 0xffff).astype(np.int64)
    slow = ((info >> 16) & 0xffff).astype(np.int64)
    lanes = ((info >> 32) & 0xffff).astype(np.int64)
    spk = ((info >> 48) & 0x7fff).astype(np.int64)
    rows.append(np.stack([dur, nmax, slow, lanes, spk], 1))
r = np.concatenate(rows)
dur, nmax, slow, lanes, spk = r.T
print(f"updates {len(r)}: dur mean {dur.mean():.2f} p50 {np.median(dur):.2f} p90 {np.percentile(dur,90):.2f} max {dur.max():.2f} us")
print(f"nmax mean {nmax.mean():.1f} max {nmax.max():.0f}; groups with slow steps {np.mean(slow>0):.2f}, with spikes {np.mean(spk>0):.2f}")
f = slow == 0
print(f"fast-only groups: {f.sum()}, dur mean {dur[f].mean():.2f} us, per iteration {1e3*(dur[f]/nmax[f]).mean():.0f} ns")
A = np.stack([np.ones_like(dur), nmax, slow, spk], 1)
coef, *_ = np.linalg.lstsq(A, dur, rcond=None)
print("least squares dur ~ a + b*nmax + c*slow_steps(max lane) + d*spiking lanes: "
      f"a {coef[0]:.2f} us, b {1e3*coef[1]:.0f} ns, c {1e3*coef[2]:.0f} ns, d {coef[3]:.2f} us")
for lo, hi in ((0, 0), (1, 5), (6, 15), (16, 1000)):
    m = (slow >= lo) & (slow <= hi)
    if m.any():
        print(f"  slow steps {lo}-{hi}: {m.sum()} groups, dur mean {dur[m].mean():.2f} max {dur[m].max():.2f}, nmax {nmax[m].mean():.1f}")
