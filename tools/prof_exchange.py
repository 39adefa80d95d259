"""Steps of the one-GPU loopback exchange for an ncu launch list: warm up W
steps, then S eager steps (deliver, plan, stage with pushes, cc_exchange_ingest)
between cudaProfilerStart/Stop (ncu --profile-from-start off)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1803_08833_b200.distributed import DistributedSimulator, _init_dist  # noqa: E402
from paper_1803_08833_b200.presets import baseline_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--warmup", type=int, default=400)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--loopback", type=int, default=1)
a = ap.parse_args()
cfg = baseline_config(a.config, "calibrated", duration_s=(a.warmup + a.steps) / 1000.0)
_init_dist()
ds = DistributedSimulator(cfg, 0, 1, chunk=100, transport="p2p", sync="device",
                          loopback=bool(a.loopback))
ds.advance(a.warmup)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.steps):
    ds.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
ds.sim.t = ds.t
ds.sim.check()
print("ok", ds.sim.ctl().x_sent)
ds.close()
dist.destroy_process_group()
