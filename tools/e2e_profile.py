"""Host-side cost of the public API: run_b200 wall vs device-timed replays."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402
from paper_1803_08833_b200.engine import Simulator, run_b200  # noqa: E402
from paper_1803_08833_b200.network import build_b200  # noqa: E402
from paper_1803_08833_b200.presets import baseline_config  # noqa: E402

cfg = baseline_config(1, "calibrated", duration_s=1.2)
net = build_b200(cfg)
sim = Simulator(cfg, net, chunk=100)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(12):
    sim._graphs[0].replay()
torch.cuda.synchronize()
dev = time.perf_counter() - t0
del sim
for rep in range(2):
    r = run_b200(cfg, 1, net=net)
    print(f"run_b200 wall {1e3 * r.sim_seconds_wall:.1f} ms vs back-to-back replays "
          f"{1e3 * dev:.1f} ms for {cfg.n_steps} steps; substeps {r.substep_seconds}")
