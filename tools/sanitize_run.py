"""Small runs for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): tiny_gauss through both planning modes (separate k_plan, planning
fused into k_stage behind its grid barrier), with and without k_stage's tail
delivery, the spill path variant, and the peer exchange in loopback; every run
is checked against the golden raster so the sanitized code is the real path.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import golden_run  # noqa: E402

from paper_1803_08833_b200.engine import run_b200  # noqa: E402

cfg, meta, arr = golden_run("tiny_gauss")
steps = int(os.environ.get("SAN_STEPS", "40"))
ok = True
for flags in ("0", "16384", "32768", "4096", "36864"):
    os.environ["CC_FLAGS"] = flags
    res = run_b200(cfg, 1, steps=steps, use_graphs=False)
    m = arr["raster_times"] < steps * cfg.timestep_ms
    same = (np.array_equal(res.raster_gids, arr["raster_gids"][m].astype(np.uint64))
            and np.array_equal(res.raster_times, arr["raster_times"][m]))
    ok &= same
    print(f"flags {flags}: {res.n_spikes} spikes, same raster {same}", flush=True)
os.environ["CC_FLAGS"] = "0"
if os.environ.get("SAN_X", "1") == "1":
    from paper_1803_08833_b200.distributed import DistributedSimulator, _init_dist
    import torch.distributed as dist
    _init_dist()
    ds = DistributedSimulator(cfg, 0, 1, chunk=steps, transport="p2p", sync="host", loopback=True)
    ds.advance(steps)
    g, t = ds.sim.raster()
    m = arr["raster_times"] < steps * cfg.timestep_ms
    same = np.array_equal(g, arr["raster_gids"][m].astype(np.uint64))
    ok &= same
    print(f"p2p loopback: same raster {same}, sent {ds.sim.ctl().x_sent}", flush=True)
    ds.close()
    dist.destroy_process_group()
print("SANITIZE_RUN_OK" if ok else "SANITIZE_RUN_MISMATCH")
