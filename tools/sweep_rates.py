"""Operating-point sweep on the GPU: mean rate (whole run and second half) per
(J_inh->exc, J_inh->inh, drive) on one BASELINE grid, the connectivity built
once per weight set (calibration_sweep of metrics.py:317-332, extended to the
inhibitory weights)."""
import argparse
import json
import os
import sys
import time

import numpy as np
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1803_08833_b200.presets import baseline_config  # noqa: E402
from paper_1803_08833_b200.engine import run_b200  # noqa: E402
from paper_1803_08833_b200.network import build_b200  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--kernel", default=None)
ap.add_argument("--grid", default=None)
ap.add_argument("--rates", default="100,200,400")
ap.add_argument("--j", default="-2:-2,-4:-4,-8:-8", help="jie:jii pairs")
ap.add_argument("--jee", type=float, default=None)
ap.add_argument("--duration", type=float, default=0.3)
a = ap.parse_args()
for pair in a.j.split(","):
    jie, jii = (float(x) for x in pair.split(":"))
    cfg0 = baseline_config(a.config, "calibrated", kernel=a.kernel, duration_s=a.duration)
    if a.grid:
        nx, ny = (int(v) for v in a.grid.split("x"))
        cfg0 = replace(cfg0, grid=replace(cfg0.grid, nx=nx, ny=ny))
    gs = replace(cfg0.genspec, j_inh_exc=jie, j_inh_inh=jii)
    if a.jee is not None:
        gs = replace(gs, j_exc_exc=a.jee, j_exc_inh=a.jee)
    cfg0 = replace(cfg0, genspec=gs)
    net = build_b200(cfg0)
    for r in [float(x) for x in a.rates.split(",")]:
        cfg = replace(cfg0, external=replace(cfg0.external, rate_per_synapse_hz=r))
        t = time.time()
        row = dict(config=a.config, grid=f"{cfg.grid.nx}x{cfg.grid.ny}", jee=gs.j_exc_exc,
                   jie=jie, jii=jii, drive=r)
        try:
            res = run_b200(cfg, 1, net=net)
        except Exception as err:
            row["error"] = str(err)[:160]
            print(json.dumps(row), flush=True)
            continue
        n = cfg.grid.n_neurons
        g = res.raster_gids.astype(int)
        exc = (g % 1240) < 992
        late = res.raster_times >= cfg.duration_s * 500
        nsteps = cfg.n_steps
        cnt = np.bincount((res.raster_times // cfg.timestep_ms).astype(int), minlength=nsteps) \
            if len(g) else np.zeros(nsteps)
        row.update(rate=round(res.mean_rate_hz, 3),
                   rate_late=round(float(late.sum() / (n * cfg.duration_s / 2)), 3),
                   e_rate=round(float(exc.sum() / (n * 0.8 * cfg.duration_s)), 3),
                   i_rate=round(float((~exc).sum() / (n * 0.2 * cfg.duration_s)), 3),
                   cv_pop=round(float(np.std(cnt[nsteps // 2:]) / max(1e-9, np.mean(cnt[nsteps // 2:]))), 3),
                   rec_per_step=round(res.recurrent_events / nsteps / 1e6, 2),
                   ext_per_step=round(res.external_events / nsteps / 1e6, 2),
                   ms_per_step=round(res.sim_seconds_wall / nsteps * 1e3, 3),
                   max_events=res.device_stats["max_events"], wall=round(time.time() - t, 1))
        print(json.dumps(row), flush=True)
    del net
