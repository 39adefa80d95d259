"""Calibration sweep on the GPU (metrics.calibration_sweep, metrics.py:317-332,
with the B200 runner): mean firing rate per external drive rate."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1803_08833_b200.presets import baseline_config  # noqa: E402
from paper_1803_08833_b200.engine import run_b200  # noqa: E402
from paper_1803_08833_b200.network import build_b200  # noqa: E402
from dataclasses import replace  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--kernel", default=None)
ap.add_argument("--rates", default="25,30,35,40,45")
ap.add_argument("--jinh", type=float, default=None)
ap.add_argument("--jii", type=float, default=None, help="inh->inh weight (default: --jinh)")
ap.add_argument("--duration", type=float, default=1.0)
a = ap.parse_args()
for r in [float(x) for x in a.rates.split(",")]:
    cfg = baseline_config(a.config, "calibrated", kernel=a.kernel, drive_hz=r, duration_s=a.duration)
    if a.jinh is not None:
        cfg = replace(cfg, genspec=replace(cfg.genspec, j_inh_exc=a.jinh, j_inh_inh=a.jinh))
    if a.jii is not None:
        cfg = replace(cfg, genspec=replace(cfg.genspec, j_inh_inh=a.jii))
    t = time.time()
    try:
        res = run_b200(cfg, 1)
    except Exception as err:             # capacity errors = runaway activity
        print(json.dumps(dict(config=a.config, drive=r, jinh=cfg.genspec.j_inh_exc, jii=cfg.genspec.j_inh_inh,
                              error=str(err)[:200])), flush=True)
        continue
    n = cfg.grid.n_neurons
    g = res.raster_gids.astype(int)
    exc = (g % 1240) < 992
    second_half = res.raster_times >= cfg.duration_s * 500
    print(json.dumps(dict(config=a.config, kernel=cfg.kernel.kind, drive=r, jinh=cfg.genspec.j_inh_exc, jii=cfg.genspec.j_inh_inh,
                          rate=res.mean_rate_hz,
                          rate_late=float(second_half.sum() / (n * cfg.duration_s / 2)),
                          e_rate=float(exc.sum() / (n * 0.8 * cfg.duration_s)),
                          i_rate=float((~exc).sum() / (n * 0.2 * cfg.duration_s)),
                          syn=res.recurrent_synapses, sim_s=res.sim_seconds_wall,
                          build_s=res.construction_seconds, ev=res.recurrent_events + res.external_events,
                          max_bin=res.device_stats["max_bin"], max_events=res.device_stats["max_events"],
                          overflow=res.device_stats["overflow"], wall=time.time() - t)), flush=True)
