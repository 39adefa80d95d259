"""Drive a network into runaway activity and check that the engine stops with
an EngineError (capacity bits) instead of faulting.  usage:
    python tools/runaway_repro.py CONFIG DRIVE_HZ STEPS [kernel]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_08833_b200.presets import baseline_config  # noqa: E402
from paper_1803_08833_b200.engine import run_b200  # noqa: E402

idx, drive, steps = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
kernel = sys.argv[4] if len(sys.argv) > 4 else None
cfg = baseline_config(idx, "calibrated", kernel=kernel, drive_hz=drive, duration_s=steps / 1000.0)
try:
    r = run_b200(cfg, 1)
    print("ok", r.n_spikes, r.mean_rate_hz, r.device_stats)
except Exception as e:
    print("raised", type(e).__name__, str(e)[:300])
