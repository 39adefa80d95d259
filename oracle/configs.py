"""BASELINE configs for the CPU oracle - test / baseline infrastructure only.

An independent statement of the BASELINE.json configs as the reference's INI
would express them, so that the CPU reference arm of
bench.py (`--impl reference`) builds its run description without importing
the product package.  tests/test_oracle_golden.py checks that these equal
paper_1803_08833_b200.presets field by field.

The objects are plain namespaces carrying the attributes the oracle reads
(corticarc/connectivity.py:60-156, engine.py:66-121, model.py:44-86).
"""

from __future__ import annotations

import math
from types import SimpleNamespace

GRIDS = {0: (2, 2), 1: (8, 8), 2: (24, 24), 3: (48, 48), 4: (96, 96)}
DURATION_S = {0: 1.0, 1: 1.0, 2: 2.0, 3: 1.0, 4: 1.0}
# Gaussian sigma 100 um truncated at 3 sigma; exponential lambda 290 um, 12 columns,
# 75 % lateral
KERNELS = {
    "gaussian": dict(kind="gaussian", amplitude_A=0.05, scale=100.0, cutoff_p=5.4717e-4,
                     local_p=0.8),
    "exponential": dict(kind="exponential", amplitude_A=0.038120, scale=290.0,
                        cutoff_p=6.0718e-4, local_p=0.4822),
}
# operating points: (drive Hz per external synapse, J_inh->exc, J_inh->inh)
REGIMES = {
    "literal": {"gaussian": (3.0, -1.2, -1.2), "exponential": (3.0, -1.2, -1.2)},
    "calibrated": {"gaussian": (40.0, -2.0, -2.0), "exponential": (55.0, -8.0, -1.0)},
    "stress": {"gaussian": (40.0, -2.0, -2.0), "exponential": (200.0, -8.0, -8.0)},
}
NEURON = dict(tau_m=20.0, C_m=1.0, E=0.0, tau_c=300.0, g_c=0.5, V_theta=20.0, V_r=15.0,
              tau_arp=2.0, alpha_c=0.01)


class _Grid(SimpleNamespace):
    @property
    def n_columns(self):
        return self.nx * self.ny

    @property
    def n_neurons(self):
        return self.n_columns * self.neurons_per_column

    @property
    def n_excitatory_per_column(self):
        return int(math.floor(self.excitatory_fraction * self.neurons_per_column))


class _Config(SimpleNamespace):
    @property
    def n_steps(self):
        return int(round(self.duration_s * 1000.0 / self.timestep_ms))

    @property
    def d_max(self):
        return self.genspec.d_max_steps


def baseline_config(index: int, regime: str = "calibrated", kernel: str | None = None,
                    duration_s: float | None = None, seed: int = 1,
                    drive_hz: float | None = None, grid: str | None = None):
    nx, ny = GRIDS[index]
    if grid:
        nx, ny = (int(v) for v in grid.lower().split("x"))
    kernel = kernel or ("gaussian" if index in (0, 1, 3) else "exponential")
    rate, j_ie, j_ii = REGIMES[regime][kernel]
    if drive_hz is not None:
        rate = drive_hz
    # corticarc.connectivity.GaussianKernel / ExponentialKernel: sigma / lambda -> scale
    ks = SimpleNamespace(**KERNELS[kernel])
    gen = SimpleNamespace(j_exc_exc=0.3, j_exc_inh=0.3, j_inh_exc=j_ie, j_inh_inh=j_ii,
                          weight_sd_frac=0.1, delay_kind="uniform", delay_min_ms=1.0,
                          delay_max_ms=20.0, delay_mean_ms=3.0, timestep_ms=1.0, d_max_steps=20)
    return _Config(
        grid=_Grid(nx=nx, ny=ny, neurons_per_column=1240, excitatory_fraction=0.8,
                   spacing_alpha=100.0),
        kernel=ks, genspec=gen,
        exc_params=SimpleNamespace(is_excitatory=True, **NEURON),
        # inhibitory cells carry no adaptation (model.py:73-77: g_c = alpha_c = 0)
        inh_params=SimpleNamespace(is_excitatory=False, **dict(NEURON, g_c=0.0, alpha_c=0.0)),
        external=SimpleNamespace(synapses_per_neuron=100.0, rate_per_synapse_hz=rate,
                                 weight_mv=0.3),
        timestep_ms=1.0,
        duration_s=DURATION_S[index] if duration_s is None else duration_s,
        seed=seed, record_raster=True)
