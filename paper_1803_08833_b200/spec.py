"""Run description types, mirrored from the reference so the drop-in needs no
reference install on the GPU host.

Field names, units, defaults and validation follow the reference classes
field for field, so a reference ``SimConfig`` and one built from this module
are interchangeable: every consumer in this package reads attributes only
(duck typing) and never checks the class.

    GridSpec          corticarc/connectivity.py:62-113
    KernelSpec        corticarc/connectivity.py:116-156
    SynapseGenSpec    corticarc/connectivity.py:312-354
    NeuronParams      corticarc/model.py:44-86
    ExternalInputSpec corticarc/engine.py:65-88
    SimConfig         corticarc/engine.py:91-121
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "GridSpec", "KernelSpec", "SynapseGenSpec", "NeuronParams",
    "ExternalInputSpec", "SimConfig", "MemoryBudgetError",
]


class MemoryBudgetError(ValueError):
    """Estimated memory exceeds the configured budget; nothing allocated
    (same contract as corticarc/engine.py:61-62)."""


@dataclass(frozen=True)
class GridSpec:
    """nx*ny columns of ``neurons_per_column`` neurons; excitatory cells take
    the first floor(fraction*n) local slots of every column."""

    nx: int
    ny: int
    neurons_per_column: int = 1240
    excitatory_fraction: float = 0.8
    spacing_alpha: float = 100.0   # um

    def __post_init__(self):
        if min(self.nx, self.ny) < 1:
            raise ValueError("grid needs at least one column per axis")
        if self.neurons_per_column < 1:
            raise ValueError("neurons_per_column must be positive")
        if not 0.0 < self.excitatory_fraction <= 1.0:
            raise ValueError("excitatory_fraction must be in (0, 1]")
        if self.spacing_alpha <= 0:
            raise ValueError("spacing_alpha must be positive")

    @property
    def n_columns(self) -> int:
        return self.nx * self.ny

    @property
    def n_neurons(self) -> int:
        return self.nx * self.ny * self.neurons_per_column

    @property
    def n_excitatory_per_column(self) -> int:
        return int(math.floor(self.excitatory_fraction * self.neurons_per_column))

    def column_index(self, ix: int, iy: int) -> int:
        return iy * self.nx + ix

    def column_coords(self, col: int):
        return col % self.nx, col // self.nx

    def gid_range(self, col: int):
        return col * self.neurons_per_column, (col + 1) * self.neurons_per_column

    def column_of(self, gid: int) -> int:
        return gid // self.neurons_per_column

    def local_index(self, gid: int) -> int:
        return gid % self.neurons_per_column

    def is_excitatory(self, gid) -> np.ndarray:
        return (np.asarray(gid) % self.neurons_per_column) < self.n_excitatory_per_column


@dataclass(frozen=True)
class KernelSpec:
    """Lateral decay law p(r) (Gaussian or exponential) plus the r=0 rule."""

    kind: str
    amplitude_A: float
    scale: float
    cutoff_p: float = 1e-3
    local_p: float = 0.8

    def __post_init__(self):
        if self.kind not in ("gaussian", "exponential"):
            raise ValueError(f"unknown kernel kind {self.kind!r}")
        if not 0.0 < self.amplitude_A <= 1.0:
            raise ValueError("amplitude_A must be in (0, 1]")
        if self.scale <= 0:
            raise ValueError("scale must be positive")
        if self.cutoff_p <= 0:
            raise ValueError("cutoff_p must be positive")
        if not 0.0 <= self.local_p <= 1.0:
            raise ValueError("local_p must be a probability")

    @classmethod
    def gaussian(cls, amplitude_A: float = 0.05, sigma: float = 100.0, **kw):
        return cls(kind="gaussian", amplitude_A=amplitude_A, scale=sigma, **kw)

    @classmethod
    def exponential(cls, amplitude_A: float = 0.03, lam: float = 290.0, **kw):
        return cls(kind="exponential", amplitude_A=amplitude_A, scale=lam, **kw)

    def cutoff_distance(self) -> float:
        if self.cutoff_p >= self.amplitude_A:
            return 0.0
        ln_ratio = math.log(self.amplitude_A / self.cutoff_p)
        if self.kind == "gaussian":
            return self.scale * math.sqrt(2.0 * ln_ratio)
        return self.scale * ln_ratio


@dataclass(frozen=True)
class SynapseGenSpec:
    """Weight law N(J, sd_frac*|J|) sign-clipped; delay law in ms quantised
    to steps and clamped to [1, d_max_steps]."""

    j_exc_exc: float = 0.4
    j_exc_inh: float = 0.4
    j_inh_exc: float = -1.6
    j_inh_inh: float = -1.6
    weight_sd_frac: float = 0.25
    delay_kind: str = "uniform"
    delay_min_ms: float = 1.0
    delay_max_ms: float = 8.0
    delay_mean_ms: float = 3.0
    timestep_ms: float = 1.0
    d_max_steps: int = 8

    def __post_init__(self):
        if self.delay_kind not in ("uniform", "exponential"):
            raise ValueError(f"unknown delay kind {self.delay_kind!r}")
        if self.timestep_ms <= 0:
            raise ValueError("timestep_ms must be positive")
        if self.d_max_steps < 1:
            raise ValueError("d_max_steps must be >= 1")
        if self.delay_kind == "uniform" and not 0 < self.delay_min_ms <= self.delay_max_ms:
            raise ValueError("need 0 < delay_min_ms <= delay_max_ms")
        if self.delay_kind == "exponential" and self.delay_mean_ms <= 0:
            raise ValueError("delay_mean_ms must be positive")
        if self.j_exc_exc < 0 or self.j_exc_inh < 0:
            raise ValueError("excitatory mean weights must be >= 0")
        if self.j_inh_exc > 0 or self.j_inh_inh > 0:
            raise ValueError("inhibitory mean weights must be <= 0")


@dataclass(frozen=True)
class NeuronParams:
    """LIF + spike-frequency-adaptation constants of one population.
    Inhibitory populations run with g_c = alpha_c = 0 (model.py:73-77)."""

    tau_m: float = 20.0
    C_m: float = 1.0
    E: float = -65.0
    tau_c: float = 150.0
    g_c: float = 0.5
    V_theta: float = -50.0
    V_r: float = -65.0
    tau_arp: float = 2.0
    alpha_c: float = 1.0
    is_excitatory: bool = True

    def __post_init__(self):
        if self.tau_m <= 0 or self.tau_c <= 0 or self.C_m <= 0:
            raise ValueError("tau_m, tau_c and C_m must be positive")
        if self.tau_arp < 0:
            raise ValueError("tau_arp must be non-negative")
        if not self.V_r < self.V_theta:
            raise ValueError("V_r must lie below V_theta")
        if not self.E < self.V_theta:
            raise ValueError("E must lie below V_theta (no spontaneous firing)")
        if not self.is_excitatory:
            object.__setattr__(self, "g_c", 0.0)
            object.__setattr__(self, "alpha_c", 0.0)

    @property
    def sfa_over_cm(self) -> float:
        return self.g_c / self.C_m


@dataclass(frozen=True)
class ExternalInputSpec:
    """Independent Poisson afferents, fixed weight."""

    synapses_per_neuron: float = 800.0
    rate_per_synapse_hz: float = 3.0
    weight_mv: float = 0.2

    def __post_init__(self):
        if min(self.synapses_per_neuron, self.rate_per_synapse_hz, self.weight_mv) < 0:
            raise ValueError("external input parameters must be non-negative")

    def mean_per_step(self, timestep_ms: float) -> float:
        # evaluation order matters for bit parity of exp(-lambda): engine.py:87-88
        return self.synapses_per_neuron * self.rate_per_synapse_hz * timestep_ms * 1e-3


@dataclass(frozen=True)
class SimConfig:
    grid: GridSpec
    kernel: KernelSpec
    genspec: SynapseGenSpec = SynapseGenSpec()
    exc_params: NeuronParams = NeuronParams(is_excitatory=True)
    inh_params: NeuronParams = NeuronParams(is_excitatory=False)
    external: ExternalInputSpec = ExternalInputSpec()
    timestep_ms: float = 1.0
    duration_s: float = 1.0
    seed: int = 1
    record_raster: bool = True
    memory_budget_bytes: int = 4 << 30

    def __post_init__(self):
        if self.timestep_ms <= 0:
            raise ValueError("timestep_ms must be positive")
        if self.duration_s < 0:
            raise ValueError("duration_s must be non-negative")
        if self.genspec.timestep_ms != self.timestep_ms:
            raise ValueError("genspec timestep differs from simulation timestep")
        if self.d_max < 1:
            raise ValueError("need d_max >= 1")

    @property
    def d_max(self) -> int:
        return self.genspec.d_max_steps

    @property
    def n_steps(self) -> int:
        return int(round(self.duration_s * 1000.0 / self.timestep_ms))
