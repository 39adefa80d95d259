"""B200-native engine for the per-millisecond loop of the DPSNN cortical
simulator (arXiv 1803.08833), drop-in for the reference package `corticarc`.

Public surface (mirrors corticarc's names where they exist):

    GridSpec, KernelSpec, SynapseGenSpec, NeuronParams, ExternalInputSpec,
    SimConfig, MemoryBudgetError          run description (spec.py)
    build_b200, import_csr, export_csr    network build on the GPU, reference-format
                                          CSR in and out (network.py)
    run_b200, Simulator, RunResult        simulate (engine.py); workers > 1 runs one
                                          process per worker (distributed.py)
    write_raster                          the reference's raster file format
    runner                                the `runner(config, workers)` seam of
                                          metrics.scaling_harness / calibration_sweep
    baseline_config                       BASELINE.json configs 0-4 (presets.py)
"""

from .spec import (ExternalInputSpec, GridSpec, KernelSpec, MemoryBudgetError,
                   NeuronParams, SimConfig, SynapseGenSpec)
from .presets import baseline_config

__version__ = "0.1.0"

__all__ = [
    "GridSpec", "KernelSpec", "SynapseGenSpec", "NeuronParams", "ExternalInputSpec",
    "SimConfig", "MemoryBudgetError", "baseline_config", "build_b200", "import_csr",
    "export_csr",
    "run_b200", "Simulator", "RunResult", "runner", "write_raster", "__version__",
]


def __getattr__(name):
    # device-facing modules load lazily so that config-only use works on CPU hosts
    if name in ("build_b200", "import_csr", "export_csr", "DeviceNetwork"):
        from . import network
        return getattr(network, name)
    if name in ("run_b200", "Simulator", "RunResult", "write_raster"):
        from . import engine
        return getattr(engine, name)
    if name == "runner":
        from .engine import run_b200
        return run_b200
    raise AttributeError(name)
