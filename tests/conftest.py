import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def golden_npz(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def golden_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def config_from_json(d):
    """Rebuild a package SimConfig from the dataclass dict stored in run_*.json."""
    from paper_1803_08833_b200 import spec as S
    return S.SimConfig(
        grid=S.GridSpec(**d["grid"]), kernel=S.KernelSpec(**d["kernel"]),
        genspec=S.SynapseGenSpec(**d["genspec"]),
        exc_params=S.NeuronParams(**d["exc_params"]),
        inh_params=S.NeuronParams(**d["inh_params"]),
        external=S.ExternalInputSpec(**d["external"]),
        timestep_ms=d["timestep_ms"], duration_s=d["duration_s"], seed=d["seed"],
        record_raster=d["record_raster"], memory_budget_bytes=d["memory_budget_bytes"])


def golden_run(name):
    meta = golden_json(f"run_{name}.json")
    arr = golden_npz(f"run_{name}.npz")
    return config_from_json(meta["config"]), meta, arr


def tiny_config(nx=4, ny=4, n_col=40, kind="gaussian", duration_s=0.1, seed=11, **over):
    """pkg/tests/conftest.py:30-47 equivalent."""
    from paper_1803_08833_b200 import spec as S
    kernel = S.KernelSpec.gaussian() if kind == "gaussian" else S.KernelSpec.exponential()
    kw = dict(grid=S.GridSpec(nx=nx, ny=ny, neurons_per_column=n_col), kernel=kernel,
              genspec=S.SynapseGenSpec(j_exc_exc=1.0, j_exc_inh=1.0,
                                       j_inh_exc=-4.0, j_inh_inh=-4.0),
              exc_params=S.NeuronParams(is_excitatory=True),
              inh_params=S.NeuronParams(is_excitatory=False),
              external=S.ExternalInputSpec(synapses_per_neuron=80,
                                           rate_per_synapse_hz=20.0, weight_mv=0.5),
              duration_s=duration_s, seed=seed)
    kw.update(over)
    return S.SimConfig(**kw)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_1803_08833_b200 import _lib
    return _lib.lib()
