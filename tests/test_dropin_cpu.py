"""Host-side drop-in pieces that need no GPU: the raster writer against the
reference's (baseline/_ref), and the reference's SimConfig being accepted by
the package's config consumers."""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def cc():
    if not os.path.isdir(os.path.join(REF, "corticarc")):
        pytest.skip("reference package not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import corticarc
    return corticarc


def test_write_raster_matches_reference(cc, tmp_path):
    from corticarc.engine import write_raster as ref_write
    from paper_1803_08833_b200.engine import write_raster
    r = np.random.default_rng(3)
    g = r.integers(0, 5000, 400).astype(np.uint64)
    t = np.round(r.uniform(0, 100, 400), 3)
    t[10:20] = t[0]                                     # ties broken by gid
    write_raster(tmp_path / "a", g, t)
    ref_write(tmp_path / "b", g, t)
    assert (tmp_path / "a").read_bytes() == (tmp_path / "b").read_bytes()


def test_reference_simconfig_drives_host_logic(cc):
    """The engine's host-side consumers accept the reference's SimConfig
    (duck-typed spec): memory estimate, bin sizing, spike bound."""
    from corticarc.connectivity import GridSpec, KernelSpec
    from corticarc.engine import SimConfig, estimate_worker_bytes as ref_est
    from paper_1803_08833_b200.engine import (_spikes_per_step_bound, default_bin_cap,
                                              estimate_worker_bytes)
    cfg = SimConfig(grid=GridSpec(nx=4, ny=4, neurons_per_column=40), kernel=KernelSpec.gaussian())
    assert estimate_worker_bytes(cfg, 2) == ref_est(cfg, 2)
    assert default_bin_cap(cfg) >= 2048 and _spikes_per_step_bound(cfg) >= 1
