"""Drop-in check against the reference package itself (corticarc, installed
offline into baseline/_ref).

The reference's own harnesses drive the B200 engine through the runner seam
`runner(SimConfig, workers) -> RunResult` (metrics.scaling_harness,
calibration_sweep, report_from_run, emit_csv; metrics.py:94-376) with the
reference's own SimConfig objects, and the results equal the reference's
own run of the same config (engine.run, engine.py:449-480)."""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def cc():
    if not os.path.isdir(os.path.join(REF, "corticarc")):
        pytest.skip("reference package not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import corticarc
    return corticarc


def _ref_config(cc, duration_s=0.1, rate=20.0):
    """The reference's own tiny test network (pkg/tests/conftest.py:30-47 shape)."""
    from corticarc.connectivity import GridSpec, KernelSpec, SynapseGenSpec
    from corticarc.engine import ExternalInputSpec, SimConfig
    return SimConfig(grid=GridSpec(nx=4, ny=4, neurons_per_column=40),
                     kernel=KernelSpec.gaussian(),
                     genspec=SynapseGenSpec(j_exc_exc=1.0, j_exc_inh=1.0, j_inh_exc=-4.0,
                                            j_inh_inh=-4.0),
                     external=ExternalInputSpec(synapses_per_neuron=80,
                                                rate_per_synapse_hz=rate, weight_mv=0.5),
                     duration_s=duration_s, seed=11)


def test_reference_simconfig_equals_reference_run(cc, cuda):
    import paper_1803_08833_b200 as b2
    from corticarc.engine import run as ref_run
    cfg = _ref_config(cc)
    ours = b2.runner(cfg, 1)
    ref = ref_run(cfg, 1)
    assert ours.construction_checksum == ref.construction_checksum
    assert ours.recurrent_synapses == ref.recurrent_synapses
    assert ours.n_spikes == ref.n_spikes > 0
    assert np.array_equal(ours.raster_gids, ref.raster_gids)
    assert np.array_equal(ours.raster_times.view(np.uint64), ref.raster_times.view(np.uint64))
    assert ours.raster_checksum == ref.raster_checksum
    assert ours.recurrent_events == ref.recurrent_events
    assert ours.external_events == ref.external_events
    assert set(ours.substep_seconds) >= {"deliver", "expand", "external", "integrate"}


def test_reference_scaling_harness_and_csv(cc, cuda):
    """metrics.scaling_harness(cfg, [1, 2, 4], runner=b200.runner): the B200
    runner spawns its workers for k > 1; every row has the same events
    (partition invariance), and the CSV round-trips through parse_csv."""
    import paper_1803_08833_b200 as b2
    from corticarc import metrics as M
    cfg = _ref_config(cc)
    table = M.scaling_harness(cfg, [1, 2, 4], runner=b2.runner)
    assert not table.failures, table.failures
    assert [r.workers for r in table.rows] == [1, 2, 4]
    assert len({r.recurrent_events for r in table.rows}) == 1
    assert len({r.external_events for r in table.rows}) == 1
    assert len({rep.n_spikes for rep in table.reports}) == 1
    csv = M.emit_csv(table)
    back = M.parse_csv(csv)
    assert [(r.workers, r.recurrent_events) for r in back] == \
        [(r.workers, r.recurrent_events) for r in table.rows]
    assert table.rows[0].speedup == 1.0


def test_reference_calibration_sweep_and_report(cc, cuda):
    import paper_1803_08833_b200 as b2
    from corticarc import metrics as M
    from corticarc.engine import run as ref_run
    cfg = _ref_config(cc, duration_s=0.05)
    rates = [10.0, 30.0]
    ours = M.calibration_sweep(cfg, rates, runner=b2.runner)
    ref = M.calibration_sweep(cfg, rates, runner=ref_run)
    assert ours == ref                                   # identical mean rates
    a, b = M.report_from_run(b2.runner(cfg, 1)), M.report_from_run(ref_run(cfg, 1))
    for f in ("grid_label", "kernel_kind", "worker_count", "sim_seconds", "n_neurons",
              "recurrent_synapses", "recurrent_events", "external_events", "n_spikes"):
        assert getattr(a, f) == getattr(b, f), f
    assert M.normalized_cost(a) > 0


def test_write_raster_byte_identical(cc, cuda, tmp_path):
    import paper_1803_08833_b200 as b2
    from corticarc.engine import write_raster as ref_write
    res = b2.runner(_ref_config(cc), 1)
    ours, ref = tmp_path / "ours.tsv", tmp_path / "ref.tsv"
    b2.write_raster(ours, res.raster_gids, res.raster_times)
    ref_write(ref, res.raster_gids, res.raster_times)
    assert ours.read_bytes() == ref.read_bytes() and len(ours.read_bytes()) > 0
