"""Generate tests/golden/* by running the REFERENCE itself (test infrastructure).

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py [--big]

Imports corticarc read-only from /root/reference/pkg/src and records its
outputs as small .npz fixtures.  The reference is never modified; probe
traces use a harness-side wrapper around NeuronBlock.integrate_sorted
(model.py:289-337), the hook point SURVEY.md 7.1 names.  `--big` adds the
1 s config-0 rasters (minutes of reference CPU time).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import corticarc  # noqa: E402
from corticarc import connectivity as rc  # noqa: E402
from corticarc import engine as re_  # noqa: E402
from corticarc import model as rm  # noqa: E402
from corticarc import network as rn  # noqa: E402
from corticarc import rng as rr  # noqa: E402
from corticarc.partition import map_columns_to_workers  # noqa: E402
from corticarc.transport import InProcessGroup  # noqa: E402

from paper_1803_08833_b200 import presets  # noqa: E402


def to_ref(cfg):
    """Rebuild a package SimConfig with the reference's own classes."""
    g, k, s, x = cfg.grid, cfg.kernel, cfg.genspec, cfg.external
    def np_(p):
        return rm.NeuronParams(tau_m=p.tau_m, C_m=p.C_m, E=p.E, tau_c=p.tau_c, g_c=p.g_c,
                               V_theta=p.V_theta, V_r=p.V_r, tau_arp=p.tau_arp,
                               alpha_c=p.alpha_c, is_excitatory=p.is_excitatory)
    return re_.SimConfig(
        grid=rc.GridSpec(nx=g.nx, ny=g.ny, neurons_per_column=g.neurons_per_column,
                         excitatory_fraction=g.excitatory_fraction,
                         spacing_alpha=g.spacing_alpha),
        kernel=rc.KernelSpec(kind=k.kind, amplitude_A=k.amplitude_A, scale=k.scale,
                             cutoff_p=k.cutoff_p, local_p=k.local_p),
        genspec=rc.SynapseGenSpec(j_exc_exc=s.j_exc_exc, j_exc_inh=s.j_exc_inh,
                                  j_inh_exc=s.j_inh_exc, j_inh_inh=s.j_inh_inh,
                                  weight_sd_frac=s.weight_sd_frac, delay_kind=s.delay_kind,
                                  delay_min_ms=s.delay_min_ms, delay_max_ms=s.delay_max_ms,
                                  delay_mean_ms=s.delay_mean_ms, timestep_ms=s.timestep_ms,
                                  d_max_steps=s.d_max_steps),
        exc_params=np_(cfg.exc_params), inh_params=np_(cfg.inh_params),
        external=re_.ExternalInputSpec(synapses_per_neuron=x.synapses_per_neuron,
                                       rate_per_synapse_hz=x.rate_per_synapse_hz,
                                       weight_mv=x.weight_mv),
        timestep_ms=cfg.timestep_ms, duration_s=cfg.duration_s, seed=cfg.seed,
        memory_budget_bytes=cfg.memory_budget_bytes)


# ------------------------------------------------------------------ configs
def tiny(nx=4, ny=4, n_col=40, kind="gaussian", duration_s=0.1, seed=11, **over):
    """The reference's tiny_config fixture (pkg/tests/conftest.py:30-47)."""
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


def cfg_to_json(cfg):
    from dataclasses import asdict
    return json.dumps(asdict(cfg), sort_keys=True)


# ------------------------------------------------------------------ fixtures
def gold_rng():
    out = {}
    xs = np.array([0, 1, 2, 0xDEADBEEF, 2**63, 2**64 - 1], dtype=np.uint64)
    out["sm_in"] = xs
    out["sm_out"] = rr.splitmix64(xs)
    a = np.array([0, 17, 4959, 79359, 11427839], dtype=np.uint64)
    out["cu_a"] = a
    out["cu_ext"] = rr.counter_uniforms(3, rr.Purpose.EXTERNAL, a[:, None], 250,
                                        np.arange(8, dtype=np.uint64)[None, :])
    out["cu_time"] = rr.counter_uniforms(9, rr.Purpose.EXTERNAL_TIME, a[:, None], 7,
                                         np.arange(8, dtype=np.uint64)[None, :])
    out["cu_init"] = rr.counter_uniforms(1, rr.Purpose.INIT_STATE, a, 0, 0)
    keys = [(1, 1, 0), (1, 2, 5), (7, 3, 12), (11, 1, 79359), (2**40 + 3, 2, 123456)]
    out["ph_keys"] = np.array(keys, dtype=np.uint64)
    out["ph_raw"] = np.stack([rr.stream(s, p, a_).bit_generator.random_raw(64)
                              for s, p, a_ in keys])
    out["ph_random"] = np.stack([rr.stream(s, p, a_).random(37) for s, p, a_ in keys])
    out["ph_normal"] = np.stack([rr.stream(s, p, a_).standard_normal(2000) for s, p, a_ in keys])
    out["ph_uniform"] = np.stack([rr.stream(s, p, a_).uniform(1.0, 20.0, 64) for s, p, a_ in keys])
    out["ph_expo"] = np.stack([rr.stream(s, p, a_).exponential(3.0, 2000) for s, p, a_ in keys])
    np.savez_compressed(os.path.join(OUT, "rng.npz"), **out)


def gold_decay():
    rs = np.random.default_rng(5)
    n = 400
    V0 = rs.uniform(-80, 25, n)
    c0 = rs.uniform(0, 10, n)
    dt = np.concatenate([rs.uniform(0, 5, n // 2), np.exp(rs.uniform(-20, 9, n // 2))])
    tau_c = rs.choice([20.0, 150.0, 300.0, 20.0 + 1e-9, 5.0], n)
    Vo, co = [], []
    for i in range(n):
        p = rm.NeuronParams(is_excitatory=True, tau_c=float(tau_c[i]))
        st = rm.decay_state(rm.NeuronState(V=float(V0[i]), c=float(c0[i])), p, float(dt[i]))
        Vo.append(st.V); co.append(st.c)
    np.savez_compressed(os.path.join(OUT, "decay.npz"), V0=V0, c0=c0, dt=dt, tau_c=tau_c,
                        V=np.array(Vo), c=np.array(co))


def gold_poisson():
    out = {}
    gids = np.arange(2000, dtype=np.uint64) * 37 + 5
    for lam in (0.09, 1.6, 3.5, 24.0):
        key = str(lam).replace(".", "p")
        out[f"counts_{key}"] = np.stack([re_._poisson_counts(4, gids, t, lam) for t in (0, 1, 999)])
    out["gids"] = gids
    spec = re_.ExternalInputSpec(synapses_per_neuron=100, rate_per_synapse_hz=35.0, weight_mv=0.3)
    w, tm = re_._external_events(1, gids, 321, spec, 1.0)
    out["ext_which"], out["ext_times"] = w, tm
    np.savez_compressed(os.path.join(OUT, "poisson.npz"), **out)


def gold_connectivity():
    """Per-source draws on small grids plus whole-network CSR and checksums."""
    out = {}
    cases = {
        "gauss": (rc.GridSpec(nx=6, ny=5, neurons_per_column=40), rc.KernelSpec.gaussian(),
                  rc.SynapseGenSpec(j_exc_exc=1.0, j_exc_inh=1.0, j_inh_exc=-4.0,
                                    j_inh_inh=-4.0), 23),
        "exp": (rc.GridSpec(nx=7, ny=6, neurons_per_column=24), rc.KernelSpec.exponential(),
                rc.SynapseGenSpec(), 5),
        "expdelay": (rc.GridSpec(nx=3, ny=3, neurons_per_column=30), rc.KernelSpec.gaussian(),
                     rc.SynapseGenSpec(delay_kind="exponential", delay_mean_ms=3.0,
                                       d_max_steps=12), 2),
    }
    meta = {}
    for name, (grid, kernel, gen, seed) in cases.items():
        group = InProcessGroup(1)
        pmap = map_columns_to_workers(grid, 1)
        net = rn.construct_network(grid, kernel, gen, pmap, seed, group.endpoint(0))
        inc = net.incoming
        out[f"{name}_sources"] = inc.sources
        out[f"{name}_offsets"] = inc.offsets
        out[f"{name}_target"] = inc.target_local
        out[f"{name}_delay"] = inc.delay
        out[f"{name}_weight"] = inc.weight
        meta[name] = dict(checksum=int(net.stats.checksum), n=int(inc.n_synapses),
                          grid=[grid.nx, grid.ny, grid.neurons_per_column],
                          kernel=[kernel.kind, kernel.amplitude_A, kernel.scale,
                                  kernel.cutoff_p, kernel.local_p],
                          gen=[gen.j_exc_exc, gen.j_exc_inh, gen.j_inh_exc, gen.j_inh_inh,
                               gen.weight_sd_frac, gen.delay_kind, gen.delay_min_ms,
                               gen.delay_max_ms, gen.delay_mean_ms, gen.timestep_ms,
                               gen.d_max_steps],
                          seed=seed)
        # 4-worker checksum equals 1-worker (partition invariance of construction)
        group4 = InProcessGroup(4)
        pm4 = map_columns_to_workers(grid, 4)
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(4) as ex:
            nets = list(ex.map(lambda r: rn.construct_network(grid, kernel, gen, pm4, seed,
                                                              group4.endpoint(r)), range(4)))
        meta[name]["checksum_w4"] = sum(int(x.stats.checksum) for x in nets) % 2**64
    # config-0 sized network (2x2x1240, literal BASELINE parameters): checksum only
    for regime in ("literal", "calibrated"):
        cfg = to_ref(presets.baseline_config(0, regime))
        group = InProcessGroup(1)
        pmap = map_columns_to_workers(cfg.grid, 1)
        net = rn.construct_network(cfg.grid, cfg.kernel, cfg.genspec, pmap, cfg.seed,
                                   group.endpoint(0))
        counts = np.diff(net.incoming.offsets)
        meta[f"config0_{regime}"] = dict(checksum=int(net.stats.checksum),
                                         n=int(net.incoming.n_synapses),
                                         row_len_sum_first100=int(counts[:100].sum()))
    np.savez_compressed(os.path.join(OUT, "connectivity.npz"), **out)
    with open(os.path.join(OUT, "connectivity.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


class Probe:
    """Harness-side wrapper recording probed neuron state after every
    integrate_sorted call (one call per step at workers=1)."""

    def __init__(self, probes, dt):
        self.probes, self.dt = np.asarray(probes), dt
        self.state, self.vend = [], []
        self.orig = rm.NeuronBlock.integrate_sorted

    def __enter__(self):
        probe = self
        def wrapped(block, tgt, t_ev, w_ev):
            res = probe.orig(block, tgt, t_ev, w_ev)
            p = probe.probes
            probe.state.append(np.stack([block.V[p], block.c[p], block.last_t[p],
                                         block.refr_until[p]], axis=1))
            t_end = (len(probe.state)) * probe.dt
            V, c, last, ru = block.V.copy(), block.c.copy(), block.last_t.copy(), block.refr_until.copy()
            block.advance(p, np.full(len(p), t_end))
            probe.vend.append(block.V[p].copy())
            block.V[:], block.c[:], block.last_t[:], block.refr_until[:] = V, c, last, ru
            return res
        rm.NeuronBlock.integrate_sorted = wrapped
        return self

    def __exit__(self, *a):
        rm.NeuronBlock.integrate_sorted = self.orig


def gold_run(name, cfg, probes=None, workers=1):
    t0 = time.time()
    rcfg = to_ref(cfg)
    if probes is not None:
        with Probe(probes, cfg.timestep_ms) as pr:
            res = re_.run(rcfg, 1)
        extra = dict(probe_ids=np.asarray(probes), probe_state=np.stack(pr.state),
                     probe_vend=np.stack(pr.vend))
    else:
        res = re_.run_multiprocess(rcfg, workers) if workers > 1 else re_.run(rcfg, 1)
        extra = {}
    np.savez_compressed(os.path.join(OUT, f"run_{name}.npz"),
                        raster_gids=res.raster_gids, raster_times=res.raster_times, **extra)
    meta = dict(n_spikes=int(res.n_spikes), recurrent_events=int(res.recurrent_events),
                external_events=int(res.external_events),
                recurrent_synapses=int(res.recurrent_synapses),
                construction_checksum=int(res.construction_checksum),
                raster_checksum=int(res.raster_checksum),
                sim_seconds_wall=float(res.sim_seconds_wall), workers=workers,
                config=json.loads(cfg_to_json(cfg)), ref_seconds=time.time() - t0)
    with open(os.path.join(OUT, f"run_{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(name, meta["n_spikes"], hex(meta["raster_checksum"]), f"{time.time()-t0:.1f}s",
          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    np.random.seed(0)
    jobs = {
        "rng": gold_rng, "decay": gold_decay, "poisson": gold_poisson,
        "connectivity": gold_connectivity,
        "runs": lambda: [
            gold_run("tiny_gauss", tiny(), probes=np.arange(0, 640, 10)),
            gold_run("tiny_exp", tiny(kind="exponential", n_col=30, duration_s=0.1, seed=3),
                     probes=np.arange(0, 480, 7)[:64]),
            gold_run("tiny_gauss_long", tiny(nx=3, ny=3, duration_s=0.3, seed=5)),
            gold_run("tiny_quiet", tiny(nx=2, ny=2, external=__import__(
                "paper_1803_08833_b200.spec", fromlist=["x"]).ExternalInputSpec(
                synapses_per_neuron=80, rate_per_synapse_hz=0.0, weight_mv=0.5))),
            gold_run("config0_literal_0p2", presets.baseline_config(0, "literal", duration_s=0.2)),
            gold_run("config0_cal_0p1", presets.baseline_config(0, "calibrated", duration_s=0.1),
                     probes=np.arange(0, 4960, 77)[:64]),
        ],
    }
    # 64-neuron probe traces over half a second of BASELINE config 0 (the north
    # star's "membrane-potential trace of 64 probed neurons" criterion)
    jobs["probes_long"] = lambda: [
        gold_run("config0_cal_0p5", presets.baseline_config(0, "calibrated", duration_s=0.5),
                 probes=np.arange(0, 4960, 77)[:64]),
    ]
    if a.big:
        jobs["big"] = lambda: [
            gold_run("config0_literal", presets.baseline_config(0, "literal"), workers=4),
            gold_run("config0_cal", presets.baseline_config(0, "calibrated"), workers=4),
        ]
    for k, fn in jobs.items():
        if a.only and k != a.only:
            continue
        t = time.time()
        fn()
        print(f"[{k}] {time.time()-t:.1f}s", flush=True)


if __name__ == "__main__":
    main()
