"""Statistical validation of the GPU connectivity generator at scale (BASELINE
north star): per-target-column synapse counts within 0.5 % of the layout
expectation, and the lateral-distance distribution matching it (KS p > 0.01,
chi-square p > 0.01).  The generator is bit-exact with the reference on the
golden networks (test_gpu_parity.py); these tests cover the sizes the reference
cannot build.  Expected counts: source column cs contributes, to target column
ct, 992 excitatory sources x sum of its layout blocks' p over ct's 1240 targets
(1239 in its own column: no autapse) plus, in its own column, 248 inhibitory
sources x local_p x 1239 (connectivity.py:357-392)."""

import numpy as np
import pytest



def expected_pairs(grid, kernel):
    from paper_1803_08833_b200.geometry import layout_blocks
    n, ne = grid.neurons_per_column, grid.n_excitatory_per_column
    blk_col, blk_p, blk_count = layout_blocks(grid, kernel)
    E = np.zeros((grid.n_columns, grid.n_columns))
    for cs in range(grid.n_columns):
        k = np.arange(blk_count[cs])
        np.add.at(E[cs], blk_col[cs, k], ne * blk_p[cs, k] * (n - (k == 0)))
        E[cs, cs] += (n - ne) * kernel.local_p * (n - 1)
    return E


def observed_pairs(net, grid):
    import torch
    n = grid.neurons_per_column
    ln = net.row_off[1:] - net.row_off[:-1]
    src = torch.repeat_interleave(torch.arange(ln.numel(), device=ln.device), ln)
    pair = (src // n) * grid.n_columns + net.syn_tgt.long() // n
    return torch.bincount(pair, minlength=grid.n_columns ** 2).cpu().numpy().reshape(
        grid.n_columns, grid.n_columns)


def _dist_tests(obs, E, grid):
    from scipy import stats
    xy = np.array([grid.column_coords(c) for c in range(grid.n_columns)])
    d2 = ((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1)
    keys = np.unique(d2[E > 0])
    o = np.array([obs[(d2 == k) & (E > 0)].sum() for k in keys], dtype=np.float64)
    e = np.array([E[(d2 == k) & (E > 0)].sum() for k in keys])
    e *= o.sum() / e.sum()
    D = np.max(np.abs(np.cumsum(o) / o.sum() - np.cumsum(e) / e.sum()))
    return stats.kstwo.sf(D, int(o.sum())), stats.chisquare(o, e).pvalue


@pytest.mark.parametrize("kind", ["gaussian", "exponential"])
def test_expected_counts_model_on_the_oracle_generator(kind):
    """The expectation model above, checked on the CPU restatement of the
    reference generator (oracle, bit-exact with the reference) at small size."""
    from oracle import corticarc_oracle as O
    from paper_1803_08833_b200 import spec as S
    grid = S.GridSpec(nx=5, ny=4, neurons_per_column=160)
    kernel = S.KernelSpec.gaussian() if kind == "gaussian" else S.KernelSpec.exponential()
    gen = S.SynapseGenSpec(j_exc_exc=0.3, j_exc_inh=0.3, j_inh_exc=-1.2, j_inh_inh=-1.2)
    net = O.build_shard(grid, kernel, gen, 7)
    n = grid.neurons_per_column
    src = np.repeat(net.sources.astype(np.int64), np.diff(net.offsets))
    pair = (src // n) * grid.n_columns + net.target_local.astype(np.int64) // n
    obs = np.bincount(pair, minlength=grid.n_columns ** 2).reshape(grid.n_columns, -1)
    E = expected_pairs(grid, kernel)
    assert obs[E == 0].sum() == 0
    assert np.max(np.abs(obs.sum(0) / E.sum(0) - 1.0)) < 0.02       # ~26 k synapses/column
    p_ks, p_chi = _dist_tests(obs, E, grid)
    assert p_ks > 0.01 and p_chi > 0.01


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["config1_gauss", "exp_12x12"])
def test_generator_column_counts_and_distance_distribution(cuda, case):
    from paper_1803_08833_b200 import baseline_config
    from paper_1803_08833_b200.network import build_b200
    from dataclasses import replace
    from paper_1803_08833_b200 import spec as S
    cfg = baseline_config(1, "calibrated")
    if case == "exp_12x12":
        cfg = replace(cfg, grid=S.GridSpec(nx=12, ny=12, neurons_per_column=1240),
                      kernel=baseline_config(2).kernel)
    grid = cfg.grid
    net = build_b200(cfg)
    obs = observed_pairs(net, grid)
    E = expected_pairs(grid, cfg.kernel)
    assert obs[E == 0].sum() == 0                       # no synapse outside the layout
    rel = obs.sum(0) / E.sum(0) - 1.0
    assert np.max(np.abs(rel)) < 0.005, np.max(np.abs(rel))
    p_ks, p_chi = _dist_tests(obs, E, grid)
    assert p_ks > 0.01 and p_chi > 0.01, (p_ks, p_chi)
