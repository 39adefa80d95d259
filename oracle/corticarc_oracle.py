"""CPU ORACLE — test infrastructure only.

A numpy restatement of the reference algorithm for the per-millisecond loop of
`corticarc` (arXiv 1803.08833 DPSNN re-creation).  It exists to CHECK the
CUDA path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import it.  The product path never does.

Pinned against the reference itself: tests/golden/* were produced by
oracle/make_golden.py importing /root/reference/pkg/src/corticarc, and
tests/test_oracle_golden.py checks this module against every fixture
(splitmix64 published vectors, Philox words, ziggurat normals, per-source
synapse draws, construction checksums, Poisson counts, decay closed form,
full-run rasters and probe traces).

Third-party arithmetic: numpy (here 2.3.5) supplies Philox4x64-10 and the
ziggurat `standard_normal` / `uniform` / `exponential` used by the reference
(corticarc/rng.py:42-52, connectivity.py:390-414).  The oracle calls the same
numpy routines; `philox4x64_words` restates Philox so the raw stream is
pinned independently of numpy's Generator.

Each function cites the reference file:line it follows.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

U64 = np.uint64
MASK64 = (1 << 64) - 1
DOMAIN = 0x636F727469636172            # rng.py:28
P_CONNECTIVITY, P_WEIGHT, P_DELAY = 1, 2, 3   # rng.py:33-39
P_INIT_STATE, P_EXTERNAL, P_EXTERNAL_TIME = 4, 5, 7
EXTERNAL_SOURCE_ID = 0xFFFFFFFF        # engine.py:58
POISSON_PAD = 20                       # engine.py:169


# ---------------------------------------------------------------- RNG
def splitmix64(x):
    """rng.py:61-71 (wrapping uint64 arithmetic)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=U64) + U64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> U64(30))) * U64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> U64(27))) * U64(0x94D049BB133111EB)
        return z ^ (z >> U64(31))


def counter_uniforms(seed, purpose, a, b, k):
    """rng.py:74-90: five chained mixes, top 53 bits -> [0,1)."""
    h = splitmix64(U64(seed & MASK64) ^ U64(DOMAIN))
    h = splitmix64(h ^ U64(purpose))
    h = splitmix64(h ^ np.asarray(a, dtype=U64))
    h = splitmix64(h ^ np.asarray(b, dtype=U64))
    h = splitmix64(h ^ np.asarray(k, dtype=U64))
    return (h >> U64(11)) * (1.0 / (1 << 53))


def generator(seed, purpose, a=0, b=0) -> np.random.Generator:
    """rng.py:42-52: Philox4x64 keyed (seed, purpose), counter (0, a, b, DOMAIN)."""
    key = np.array([seed & MASK64, purpose & MASK64], dtype=U64)
    ctr = np.array([0, a & MASK64, b & MASK64, DOMAIN], dtype=U64)
    return np.random.Generator(np.random.Philox(key=key, counter=ctr))


_PH_M0, _PH_M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
_PH_W0, _PH_W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B


def philox4x64_words(seed, purpose, a, n_words, b=0):
    """Independent pure-Python Philox4x64-10 (Salmon et al. 2011): word j of
    the stream behind generator(seed, purpose, a, b) is lane j%4 of block
    j//4, and block i is keyed with counter (i+1, a, b, DOMAIN) because numpy
    increments the 256-bit counter before each block."""
    out = []
    blk = 0
    while len(out) < n_words:
        blk += 1
        c = [blk & MASK64, a & MASK64, b & MASK64, DOMAIN]
        k0, k1 = seed & MASK64, purpose & MASK64
        for _ in range(10):
            p0 = _PH_M0 * c[0]
            p1 = _PH_M1 * c[2]
            hi0, lo0 = p0 >> 64, p0 & MASK64
            hi1, lo1 = p1 >> 64, p1 & MASK64
            c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
            k0 = (k0 + _PH_W0) & MASK64
            k1 = (k1 + _PH_W1) & MASK64
        out.extend(c)
    return out[:n_words]


# ------------------------------------------------------- connectivity
def stencil_active(kernel, grid):
    """connectivity.py:201-228 then Stencil.active (:189-192)."""
    if kernel.cutoff_p >= kernel.amplitude_A:
        r_cut = 0.0
    else:
        ln_ratio = math.log(kernel.amplitude_A / kernel.cutoff_p)
        r_cut = kernel.scale * (math.sqrt(2.0 * ln_ratio) if kernel.kind == "gaussian"
                                else ln_ratio)
    radius = int(math.ceil(r_cut / grid.spacing_alpha)) if r_cut > 0 else 0
    if radius == 0:
        return np.empty((0, 2), dtype=np.int64), np.empty(0)
    ax = np.arange(-radius, radius + 1)
    dj, di = np.meshgrid(ax, ax, indexing="ij")
    di, dj = di.ravel(), dj.ravel()
    keep = ~((di == 0) & (dj == 0))
    di, dj = di[keep], dj[keep]
    r = grid.spacing_alpha * np.hypot(di, dj)
    if kernel.kind == "gaussian":
        p = kernel.amplitude_A * np.exp(-(r * r) / (2.0 * kernel.scale ** 2))
    else:
        p = kernel.amplitude_A * np.exp(-r / kernel.scale)
    p = np.where(p > kernel.cutoff_p, p, 0.0)
    m = p > 0
    return np.column_stack([di, dj])[m], p[m]


def candidates(grid, kernel, col, exc):
    """connectivity.py:357-380: own column first, then in-grid active offsets."""
    n = grid.neurons_per_column
    ix, iy = col % grid.nx, col // grid.nx
    gids = [np.arange(col * n, col * n + n, dtype=np.uint32)]
    ps = [np.full(n, kernel.local_p)]
    if exc:
        offs, probs = stencil_active(kernel, grid)
        for (di, dj), p in zip(offs, probs):
            tx, ty = ix + int(di), iy + int(dj)
            if 0 <= tx < grid.nx and 0 <= ty < grid.ny:
                t0 = (ty * grid.nx + tx) * n
                gids.append(np.arange(t0, t0 + n, dtype=np.uint32))
                ps.append(np.full(n, p))
    return np.concatenate(gids), np.concatenate(ps)


def draw_source(gid, cand_gids, cand_p, grid, gen, seed):
    """connectivity.py:383-417: Bernoulli, weight and delay draws of one source.
    Returns (targets u32, delay u16, weight f32) in layout order."""
    n = grid.neurons_per_column
    exc_n = int(math.floor(grid.excitatory_fraction * n))
    p = cand_p.copy()
    p[gid - (gid // n) * n] = 0.0          # autapse slot (own block is first)
    sel = generator(seed, P_CONNECTIVITY, gid).random(len(p)) < p
    tgt = cand_gids[sel]
    k = int(tgt.size)
    src_exc = (gid % n) < exc_n
    tgt_exc = (tgt.astype(np.int64) % n) < exc_n
    if src_exc:
        j = np.where(tgt_exc, gen.j_exc_exc, gen.j_exc_inh)
    else:
        j = np.where(tgt_exc, gen.j_inh_exc, gen.j_inh_inh)
    z = generator(seed, P_WEIGHT, gid).standard_normal(k)
    w = j * (1.0 + gen.weight_sd_frac * z)
    w = np.maximum(w, 0.0) if src_exc else np.minimum(w, 0.0)
    dg = generator(seed, P_DELAY, gid)
    if gen.delay_kind == "uniform":
        d_ms = dg.uniform(gen.delay_min_ms, gen.delay_max_ms, k)
    else:
        d_ms = dg.exponential(gen.delay_mean_ms, k)
    d = np.clip(np.rint(d_ms / gen.timestep_ms).astype(np.int64), 1, gen.d_max_steps)
    return tgt, d.astype(np.uint16), w.astype(np.float32)


def source_synapses(gid, grid, kernel, gen, seed):
    n = grid.neurons_per_column
    exc = (gid % n) < int(math.floor(grid.excitatory_fraction * n))
    cg, cp = candidates(grid, kernel, gid // n, exc)
    return draw_source(gid, cg, cp, grid, gen, seed)


def wire_mix_sum(src, tgt, delay, flags, weight) -> int:
    """network.py:70-88 over 16 B records (src u32, tgt u32, delay u16,
    flags u16, weight f32): sum of splitmix(lo ^ splitmix(hi)) mod 2^64."""
    if len(src) == 0:
        return 0
    lo = np.asarray(src, U64) | (np.asarray(tgt, U64) << U64(32))
    wbits = np.asarray(weight, np.float32).view(np.uint32).astype(U64)
    hi = (np.asarray(delay, U64) | (np.asarray(flags, U64) << U64(16))
          | (wbits << U64(32)))
    return int(np.sum(splitmix64(lo ^ splitmix64(hi)), dtype=U64))


def raster_checksum(gids, times) -> int:
    """network.py:91-97."""
    if len(gids) == 0:
        return 0
    lo = np.asarray(gids, dtype=U64)
    hi = np.asarray(times, dtype=np.float64).view(U64)
    return int(np.sum(splitmix64(lo ^ splitmix64(hi)), dtype=U64))


@dataclass
class ShardNet:
    """Target-side CSR of one shard (network.py:114-152, 254-271):
    rows keyed by source gid, each row sorted by delay (stable, so layout
    order inside a delay), target stored as the shard-local index."""
    sources: np.ndarray          # u64, ascending
    offsets: np.ndarray          # i64 len(sources)+1
    target_local: np.ndarray     # u32
    delay: np.ndarray            # u16
    weight: np.ndarray           # f32
    checksum: int                # partial construction checksum of records generated here
    n_generated: int


def owned_columns(grid, rank, size):
    """partition.py:83-112 tiling (restated for the oracle's shard runs)."""
    best = None
    for py in range(1, math.isqrt(size) + 1):
        if size % py:
            continue
        px = size // py
        for cx, cy in ((px, py), (py, px)):
            if cx <= grid.nx and cy <= grid.ny:
                key = (abs(cx - cy), -cx, cx, cy)
                best = key if best is None or key < best else best
    px, py = best[2], best[3]
    xs = (np.arange(px + 1) * grid.nx) // px
    ys = (np.arange(py + 1) * grid.ny) // py
    wx, wy = rank % px, rank // px
    cx = np.arange(xs[wx], xs[wx + 1])
    cy = np.arange(ys[wy], ys[wy + 1])
    return np.sort((cy[:, None] * grid.nx + cx[None, :]).ravel())


def build_shard(grid, kernel, gen, seed, rank=0, size=1) -> ShardNet:
    """Incoming-synapse store of one shard.  Equivalent to the two-step
    construction exchange of network.py:189-295 because every source's draws
    are a pure function of (seed, gid) (connectivity.py:420-434)."""
    n = grid.neurons_per_column
    exc_n = int(math.floor(grid.excitatory_fraction * n))
    cols = owned_columns(grid, rank, size)
    col_rank = {int(c): i for i, c in enumerate(cols)}
    # sources that can reach an owned column: own-column plus reverse stencil
    offs, _ = stencil_active(kernel, grid)
    src_cols = set(int(c) for c in cols)
    for c in cols:
        ix, iy = int(c) % grid.nx, int(c) // grid.nx
        for di, dj in offs:
            sx, sy = ix - int(di), iy - int(dj)
            if 0 <= sx < grid.nx and 0 <= sy < grid.ny:
                src_cols.add(sy * grid.nx + sx)
    parts = []
    checksum = 0
    n_gen = 0
    own_set = set(int(c) for c in cols)
    for sc in sorted(src_cols):
        exc_layout = candidates(grid, kernel, sc, True)
        inh_layout = candidates(grid, kernel, sc, False)
        for gid in range(sc * n, sc * n + n):
            lay = exc_layout if (gid - sc * n) < exc_n else inh_layout
            tgt, d, w = draw_source(gid, lay[0], lay[1], grid, gen, seed)
            if sc in own_set:   # construction checksum is summed by the generating worker
                n_gen += len(tgt)
                flags = np.full(len(tgt), 1 if (gid - sc * n) < exc_n else 0, np.uint16)
                checksum = (checksum + wire_mix_sum(np.full(len(tgt), gid, np.uint32),
                                                    tgt, d, flags, w)) & MASK64
            tcol = tgt.astype(np.int64) // n
            keep = np.isin(tcol, cols)
            if not np.any(keep):
                continue
            parts.append((np.full(int(keep.sum()), gid, np.uint64), tgt[keep], d[keep], w[keep]))
    if parts:
        src = np.concatenate([p[0] for p in parts])
        tgt = np.concatenate([p[1] for p in parts]).astype(np.int64)
        dly = np.concatenate([p[2] for p in parts])
        wgt = np.concatenate([p[3] for p in parts])
    else:
        src = np.empty(0, U64); tgt = np.empty(0, np.int64)
        dly = np.empty(0, np.uint16); wgt = np.empty(0, np.float32)
    order = np.lexsort((dly, src))                       # network.py:257
    src, tgt, dly, wgt = src[order], tgt[order], dly[order], wgt[order]
    sources, starts = np.unique(src, return_index=True)
    offsets = np.concatenate([starts, [len(src)]]).astype(np.int64)
    lut = np.array([col_rank.get(c, -1) for c in range(grid.n_columns)], np.int64)
    tl = (lut[tgt // n] * n + tgt % n).astype(np.uint32)
    return ShardNet(sources.astype(U64), offsets, tl, dly.copy(), wgt.copy(), checksum, n_gen)


# ---------------------------------------------------------- neurons
class Neurons:
    """SoA neuron state of one shard (model.py:235-341)."""

    def __init__(self, exc_p, inh_p, is_exc):
        self.n = len(is_exc)
        def col(name):
            v = np.full(self.n, getattr(exc_p, name), dtype=np.float64)
            v[~is_exc] = getattr(inh_p, name)
            return v
        self.tau_m, self.tau_c, self.E = col("tau_m"), col("tau_c"), col("E")
        self.V_theta, self.V_r, self.tau_arp = col("V_theta"), col("V_r"), col("tau_arp")
        self.alpha_c = col("alpha_c")
        self.sfa = col("g_c") / col("C_m")
        self.V = self.E.copy()
        self.c = np.zeros(self.n)
        self.last = np.zeros(self.n)
        self.ru = np.full(self.n, -np.inf)

    @staticmethod
    def decay(V, c, dt, E, tau_m, tau_c, sfa):
        """model.py:116-143 closed form; expm1 branch for |x| <= 1."""
        em = np.exp(-dt / tau_m)
        ec = np.exp(-dt / tau_c)
        x = dt * (tau_c - tau_m) / (tau_m * tau_c)
        small = np.abs(x) <= 1.0
        xs = np.where(x == 0.0, 1.0, x)
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            f_small = np.where(x == 0.0, dt * em,
                               dt * em * np.expm1(np.where(small, x, 0.0)) / xs)
            f_large = dt * (ec - em) / xs
        f = np.where(small, f_small, f_large)
        return E + (V - E) * em - sfa * c * f, c * ec

    def peek(self, idx, t):
        """State advanced to t without committing (model.py:272-287)."""
        V, c, last, ru = self.V[idx], self.c[idx], self.last[idx], self.ru[idx]
        free_from = np.minimum(np.maximum(last, ru), t)
        c_s = c * np.exp(-(free_from - last) / self.tau_c[idx])
        V_s = np.where(last < ru, self.V_r[idx], V)
        V_t, c_t = self.decay(V_s, c_s, t - free_from, self.E[idx], self.tau_m[idx],
                              self.tau_c[idx], self.sfa[idx])
        return np.where(t < ru, self.V_r[idx], V_t), c_t

    def integrate(self, tgt, t_ev, w_ev):
        """Events sorted by (tgt, t, src, w); event rounds as model.py:289-337."""
        if len(tgt) == 0:
            return np.empty(0, np.int64), np.empty(0)
        counts = np.bincount(tgt, minlength=self.n)
        who = np.flatnonzero(counts)
        first = np.zeros(self.n, np.int64)
        first[who] = np.cumsum(counts[who]) - counts[who]
        k = counts[who]
        out_i, out_t = [], []
        for r in range(int(k.max())):
            idx = who[k > r]
            ev = first[idx] + r
            t = t_ev[ev]
            V, c = self.peek(idx, t)
            self.c[idx] = c
            self.last[idx] = t
            live = t >= self.ru[idx]
            V = np.where(live, V + w_ev[ev], self.V_r[idx])
            fire = live & (V > self.V_theta[idx])
            self.V[idx] = np.where(fire, self.V_r[idx], V)
            if fire.any():
                f = idx[fire]
                self.c[f] += self.alpha_c[f]
                self.ru[f] = t[fire] + self.tau_arp[f]
                out_i.append(f)
                out_t.append(t[fire])
        if out_i:
            return np.concatenate(out_i), np.concatenate(out_t)
        return np.empty(0, np.int64), np.empty(0)


def poisson_counts(seed, gids, t_step, lam):
    """engine.py:172-188: #{k : prod_{i<=k} u_i > exp(-lam)}, budget
    ceil(lam + 12 sqrt(lam)) + 20 draws."""
    if lam <= 0 or len(gids) == 0:
        return np.zeros(len(gids), dtype=np.int64)
    m = int(math.ceil(lam + 12.0 * math.sqrt(lam))) + POISSON_PAD
    u = counter_uniforms(seed, P_EXTERNAL, np.asarray(gids, U64)[:, None], t_step,
                         np.arange(m, dtype=U64)[None, :])
    cnt = np.sum(np.cumprod(u, axis=1) > math.exp(-lam), axis=1)
    if cnt.max(initial=0) >= m:
        raise AssertionError("Poisson draw budget exceeded")
    return cnt.astype(np.int64)


def external_events(seed, gids, t_step, ext, dt):
    """engine.py:191-206: (local index, time) of every external event."""
    lam = ext.synapses_per_neuron * ext.rate_per_synapse_hz * dt * 1e-3
    cnt = poisson_counts(seed, gids, t_step, lam)
    tot = int(cnt.sum())
    if tot == 0:
        return np.empty(0, np.int64), np.empty(0)
    which = np.repeat(np.arange(len(gids)), cnt)
    j = np.arange(tot) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    u = counter_uniforms(seed, P_EXTERNAL_TIME, np.asarray(gids, U64)[which], t_step, j)
    return which, (t_step + u) * dt


# ------------------------------------------------------------- loop
@dataclass
class OracleResult:
    raster_gids: np.ndarray
    raster_times: np.ndarray
    n_spikes: int
    recurrent_events: int
    external_events: int
    recurrent_synapses: int
    construction_checksum: int
    raster_checksum: int
    sim_seconds_wall: float
    probe_state: Optional[np.ndarray] = None   # [steps, P, 4] (V, c, last, ru) after each step
    probe_v_end: Optional[np.ndarray] = None   # [steps, P] V advanced to (t+1)*dt
    n_steps_run: int = 0


class ShardSim:
    """One shard's loop state; `step` runs engine.py:318-394 for one step given
    the AER events received for it (a list of (gids, times) arrays)."""

    def __init__(self, cfg, net: ShardNet, rank=0, size=1):
        grid = cfg.grid
        n = grid.neurons_per_column
        self.cfg, self.net = cfg, net
        cols = owned_columns(grid, rank, size)
        self.gids = (cols[:, None] * n + np.arange(n)[None, :]).ravel().astype(U64)
        exc_n = int(math.floor(grid.excitatory_fraction * n))
        self.neurons = Neurons(cfg.exc_params, cfg.inh_params,
                               (self.gids.astype(np.int64) % n) < exc_n)
        u0 = counter_uniforms(cfg.seed, P_INIT_STATE, self.gids, 0, 0)   # engine.py:301-302
        nb = self.neurons
        nb.V[:] = nb.V_r + u0 * (nb.V_theta - nb.V_r)
        D = cfg.genspec.d_max_steps
        self.ring: List[List[tuple]] = [[] for _ in range(D)]
        self.rec = 0
        self.ext = 0
        self.prev_idx = np.empty(0, np.int64)
        self.prev_t = np.empty(0)

    def outgoing(self):
        """Spikes of the previous step as (gids, times) sorted by (time, gid)."""
        g = self.gids[self.prev_idx]
        o = np.lexsort((g, self.prev_t))
        return g[o], self.prev_t[o]

    def step(self, t, incoming):
        cfg, net, dt = self.cfg, self.net, self.cfg.timestep_ms
        D = len(self.ring)
        for g, tm in incoming:                                 # engine.py:338-367
            if len(g) == 0 or len(net.sources) == 0:
                continue
            g = np.asarray(g, U64)
            pos = np.minimum(np.searchsorted(net.sources, g), len(net.sources) - 1)
            hit = net.sources[pos] == g
            rows, tm, g = pos[hit], np.asarray(tm)[hit], g[hit]
            a, b = net.offsets[rows], net.offsets[rows + 1]
            ln = b - a
            tot = int(ln.sum())
            if tot == 0:
                continue
            flat = np.arange(tot) - np.repeat(np.cumsum(ln) - ln, ln) + np.repeat(a, ln)
            d = net.delay[flat].astype(np.int64)
            arr = (t - 1) + d
            rec = (net.target_local[flat].astype(np.int64), net.weight[flat].astype(np.float64),
                   np.repeat(tm, ln) + d * dt, np.repeat(g, ln))
            for s in np.unique(arr):
                m = arr == s
                self.ring[int(s) % D].append((int(s),) + tuple(x[m] for x in rec))
            self.rec += tot
        chunks = self.ring[t % D]                               # engine.py:151-163
        self.ring[t % D] = []
        assert all(c[0] == t for c in chunks), "delay ring wrapped"
        if chunks:
            tgt = np.concatenate([c[1] for c in chunks])
            w = np.concatenate([c[2] for c in chunks])
            tm = np.concatenate([c[3] for c in chunks])
            src = np.concatenate([c[4] for c in chunks]).astype(U64)
        else:
            tgt, w, tm, src = (np.empty(0, np.int64), np.empty(0), np.empty(0),
                               np.empty(0, U64))
        which, ext_t = external_events(cfg.seed, self.gids, t, cfg.external, dt)
        if len(which):
            self.ext += len(which)
            tgt = np.concatenate([tgt, which])
            w = np.concatenate([w, np.full(len(which), cfg.external.weight_mv)])
            tm = np.concatenate([tm, ext_t])
            src = np.concatenate([src, np.full(len(which), U64(EXTERNAL_SOURCE_ID))])
        o = np.lexsort((w, src, tm, tgt))                     # engine.py:386
        self.prev_idx, self.prev_t = self.neurons.integrate(tgt[o], tm[o], w[o])
        return self.gids[self.prev_idx], self.prev_t


def run_oracle(cfg, steps=None, probes=None, net: Optional[ShardNet] = None) -> OracleResult:
    """Single-shard run (workers=1) of engine.run_worker (engine.py:286-411)."""
    if net is None:
        net = build_shard(cfg.grid, cfg.kernel, cfg.genspec, cfg.seed)
    n_steps = cfg.n_steps if steps is None else steps
    sim = ShardSim(cfg, net)
    probes = None if probes is None else np.asarray(probes, np.int64)
    ps = pv = None
    if probes is not None:
        ps = np.zeros((n_steps, len(probes), 4))
        pv = np.zeros((n_steps, len(probes)))
    rg, rt = [], []
    t0 = time.perf_counter()
    for t in range(n_steps):
        inc = [sim.outgoing()] if len(sim.prev_idx) else []
        g, tm = sim.step(t, inc)
        if len(g):
            rg.append(g); rt.append(tm.copy())
        if probes is not None:
            nb = sim.neurons
            ps[t, :, 0], ps[t, :, 1] = nb.V[probes], nb.c[probes]
            ps[t, :, 2], ps[t, :, 3] = nb.last[probes], nb.ru[probes]
            pv[t] = nb.peek(probes, np.full(len(probes), (t + 1) * cfg.timestep_ms))[0]
    wall = time.perf_counter() - t0
    g = np.concatenate(rg) if rg else np.empty(0, U64)
    tm = np.concatenate(rt) if rt else np.empty(0)
    o = np.lexsort((g, tm))
    g, tm = g[o], tm[o]
    return OracleResult(g, tm, len(g), sim.rec, sim.ext, len(net.target_local),
                        net.checksum, raster_checksum(g, tm), wall, ps, pv, n_steps)
