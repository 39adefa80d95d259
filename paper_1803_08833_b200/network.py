"""Device-side incoming-synapse store of one shard: generation and import.

`build_b200` is the drop-in for the reference's network-build entry point
`construct_network` (corticarc/network.py:189-295).  Instead of generating
outgoing synapses and shipping 16 B wire records to their owners, every GPU
regenerates exactly its incoming synapses from the counter-based streams
(cc_gen_count / cc_gen_fill), so construction needs no collective.  The
resulting CSR is keyed by global source id (a dense int64 row index over all
neurons, 8 B/neuron) with 9 B per synapse in three SoA arrays:

    syn_tgt int32 (shard-local target)   syn_w float32   syn_d uint8

`import_csr` accepts the reference's own arrays (IncomingSynapses fields,
network.py:114-152) for runs on reference-generated connectivity.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .geometry import layout_blocks
from .partition import map_columns_to_workers

__all__ = ["DeviceNetwork", "build_b200", "import_csr", "export_csr", "halo_source_columns"]

MASK64 = (1 << 64) - 1


@dataclass
class DeviceNetwork:
    grid: object
    rank: int
    size: int
    owned_columns: np.ndarray
    src_gids: np.ndarray          # sources that may have rows here (ascending)
    row_off: "object"             # torch int64 [n_neurons + 1] on device
    syn_tgt: "object"             # torch int32 [S]
    syn_w: "object"               # torch float32 [S]
    syn_d: "object"               # torch uint8 [S]
    n_synapses: int
    checksum: int                 # wire-record checksum of the records stored here
    construction_seconds: float
    row_len_max: int
    dseg_cache: dict = field(default_factory=dict)    # delay-segment tables per (d_max, stride)

    @property
    def n_local(self) -> int:
        return len(self.owned_columns) * self.grid.neurons_per_column

    @property
    def steady_bytes(self) -> int:
        """9 B per synapse + the dense row index (paper's 12 B/syn study)."""
        return 9 * self.n_synapses + 8 * (self.grid.n_neurons + 1)

    @property
    def peak_bytes(self) -> int:
        return self.steady_bytes + 4 * len(self.src_gids) * 3

    def delay_segments(self, d_max: int, stride: int):
        """[n_rows, stride] int16 (u16 bits) table: synapses of each row with
        delay <= d, d = 0..d_max (rows are sorted by delay, network.py:257);
        the delivery kernel reads a spike's delay-d segment from it."""
        key = (d_max, stride)
        if key not in self.dseg_cache:
            import torch
            from . import _lib
            L = _lib.lib()
            n_rows = self.row_off.numel() - 1
            out = torch.zeros((max(1, n_rows), stride), dtype=torch.int16,
                              device=self.row_off.device)
            err = torch.zeros(1, dtype=torch.int32, device=self.row_off.device)
            stream = torch.cuda.current_stream(self.row_off.device).cuda_stream
            _lib.check(L.cc_build_dseg(self.row_off.data_ptr(), self.syn_d.data_ptr(), n_rows,
                                       d_max, stride, out.data_ptr(), err.data_ptr(), stream),
                       "cc_build_dseg")
            if int(err.item()):
                raise _lib.EngineError("cc_build_dseg: " + _lib.decode_errors(int(err.item())))
            self.dseg_cache[key] = out
        return self.dseg_cache[key]

    def nonempty_rows(self) -> int:
        ln = self.row_off[1:] - self.row_off[:-1]
        return int((ln > 0).sum().item())

    def host_csr(self):
        """(row_off, syn_tgt, syn_w, syn_d) as numpy (for oracles and tests)."""
        return (self.row_off.cpu().numpy(), self.syn_tgt.cpu().numpy(),
                self.syn_w.cpu().numpy(), self.syn_d.cpu().numpy())


def halo_source_columns(grid, kernel, owned_cols) -> np.ndarray:
    """Source columns whose candidate layout touches an owned column."""
    blk_col, _, blk_count = layout_blocks(grid, kernel)
    owned = np.zeros(grid.n_columns, bool)
    owned[owned_cols] = True
    keep = [c for c in range(grid.n_columns) if owned[blk_col[c, :blk_count[c]]].any()]
    return np.asarray(keep, dtype=np.int64)


def _gen_struct(cfg, col_local_t, tabs):
    g, gen = cfg.grid, cfg.genspec
    blk_col_t, blk_p_t, blk_count_t, kmax = tabs
    s = _lib.Gen()
    s.seed = cfg.seed & MASK64
    s.n_col = g.neurons_per_column
    s.n_exc_col = g.n_excitatory_per_column
    s.n_columns = g.n_columns
    s.kmax = kmax
    s.blk_col, s.blk_p = blk_col_t.data_ptr(), blk_p_t.data_ptr()
    s.blk_count, s.col_local = blk_count_t.data_ptr(), col_local_t.data_ptr()
    s.j_ee, s.j_ei, s.j_ie, s.j_ii = gen.j_exc_exc, gen.j_exc_inh, gen.j_inh_exc, gen.j_inh_inh
    s.sd_frac = gen.weight_sd_frac
    if gen.delay_kind == "uniform":
        s.delay_kind, s.d_lo, s.d_scale = 0, gen.delay_min_ms, gen.delay_max_ms - gen.delay_min_ms
    else:
        s.delay_kind, s.d_lo, s.d_scale = 1, 0.0, gen.delay_mean_ms
    s.dt = gen.timestep_ms
    s.d_max = gen.d_max_steps
    return s


def build_b200(cfg, rank: int = 0, size: int = 1, device=None) -> DeviceNetwork:
    """Generate this shard's incoming CSR on the GPU (bit-exact with
    connectivity.py:383-417 for targets, weights and delays)."""
    import torch
    L = _lib.lib()
    if cfg.genspec.d_max_steps > 255:
        raise ValueError("d_max_steps > 255 does not fit the uint8 delay table")
    if cfg.grid.n_neurons >= 2 ** 31:
        raise ValueError("grid too large for int32 target ids")
    dev = torch.device(device or f"cuda:{torch.cuda.current_device()}")
    t0 = time.perf_counter()
    grid = cfg.grid
    pmap = map_columns_to_workers(grid, size)
    owned = pmap.owned_columns(rank)
    blk_col, blk_p, blk_count = layout_blocks(grid, cfg.kernel)
    kmax = blk_col.shape[1]
    col_local = np.full(grid.n_columns, -1, np.int32)
    col_local[owned] = np.arange(len(owned), dtype=np.int32)
    owned_mask = col_local >= 0
    halo = [c for c in range(grid.n_columns) if owned_mask[blk_col[c, :blk_count[c]]].any()]
    n = grid.neurons_per_column
    src = (np.asarray(halo, np.int64)[:, None] * n + np.arange(n)[None, :]).ravel()
    src_t = torch.from_numpy(src.astype(np.uint32).view(np.int32)).to(dev)
    tabs = (torch.from_numpy(np.ascontiguousarray(blk_col)).to(dev),
            torch.from_numpy(np.ascontiguousarray(blk_p)).to(dev),
            torch.from_numpy(blk_count).to(dev), kmax)
    col_local_t = torch.from_numpy(col_local).to(dev)
    gs = _gen_struct(cfg, col_local_t, tabs)
    stream = torch.cuda.current_stream(dev).cuda_stream
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    row_len = torch.zeros(len(src), dtype=torch.int64, device=dev)
    _lib.check(L.cc_gen_count(C.byref(gs), src_t.data_ptr(), len(src), row_len.data_ptr(),
                              err.data_ptr(), stream), "cc_gen_count")
    counts = torch.zeros(grid.n_neurons, dtype=torch.int64, device=dev)
    counts[torch.from_numpy(src).to(dev)] = row_len
    row_off = torch.zeros(grid.n_neurons + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=row_off[1:])
    S = int(row_off[-1].item())
    max_row = int(row_len.max().item()) if len(src) else 0
    src_dev = torch.from_numpy(src).to(dev)
    row_start = torch.cat([row_off[src_dev], row_off[-1:]]) if len(src) else row_off[:1]
    syn_tgt = torch.empty(S, dtype=torch.int32, device=dev)
    syn_w = torch.empty(S, dtype=torch.float32, device=dev)
    syn_d = torch.empty(S, dtype=torch.uint8, device=dev)
    csum = torch.zeros(1, dtype=torch.int64, device=dev)
    if S:
        per_warp = 3 * max_row + 3
        scratch = torch.empty(int(L.cc_gen_warps()) * per_warp, dtype=torch.float32, device=dev)
        _lib.check(L.cc_gen_fill(C.byref(gs), src_t.data_ptr(), len(src), row_start.data_ptr(),
                                 syn_tgt.data_ptr(), syn_w.data_ptr(), syn_d.data_ptr(),
                                 csum.data_ptr(), scratch.data_ptr(), per_warp, err.data_ptr(),
                                 stream), "cc_gen_fill")
        del scratch
    torch.cuda.synchronize(dev)
    if int(err.item()):
        raise _lib.EngineError("generator: " + _lib.decode_errors(int(err.item())))
    return DeviceNetwork(grid=grid, rank=rank, size=size, owned_columns=owned, src_gids=src,
                         row_off=row_off, syn_tgt=syn_tgt, syn_w=syn_w, syn_d=syn_d,
                         n_synapses=S, checksum=int(csum.item()) & MASK64,
                         construction_seconds=time.perf_counter() - t0, row_len_max=max_row)


def import_csr(cfg, sources, offsets, target_local, delay, weight, rank: int = 0,
               size: int = 1, device=None) -> DeviceNetwork:
    """Upload a reference-format incoming store (IncomingSynapses fields,
    network.py:114-152: rows by source gid, local target index)."""
    import torch
    L = _lib.lib()
    dev = torch.device(device or f"cuda:{torch.cuda.current_device()}")
    t0 = time.perf_counter()
    grid = cfg.grid
    pmap = map_columns_to_workers(grid, size)
    owned = pmap.owned_columns(rank)
    sources = np.asarray(sources, np.int64)
    offsets = np.asarray(offsets, np.int64)
    counts = np.zeros(grid.n_neurons, np.int64)
    counts[sources] = np.diff(offsets)
    row_off_h = np.zeros(grid.n_neurons + 1, np.int64)
    np.cumsum(counts, out=row_off_h[1:])
    # rows must be contiguous in source order: the reference's are (sorted sources)
    if len(sources) and not np.all(np.diff(sources) > 0):
        raise ValueError("sources must be strictly ascending")
    S = int(offsets[-1]) if len(offsets) else 0
    row_off = torch.from_numpy(row_off_h).to(dev)

    def up(a, narrow):
        """Host array -> device in its own width (no widened host copy); the
        reference store holds u32 targets, u16 delays, f32 weights."""
        a = np.ascontiguousarray(a)
        if a.dtype.kind == "u" and a.dtype.itemsize in (2, 4):     # torch has no u16 / u32
            a = a.view(np.int16 if a.dtype.itemsize == 2 else np.int32)
        t = torch.from_numpy(a).to(dev)
        return t if t.dtype == narrow else t.to(narrow)

    if len(delay) and int(np.max(delay)) > cfg.genspec.d_max_steps:
        raise ValueError("imported delay exceeds d_max")
    if len(target_local) and int(np.max(target_local)) >= len(owned) * grid.neurons_per_column:
        raise ValueError("imported target index outside the shard")
    syn_tgt = up(target_local, torch.int32)
    syn_w = up(weight, torch.float32)
    syn_d = up(delay, torch.uint8)
    n = grid.neurons_per_column
    # global target gid of every synapse (construction checksum), on the device
    # in pieces of 64 M synapses
    owned_t = torch.from_numpy(np.asarray(owned, np.int64)).to(dev)
    tgt_global = torch.empty(S, dtype=torch.int32, device=dev)
    for a0 in range(0, S, 1 << 26):
        tl = syn_tgt[a0:a0 + (1 << 26)].to(torch.int64)
        tgt_global[a0:a0 + (1 << 26)] = (owned_t[tl // n] * n + tl % n).to(torch.int32)
    del owned_t
    src_t = torch.from_numpy(sources.astype(np.uint32).view(np.int32)).to(dev)
    csum = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(L.cc_csr_checksum(row_off.data_ptr(), src_t.data_ptr(), len(sources),
                                 tgt_global.data_ptr(), syn_w.data_ptr(), syn_d.data_ptr(),
                                 n, grid.n_excitatory_per_column, csum.data_ptr(), stream),
               "cc_csr_checksum")
    torch.cuda.synchronize(dev)
    return DeviceNetwork(grid=grid, rank=rank, size=size, owned_columns=owned,
                         src_gids=sources, row_off=row_off, syn_tgt=syn_tgt, syn_w=syn_w,
                         syn_d=syn_d, n_synapses=S, checksum=int(csum.item()) & MASK64,
                         construction_seconds=time.perf_counter() - t0,
                         row_len_max=int(np.diff(offsets).max()) if len(sources) else 0)


def export_csr(net: DeviceNetwork) -> dict:
    """The shard's store in the reference's IncomingSynapses layout
    (network.py:114-152): rows of the sources that have synapses here, in
    ascending gid order, each sorted by delay (network.py:257).  Returns numpy
    arrays sources u64, offsets i64, target_local u32, delay u16, weight f32 -
    what import_csr takes back (round trip), plus the construction checksum."""
    row_off, tgt, w, d = net.host_csr()
    ln = np.diff(row_off)
    src = np.flatnonzero(ln).astype(np.int64)
    offsets = np.concatenate([[0], np.cumsum(ln[src])]).astype(np.int64)
    return dict(sources=src.astype(np.uint64), offsets=offsets,
                target_local=tgt.astype(np.uint32), delay=d.astype(np.uint16),
                weight=w.astype(np.float32), checksum=net.checksum)
