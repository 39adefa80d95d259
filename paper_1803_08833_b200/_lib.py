"""ctypes binding of libcorticarc_b200.so (the C ABI in include/corticarc_b200.h).

The product path has no fallback: if the library is missing or CUDA is not
available, `lib()` raises.  Struct mirrors are checked against the sizes the
library was compiled with.
"""

from __future__ import annotations

import ctypes as C
import os

__all__ = ["lib", "Pop", "Ctl", "Shard", "Gen", "XPeer", "check", "EngineError", "ERR_BITS",
           "LIB_PATH"]

LIB_PATH = os.environ.get("CC_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libcorticarc_b200.so")
ABI_VERSION = 29
ITEM_CLASSES = 8
L1_MAX_REGIONS, L1_MAX_LISTS, L1_STRIDE, L1_NCNT_MAX_RB = 2048, 1024, 32, 12   # CC_L1_* (include/corticarc_b200.h)
FLAG_NO_TAIL_DELIVERY = 0x1000   # CC_FLAG_NO_TAIL_DELIVERY (include/corticarc_b200.h)

ERR_BITS = {
    0x01: "spike log full (more spikes in one step than planned)",
    0x02: "CSR row longer than 65535 synapses (delay-segment table)",
    0x04: "input-list overflow list full",
    0x08: "event staging scratch exhausted",
    0x10: "Poisson draw budget exceeded (engine.py:187)",
    0x20: "raster buffer full",
    0x40: "exchange out-list full",
    0x80: "generator row larger than planned",
    0x100: "ordered-input record buffer full (inputs of one step)",
    0x200: "k_stage grid barrier timed out (blocks not co-resident)",
    0x400: "peer exchange: a source rank's spikes of the step did not arrive in time",
    0x800: "peer exchange: destination region full",
    0x1000: "checked build: bounds / protocol assertion failed (error step = source line)",
}


class EngineError(RuntimeError):
    """A device-side capacity or protocol violation, naming the step; .bits
    holds the cc_ctl.error_bits when it came from the device."""

    def __init__(self, msg: str = "", bits: int = 0):
        super().__init__(msg)
        self.bits = int(bits)

    def __reduce__(self):                     # picklable across worker processes
        return (EngineError, (str(self), self.bits))


class Pop(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("tau_m", "tau_c", "E", "V_theta", "V_r", "tau_arp", "alpha_c", "sfa", "k1", "k2",
                 "r_tau_m", "r_tau_c", "r_k2")]


class Ctl(C.Structure):
    _fields_ = [
        ("t", C.c_longlong), ("rec_events", C.c_ulonglong), ("ext_events", C.c_ulonglong),
        ("n_spikes", C.c_ulonglong), ("raster_n", C.c_ulonglong),
        ("pad2", C.c_uint), ("error_bits", C.c_uint), ("error_step", C.c_longlong),
        ("max_bin", C.c_uint), ("max_events", C.c_uint), ("scratch_used", C.c_ulonglong),
        ("out_n", C.c_uint), ("pad0", C.c_uint), ("spilled_total", C.c_ulonglong),
        ("ovf_total", C.c_ulonglong), ("done_deliver", C.c_uint), ("ovf_grouped", C.c_uint),
        ("stream_used", C.c_ulonglong), ("done_stage", C.c_uint), ("n_rounds", C.c_uint),
        ("round_next", C.c_uint), ("pad1", C.c_uint), ("cls_n", C.c_uint * 8),
        ("del_events", C.c_ulonglong), ("tail_events", C.c_ulonglong),
        ("x_sent", C.c_ulonglong), ("x_recv", C.c_ulonglong),
    ]


class XPeer(C.Structure):
    """cc_xpeer: one source/destination region of the peer exchange."""
    _fields_ = [("rec", C.c_uint64 * 2), ("flag", C.c_uint64 * 2), ("cap", C.c_uint32),
                ("pad", C.c_uint32)]


_P = C.c_void_p


class Shard(C.Structure):
    _fields_ = [
        ("n_local", C.c_int32), ("n_col", C.c_int32), ("n_exc_col", C.c_int32),
        ("d_max", C.c_int32), ("bin_cap", C.c_int32), ("log_slots", C.c_int32),
        ("spk_cap", C.c_int32), ("seg_stride", C.c_int32),
        ("ovf_cap", C.c_int64), ("pad64_", C.c_int64), ("raster_cap", C.c_int64),
        ("scratch_cap", C.c_int64), ("n_rows", C.c_int64),
        ("out_cap", C.c_int32), ("ext_budget", C.c_int32), ("n_probe", C.c_int32),
        ("direct_log", C.c_int32), ("flags", C.c_int32), ("plan_in_stage", C.c_int32),
        ("del_lps_log2", C.c_int32), ("n_sub", C.c_int32),
        ("h2_ext", C.c_uint64), ("h2_time", C.c_uint64), ("h2_init", C.c_uint64),
        ("dt", C.c_double), ("ext_weight", C.c_double), ("ext_thresh", C.c_double),
        ("pop", Pop * 2),
        ("gid", _P), ("state", _P),
        ("row_off", _P), ("syn_tgt", _P), ("syn_w", _P), ("syn_d", _P),
        ("n_groups", C.c_int32), ("bin_pad", C.c_int32),
        ("bin_cnt", _P), ("bin_rec", _P), ("grp_n", _P), ("grp_sub", _P), ("ovf_rec", _P), ("ovf_cnt", _P),
        ("ovf_sorted", _P), ("ovf_off", _P), ("ovf_fill", _P),
        ("log_t", _P), ("log_gid", _P), ("log_ctr", _P), ("log_len", _P),
        ("log_r0", _P), ("log_dseg", _P), ("dseg", _P),
        ("raster_gid", _P), ("raster_t", _P), ("out_gid", _P), ("out_t", _P),
        ("scratch", _P), ("ev_n", _P), ("ev_nr", _P),
        ("evrec", _P), ("evrec_cap", C.c_int64), ("ev_off", _P), ("grp_items", _P),
        ("grp_done", _P), ("rounds", _P), ("round_cap", C.c_int64),
        ("probe_map", _P), ("probe_out", _P),
        ("probe_steps", C.c_int64), ("ctl", _P), ("tailc", _P), ("remote", _P),
        ("n_ranks", C.c_int32), ("rank", C.c_int32), ("xmask", _P), ("xdst", _P), ("xsrc", _P),
        ("xcnt", _P), ("xwait_ns", C.c_int64),
        ("l1_rb", C.c_int32), ("n_regions", C.c_int32), ("l1_cap", C.c_int64),
        ("l1_cnt", _P), ("l1_ref", _P), ("l1_w", _P), ("l1_tgt", _P), ("l1_ncnt", _P),
    ]


class Gen(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64), ("n_col", C.c_int32), ("n_exc_col", C.c_int32),
        ("n_columns", C.c_int32), ("kmax", C.c_int32),
        ("blk_col", _P), ("blk_p", _P), ("blk_count", _P), ("col_local", _P),
        ("j_ee", C.c_double), ("j_ei", C.c_double), ("j_ie", C.c_double), ("j_ii", C.c_double),
        ("sd_frac", C.c_double), ("delay_kind", C.c_int32),
        ("d_lo", C.c_double), ("d_scale", C.c_double), ("dt", C.c_double),
        ("d_max", C.c_int32),
    ]


_lib = None

_SIGS = {
    "cc_abi_version": (C.c_int, []),
    "cc_last_error": (C.c_char_p, []),
    "cc_sizeof_shard": (C.c_int64, []),
    "cc_sizeof_ctl": (C.c_int64, []),
    "cc_sizeof_gen": (C.c_int64, []),
    "cc_sizeof_xpeer": (C.c_int64, []),
    "cc_timer_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    "cc_timer_record": (C.c_int, [C.c_void_p, C.c_int32, _P]),
    "cc_timer_elapsed_ms": (C.c_float, [C.c_void_p, C.c_int32, C.c_int32]),
    "cc_timer_destroy": (C.c_int, [C.c_void_p]),
    "cc_init_state": (C.c_int, [C.POINTER(Shard), _P]),
    "cc_deliver": (C.c_int, [C.POINTER(Shard), _P]),
    "cc_prepare": (C.c_int, []),
    "cc_neuron_step": (C.c_int, [C.POINTER(Shard), _P]),
    "cc_ingest": (C.c_int, [C.POINTER(Shard), _P, _P, _P, _P]),
    "cc_pack_aer": (C.c_int, [C.POINTER(Shard), _P, C.c_int32, C.c_int32, _P, _P, _P]),
    "cc_ingest_aer": (C.c_int, [C.POINTER(Shard), _P, C.c_int32, C.c_int32, _P]),
    "cc_gen_count": (C.c_int, [C.POINTER(Gen), _P, C.c_int64, _P, _P, _P]),
    "cc_gen_fill": (C.c_int, [C.POINTER(Gen), _P, C.c_int64, _P, _P, _P, _P, _P, _P,
                              C.c_int64, _P, _P]),
    "cc_gen_warps": (C.c_int64, []),
    "cc_build_dseg": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.c_int32, _P, _P, _P]),
    "cc_exchange_ingest": (C.c_int, [C.POINTER(Shard), _P]),
    "cc_xwin_alloc": (C.c_int, [C.c_int64, C.POINTER(C.c_void_p), C.c_char_p]),
    "cc_xwin_open": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "cc_xwin_close": (C.c_int, [_P]),
    "cc_xwin_free": (C.c_int, [_P]),
    "cc_cnt_stride": (C.c_int32, [C.c_int32]),
    "cc_kernels_per_step": (C.c_int32, [_P]),
    "cc_stage_warps": (C.c_int32, [_P]),
    "cc_csr_checksum": (C.c_int, [_P, _P, C.c_int64, _P, _P, _P, C.c_int32, C.c_int32, _P, _P]),
    "cc_test_philox": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, C.c_int32,
                                 _P, _P]),
    "cc_test_math": (C.c_int, [C.c_int32, _P, _P, C.c_int64, _P]),
    "cc_test_counter_uniforms": (C.c_int, [C.c_uint64, C.c_uint64, _P, C.c_uint64, _P,
                                           C.c_int64, _P, _P]),
}


def load_library(path: str = LIB_PATH):
    """Load and type the library without touching CUDA (CPU-safe)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with "
                          "`python -m paper_1803_08833_b200.build` (there is no CPU fallback)")
    L = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    if L.cc_abi_version() != ABI_VERSION:
        raise ImportError(f"ABI mismatch: library {L.cc_abi_version()} != {ABI_VERSION}")
    for name, st in (("cc_sizeof_shard", Shard), ("cc_sizeof_ctl", Ctl), ("cc_sizeof_gen", Gen),
                     ("cc_sizeof_xpeer", XPeer)):
        if getattr(L, name)() != C.sizeof(st):
            raise ImportError(f"struct layout mismatch for {name}: "
                              f"{getattr(L, name)()} != {C.sizeof(st)}")
    _lib = L
    return L


def cnt_stride(n_sub: int) -> int:
    """u32 words between the fill counters of consecutive input lists for a
    shard with n_sub sub-lists per group; raises if the library does not carry
    that variant (include/corticarc_b200.h: CC_NSUB_A, CC_NSUB_B)."""
    st = int(load_library().cc_cnt_stride(int(n_sub)))
    if st <= 0:
        raise ValueError(f"the library has no step kernels for {n_sub} sub-lists per group")
    return st



def lib():
    """The library, for device work: fails loudly without a CUDA device."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1803_08833_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    return load_library()


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = _lib.cc_last_error().decode() if _lib is not None else "?"
        raise EngineError(f"{what}: {msg}" if what else msg)


# buffers sized by expectation (run_b200 re-runs with more capacity): overflow
# list, spill staging, ordered-input records
CAPACITY_BITS = 0x04 | 0x08 | 0x100


def capacity_error(err: "EngineError") -> bool:
    """True when an EngineError is only a capacity overflow of the
    expectation-sized buffers (no other error bit set)."""
    bits = getattr(err, "bits", 0)
    return bool(bits) and not (bits & ~CAPACITY_BITS)


_GROW = {0x04: "ovf", 0x08: "scratch", 0x100: "evrec"}


def grow_capacity(err: "EngineError", capacity: dict, limit: int = 32):
    """The capacity multipliers for a re-run after `err`: the overflowed
    buffers doubled, or None if err is not (only) such an overflow or a
    buffer is already at `limit`."""
    if not capacity_error(err):
        return None
    out = dict(capacity)
    for bit, key in _GROW.items():
        if err.bits & bit:
            if out.get(key, 1) >= limit:
                return None
            out[key] = out.get(key, 1) * 2
    return out


def decode_errors(bits: int) -> str:
    return "; ".join(v for k, v in ERR_BITS.items() if bits & k) or f"0x{bits:x}"
