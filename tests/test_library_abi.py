"""The C-ABI library loads on a CPU host and exports every symbol the header
declares, with struct layouts matching the ctypes mirrors (no compute calls)."""

import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "corticarc_b200.h")


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(cc_\w+)\s*\(",
                                 txt, flags=re.M)))


def test_library_exports_header_symbols():
    from paper_1803_08833_b200 import _lib
    L = _lib.load_library()
    names = declared_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_abi_and_layout():
    import ctypes as C
    from paper_1803_08833_b200 import _lib
    L = _lib.load_library()
    assert L.cc_abi_version() == _lib.ABI_VERSION
    assert L.cc_sizeof_shard() == C.sizeof(_lib.Shard)
    assert L.cc_sizeof_ctl() == C.sizeof(_lib.Ctl)
    assert L.cc_sizeof_gen() == C.sizeof(_lib.Gen)
    assert L.cc_sizeof_xpeer() == C.sizeof(_lib.XPeer) == 40


def test_product_path_refuses_cpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_1803_08833_b200 import _lib
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.lib()
    from paper_1803_08833_b200.engine import run_b200
    from conftest import tiny_config
    with pytest.raises(RuntimeError):
        run_b200(tiny_config(), 1)


def test_library_is_sm100a():
    import subprocess
    from paper_1803_08833_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_capacity_retry_policy():
    """Only overflows of the expectation-sized buffers trigger a re-run, each
    doubling the buffer that overflowed, up to a limit; EngineError keeps its
    bits across processes (pickling)."""
    import pickle
    from paper_1803_08833_b200 import _lib
    cap = dict(ovf=1, scratch=1, evrec=1)
    e = _lib.EngineError("step 3: event staging scratch exhausted", 0x08)
    assert _lib.capacity_error(e)
    assert _lib.grow_capacity(e, cap) == dict(ovf=1, scratch=2, evrec=1)
    both = _lib.EngineError("x", 0x08 | 0x100)
    assert _lib.grow_capacity(both, cap) == dict(ovf=1, scratch=2, evrec=2)
    assert _lib.grow_capacity(e, dict(cap, scratch=32)) is None          # at the limit
    for bits in (0x01, 0x20, 0x08 | 0x20, 0x400, 0x1000, 0):
        assert _lib.grow_capacity(_lib.EngineError("x", bits), cap) is None
    back = pickle.loads(pickle.dumps(e))
    assert isinstance(back, _lib.EngineError) and back.bits == 0x08 and str(back) == str(e)
