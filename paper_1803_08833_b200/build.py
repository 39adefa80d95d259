"""In-tree build of libcorticarc_b200.so for sm_100a (nvcc, no torch JIT).

    python -m paper_1803_08833_b200.build          # or __graft_entry__.build()

The shared library is written next to this file so it travels with the repo
snapshot to the GPU host; `-fmad=false` keeps every float64 expression in the
reference's evaluation order (no contracted multiply-adds).
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
GEN = os.path.join(CSRC, "_gen")
LIB = os.path.join(PKG, "libcorticarc_b200.so")
SOURCES = ["capi.cu", "dispatch.cu", "sim_kernels.cu", "gen_kernels.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false",
         "-gencode", "arch=compute_100a,code=sm_100a",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "--extended-lambda"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)
            if f.endswith((".cu", ".cuh", ".py"))]
    deps.append(os.path.join(ROOT, "include", "corticarc_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def _defined(defines, key, default):
    for d in defines:
        if d.split("=")[0] == key:
            return d.split("=", 1)[1]
    return default


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile the library; `out`/`defines` build tuning variants (tools/).

    sim_kernels.cu is compiled once per sub-list variant (CC_NSUB_A and
    CC_NSUB_B sub-lists per group, include/corticarc_b200.h; a `CC_SUBLISTS=n`
    define builds that single variant instead), the objects in parallel."""
    target = out or LIB
    os.makedirs(os.path.dirname(os.path.abspath(target)), exist_ok=True)
    if out is None and not force and not _stale():
        return LIB
    sys.path.insert(0, CSRC)
    try:
        import gen_ziggurat
    finally:
        sys.path.pop(0)
    gen_ziggurat.emit(os.path.join(GEN, "cc_ziggurat_tables.h"))
    defines = tuple(defines)
    single = _defined(defines, "CC_SUBLISTS", None)
    if single is not None:          # one variant: both slots name it
        defines = tuple(d for d in defines if d.split("=")[0] != "CC_SUBLISTS")
        defines += (f"CC_NSUB_A={single}", f"CC_NSUB_B={single}")
    nsub = sorted({_defined(defines, "CC_NSUB_A", "1"), _defined(defines, "CC_NSUB_B", "8")})
    objdir = os.path.join(GEN, "obj_" + os.path.basename(target).replace(".", "_"))
    os.makedirs(objdir, exist_ok=True)
    common = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"),
              "-I", CSRC, "-I", GEN]
    jobs = [(os.path.join(objdir, name.replace(".cu", ".o")), [os.path.join(CSRC, name)], [])
            for name in SOURCES if name != "sim_kernels.cu"]
    jobs += [(os.path.join(objdir, f"sim_kernels_s{n}.o"), [os.path.join(CSRC, "sim_kernels.cu")],
              [f"-DCC_SUBLISTS={n}"]) for n in nsub]
    procs = [(obj, subprocess.Popen([*common, *extra, "-c", *src, "-o", obj],
                                    stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
             for obj, src, extra in jobs]
    log, failed = [], None
    for obj, pr in procs:
        so, se = pr.communicate()
        log.append(f"==== {os.path.basename(obj)}\n{so}{se}")
        if pr.returncode != 0 and failed is None:
            failed = se
    with open(os.path.join(GEN, "ptxas.log"), "w") as fh:
        fh.write("\n".join(log))
    if failed is not None:
        raise RuntimeError("nvcc failed:\n" + failed[-6000:])
    res = subprocess.run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
                          *[obj for obj, _, _ in jobs], "-o", target + ".tmp"],
                         capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("link failed:\n" + res.stderr[-6000:])
    os.replace(target + ".tmp", target)
    if verbose:
        print("\n".join(log))
    return target


# A 4-input staging window: most neuron-steps overflow the shared-memory
# window and take the global-scratch path (tests/test_gpu_parity.py).
SPILL_VARIANT = os.path.join(PKG, "libcorticarc_b200_w4.so")


# Bounds and protocol assertions compiled in (CC_CHK in cc_common.cuh): the
# parity tests run small cases through it in place of compute-sanitizer.
CHECKED_VARIANT = os.path.join(PKG, "libcorticarc_b200_chk.so")


def build_test_variants(force: bool = False) -> None:
    for path, defines in ((SPILL_VARIANT, ("CC_NEURON_WCAP=4", "CC_UPD_PIPE=0")),
                          (CHECKED_VARIANT, ("CC_CHECKS=1", "CC_RT_PER_THREAD=1", "CC_BN_PER_THREAD=1",
                                             "CC_RT_BLOCKS=3"))):
        if force or not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(LIB):
            build(force=True, out=path, defines=defines)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    if "--variants" in sys.argv:
        build_test_variants(force=True)
