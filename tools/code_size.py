"""Code size (bytes of SASS) of the simulation kernels and their out-of-line
device functions in a built library:

    python tools/code_size.py paper_1803_08833_b200/libcorticarc_b200.so

k_stage is instruction-cache sensitive: its hot loops
should stay small; cold paths are kept out of line."""
import os
import re
import subprocess
import sys
import tempfile

lib = os.path.abspath(sys.argv[1])
with tempfile.TemporaryDirectory() as tmp:
    subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, check=True, capture_output=True)
    for c in sorted(os.listdir(tmp)):
        if "sim_kernels" not in c or c.count("-"):
            continue
        out = subprocess.run(["nvdisasm", "-c", os.path.join(tmp, c)], capture_output=True,
                             text=True).stdout
        sizes, cur = {}, None
        for line in out.splitlines():
            m = re.match(r"\s*\.(?:global|weak)?\s*", line)
            if line.startswith("\t.type") or line.startswith(".type"):
                continue
            m = re.match(r"^([\w$.]+):\s*$", line)
            if m and not m.group(1).startswith(".L"):
                cur = m.group(1)
                sizes.setdefault(cur, 0)
            elif cur and re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
                sizes[cur] += 16
        for name, sz in sorted(sizes.items(), key=lambda kv: -kv[1])[:16]:
            short = re.sub(r"_ZN\d+_GLOBAL__N__[0-9a-f_]+sim_kernels_cu_[0-9a-f]+", "", name)
            print(f"{sz:8d}  {short}")
