"""Build k_stage tuning variants into build_variants/ (here, no GPU needed) and
print the gpurun command that benches each one (CC_LIB_PATH selects the .so).

    python tools/sweep_variants.py w192:CC_NEURON_WCAP=192 b16:CC_NBUCKET=16 ...
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1803_08833_b200.build import build  # noqa: E402


def main(specs):
    names = []
    for spec in specs:
        name, _, defs = spec.partition(":")
        build(force=True, out=os.path.join(ROOT, "build_variants", f"lib_{name}.so"),
              defines=tuple(d for d in defs.split(",") if d))
        names.append(name)
    loop = " ".join(names)
    print(f"for v in {loop}; do CC_LIB_PATH=build_variants/lib_$v.so python bench.py --no-cpu "
          f"--no-e2e --steps 1000 --warmup 200 > gpurun_out/var_$v.json; done")


if __name__ == "__main__":
    main(sys.argv[1:])
