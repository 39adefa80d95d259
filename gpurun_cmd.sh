set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for a in "" "--no-split"; do python bench.py --no-cpu --no-e2e --steps 1000 --warmup 200 $a > gpurun_out/split$a.json 2>gpurun_out/split$a.err; python -c "import json;d=json.load(open('gpurun_out/split$a.json'));print('$a',d['ms_per_step'],d['value'],json.dumps(d['kernels']))"; done
for v in b2 b4; do CC_LIB_PATH=build_variants/lib_$v.so python bench.py --no-cpu --no-e2e --steps 1000 --warmup 200 > gpurun_out/split_$v.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/split_$v.json'));print('$v',d['ms_per_step'],d['value'],json.dumps(d['kernels']))"; done
