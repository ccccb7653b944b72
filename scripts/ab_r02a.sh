#!/bin/bash
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/r02h_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02h_tests.log
bash scripts/ab.sh c4 - SYMEL_MORTON_PER_AXIS=1
bash scripts/ab.sh c5 - SYMEL_MORTON_PER_AXIS=1
for c in c2 c3; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$c', '%.3f ms kernel %.3f frac %.3f' % (d['ms_per_step'], r['kernel_ms'], r['frac']), d['details']['tile_plan'])"; done
python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['details']['tile_plan'])"
