#!/bin/bash
python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r02n_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02n_tests.log
SYMEL_EARLY_SEGMD=1 python -m pytest tests/test_gpu_parity.py -m gpu -x -q >> gpurun_out/r02n_tests.log 2>&1; echo "tests early rc=$?" >> gpurun_out/r02n_tests.log
BENCH_FLAGS=--no-spd bash scripts/ab.sh c2 - SYMEL_EARLY_SEGMD=1
bash scripts/ab.sh c2 - SYMEL_EARLY_SEGMD=1
bash scripts/ab.sh c4 - SYMEL_EARLY_SEGMD=1
bash scripts/ab.sh c3 - SYMEL_EARLY_SEGMD=1
bash scripts/ab.sh c5 - SYMEL_EARLY_SEGMD=1
