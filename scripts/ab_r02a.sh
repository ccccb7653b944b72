#!/bin/bash
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -m gpu -x -q > gpurun_out/r02d_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02d_tests.log
BENCH_FLAGS=--no-spd bash scripts/ab.sh c2 - SYMEL_NO_L2PF=1 SYMEL_NO_BULK_PLAN=1 "SYMEL_NO_L2PF=1 SYMEL_NO_BULK_PLAN=1"
bash scripts/ab.sh c2 - "SYMEL_NO_L2PF=1 SYMEL_NO_BULK_PLAN=1"
bash scripts/ab.sh c4 - "SYMEL_NO_L2PF=1 SYMEL_NO_BULK_PLAN=1"
bash scripts/ab.sh c5 - "SYMEL_NO_L2PF=1 SYMEL_NO_BULK_PLAN=1"
