#!/bin/bash
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -m gpu -x -q > gpurun_out/r02k_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02k_tests.log
bash scripts/ab.sh c3 - SYMEL_QUAD_SHFL=1 SYMEL_NO_QUAD_REDUCE=1
