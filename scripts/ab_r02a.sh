#!/bin/bash
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -m gpu -x -q > gpurun_out/r02i_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02i_tests.log
bash scripts/ab.sh c4 - SYMEL_FIXUP_U1=1
bash scripts/ab.sh c2 - SYMEL_FIXUP_U1=1
bash scripts/ab.sh c5 - SYMEL_FIXUP_U1=1
