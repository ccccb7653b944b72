#!/bin/bash
python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r02l_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02l_tests.log
bash scripts/ab.sh c4 - SYMEL_NO_SOA_PF=1
bash scripts/ab.sh c5 - SYMEL_NO_SOA_PF=1
