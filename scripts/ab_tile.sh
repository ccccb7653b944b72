#!/bin/bash
# tile-size sweep: parity of the small cases, then timing of every config per SYMEL_TILE_THREADS
for T in 64 96; do
  SYMEL_TILE_THREADS=$T python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -x -q -m gpu 2>&1 | tail -2
done
for cfg in c2 c4 c5 c3; do
  bash scripts/ab.sh $cfg "SYMEL_TILE_THREADS=64" "SYMEL_TILE_THREADS=96" "-"
done
BENCH_FLAGS=--no-spd bash scripts/ab.sh c2 "SYMEL_TILE_THREADS=64" "SYMEL_TILE_THREADS=96" "-"
