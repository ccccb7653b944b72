#!/bin/bash
# ncu evidence for profiles/: (1) launch list of two bench steps (cold-cache, serialised),
# (2) one --set full capture of the headline tile kernel. Each ncu run follows an identical
# plain run that exited 0.
set -e
python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof_bench_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
python scripts/profile_step.py --config c2 --steps 3 --spd > gpurun_out/prof_plain2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sy_7 -s 1 -c 1 -o gpurun_out/prof_r01_c2_spd_tile \
    python scripts/profile_step.py --config c2 --steps 3 --spd > gpurun_out/ncu_full.log 2>&1
echo done
