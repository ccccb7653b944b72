#!/bin/bash
# ncu evidence for profiles/ (round 2), one gpurun call. Every ncu command follows the same
# command run plainly (exit 0). Outputs under gpurun_out/; summarised by
# scripts/ncu_kernel_table.py + scripts/profile_summaries.py into profiles/.
#   (1) launch list of the default bench command (config 2 + SPD), cold-cache, serialised
#   (2) --set full of EVERY kernel of a first assemble of config 2 + SPD (pattern, slot map,
#       Morton tile order, tile plan, SoA/connectivity copies, tile kernel, fix-ups, energy
#       trees) plus energy_only / guard_min / SpMV / block-Jacobi / PCG kernels
#   (3) --set full of EVERY kernel of a steady-state assemble of configs 2 (no SPD), 3, 4, 5
set -e
python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c2.csv \
    python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_launches.log 2>&1
run_full() {  # name, extra ncu flags, profile_step args
  python scripts/profile_step.py $3 > gpurun_out/r02_plain_$1.log 2>&1
  ncu --set full --clock-control none --import-source on $2 -c 400 -o gpurun_out/prof_r02_$1 \
      python scripts/profile_step.py $3 > gpurun_out/r02_ncu_$1.log 2>&1
}
run_full c2_first_assemble "" "--config c2 --steps 1 --extras"
run_full c2_steady "--profile-from-start off" "--config c2 --steps 1 --warm 2"
run_full c2_nospd_steady "--profile-from-start off" "--config c2 --no-spd --steps 1 --warm 2"
run_full c3_steady "--profile-from-start off" "--config c3 --steps 1 --warm 2"
run_full c4_steady "--profile-from-start off" "--config c4 --steps 1 --warm 2"
run_full c5_steady "--profile-from-start off" "--config c5 --steps 1 --warm 2"
echo done
