#!/bin/bash
# ncu source-region A/B of the c2 SPD tile kernel: full QL vs smaller-set clamp
set -e
mkdir -p gpurun_out/src
for v in full ss; do
  if [ $v = full ]; then export SYMEL_SPD_FULL_QL=1; else unset SYMEL_SPD_FULL_QL; fi
  python scripts/dump_kernel_source.py tet4 1 gpurun_out/src_$v > /dev/null 2>&1
  python scripts/profile_step.py --config c2 --steps 1 --warm 1 > gpurun_out/pab_plain_$v.log 2>&1
  ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:sy_7 -c 1 \
      -o gpurun_out/pab_$v python scripts/profile_step.py --config c2 --steps 1 --warm 1 > gpurun_out/pab_ncu_$v.log 2>&1
  python scripts/ncu_regions.py gpurun_out/pab_$v.ncu-rep gpurun_out/src_$v/tet4_spd_elastic.cu > gpurun_out/pab_regions_$v.txt 2>&1 || true
  ncu -i gpurun_out/pab_$v.ncu-rep --page raw --csv > gpurun_out/pab_raw_$v.csv 2>&1 || true
done
