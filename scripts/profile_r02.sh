#!/bin/bash
# ncu evidence for profiles/ (round 2). usage: profile_r02.sh PART   (PART = c2 | others)
# Every ncu command follows the same command run plainly (exit 0). Reports are exported on the
# box (raw metrics CSV for every kernel, details text, source regions of the generated tile
# kernels) and only the dominant kernel's report is kept, so gpurun_out stays small.
set -e
mkdir -p gpurun_out/r02
O=gpurun_out/r02
src() { python scripts/dump_kernel_source.py $1 $2 $O/src > /dev/null 2>&1; }
run_full() {  # name, extra ncu flags, profile_step args
  python scripts/profile_step.py $3 > $O/plain_$1.log 2>&1
  ncu --set full --clock-control none --import-source on $2 -o $O/prof_$1 \
      python scripts/profile_step.py $3 > $O/ncu_$1.log 2>&1
  ncu -i $O/prof_$1.ncu-rep --page raw --csv > $O/raw_$1.csv
  ncu -i $O/prof_$1.ncu-rep --page details > $O/details_$1.txt
}
regions() {  # name, kernel, source file
  NCU_FILTER="--kernel-name $2" python scripts/ncu_regions.py $O/prof_$1.ncu-rep $O/src/$3 > $O/regions_$1_$2.txt 2>&1 || true
}
if [ "$1" = c2 ]; then
  src tet4 1; src tet4 0
  python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_bench.log 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv \
      python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
  run_full c2_first_assemble "-c 400" "--config c2 --steps 1 --extras"
  rm -f $O/prof_c2_first_assemble.ncu-rep
  run_full c2_steady "--profile-from-start off" "--config c2 --steps 1 --warm 2"
  regions c2_steady sy_7 tet4_spd_elastic.cu
  run_full c2_nospd_steady "--profile-from-start off" "--config c2 --no-spd --steps 1 --warm 2"
  regions c2_nospd_steady sy_6 tet4_elastic.cu
  rm -f $O/prof_c2_nospd_steady.ncu-rep
else
  src contact 1; src cloth 0; src tet10 0
  run_full c3_steady "--profile-from-start off" "--config c3 --steps 1 --warm 2"
  regions c3_steady sy_6 tet10_elastic.cu
  rm -f $O/prof_c3_steady.ncu-rep
  run_full c4_steady "--profile-from-start off" "--config c4 --steps 1 --warm 2"
  regions c4_steady sy_6 cloth_bending.cu
  rm -f $O/prof_c4_steady.ncu-rep
  run_full c5_steady "--profile-from-start off" "--config c5 --steps 1 --warm 2"
  regions c5_steady sy_7 contact_spd_contact.cu
  rm -f $O/prof_c5_steady.ncu-rep
fi
du -sh $O
echo done
