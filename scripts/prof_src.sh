#!/bin/bash
# per-line ncu source page of a generated tile kernel, exported on the box:
#   prof_src.sh NAME "profile_step args" KERNEL KIND SPD SRCFILE [KERNEL_ID]
set -e
O=gpurun_out/ps; mkdir -p $O
name=$1; args=$2; kern=$3; kind=$4; spd=$5; srcf=$6; kid=${7:-0}
python scripts/dump_kernel_source.py $kind $spd $O/src > /dev/null 2>&1
python scripts/profile_step.py $args --steps 1 --warm 2 > $O/plain_$name.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name $kern -o $O/$name \
    python scripts/profile_step.py $args --steps 1 --warm 2 > $O/ncu_$name.log 2>&1
ncu -i $O/$name.ncu-rep --page raw --csv > $O/raw_$name.csv
ncu -i $O/$name.ncu-rep --page details > $O/details_$name.txt
for k in 0 1; do
ncu -i $O/$name.ncu-rep --launch-skip $k --launch-count 1 --page source --csv --print-source cuda,sass --resolve-source-file $O/src/$srcf > $O/source_${name}_$k.csv 2>&1 || true
ncu -i $O/$name.ncu-rep --launch-skip $k --launch-count 1 --page source --csv --print-source sass > $O/sass_${name}_$k.csv 2>&1 || true
done
rm -f $O/$name.ncu-rep
ls -la $O
