#!/bin/bash
# quick ncu capture of one kernel of a steady assemble: prof_quick.sh NAME KERNEL "profile_step args" [env...]
set -e
O=gpurun_out/q; mkdir -p $O
name=$1; kern=$2; args=$3; shift 3
env "$@" python scripts/profile_step.py $args --steps 1 --warm 2 > $O/plain_$name.log 2>&1
env "$@" ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:$kern -c 1 -o $O/$name \
    python scripts/profile_step.py $args --steps 1 --warm 2 > $O/ncu_$name.log 2>&1
ncu -i $O/$name.ncu-rep --page raw --csv > $O/raw_$name.csv
ncu -i $O/$name.ncu-rep --page source --csv --print-source sass > $O/sass_$name.csv 2>/dev/null || true
rm -f $O/$name.ncu-rep
