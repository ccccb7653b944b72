#!/bin/bash
# ncu --set full of every kernel of one steady assemble: prof_cfg.sh NAME "profile_step args" [env...]
set -e
O=gpurun_out/q; mkdir -p $O
name=$1; args=$2; shift 2
env "$@" python scripts/profile_step.py $args --steps 1 --warm 2 > $O/plain_$name.log 2>&1
env "$@" ncu --set full --clock-control none --profile-from-start off -o $O/$name \
    python scripts/profile_step.py $args --steps 1 --warm 2 > $O/ncu_$name.log 2>&1
ncu -i $O/$name.ncu-rep --page raw --csv > $O/raw_$name.csv
rm -f $O/$name.ncu-rep
