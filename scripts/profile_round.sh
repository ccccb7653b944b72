#!/bin/bash
# ncu evidence for profiles/ (one gpurun call): (1) launch list of the default bench command
# (config 2, SPD; cold-cache, serialised), (2) one --set full capture of the dominant tile kernel
# of each config (c2 SPD, c2 without SPD, c3, c4 bending, c5 contact + its tets). Every ncu run
# follows an identical plain run that exited 0.
set -e
python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof_bench_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
full() {  # name, kernel regex, launch-skip, launch-count, profile_step args
  python scripts/profile_step.py $5 > gpurun_out/prof_plain_$1.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c $4 -o gpurun_out/prof_r01_$1 \
      python scripts/profile_step.py $5 > gpurun_out/ncu_full_$1.log 2>&1
}
full c2_spd_tile sy_7 1 1 "--config c2 --steps 3"
full c2_nospd_tile sy_6 1 1 "--config c2 --no-spd --steps 3"
full c5_tiles sy_7 2 2 "--config c5 --steps 3"
full c4_tiles sy_6 2 2 "--config c4 --steps 3"
full c3_tile sy_6 1 1 "--config c3 --steps 3"
echo done
