#!/bin/bash
# launch lists (gpu__time_duration per kernel) for configs 3-5, one steady step after warm-up
for cfg in c3 c4 c5; do
  python scripts/profile_step.py --config $cfg --steps 3 > gpurun_out/plain_$cfg.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv \
      python scripts/profile_step.py --config $cfg --steps 3 > gpurun_out/ncu_$cfg.log 2>&1
done
echo done
