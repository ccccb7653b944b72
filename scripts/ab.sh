#!/bin/bash
# A/B timing of environment switches on one box: ab.sh CONFIG "ENV1" "ENV2" ...  (use "-" for none)
cfg=$1; shift
for rep in 1 2; do
for e in "$@"; do
  [ "$e" = "-" ] && e=""
  env $e python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('%-44s %s  %.3f ms  kernel %.3f ms  frac %.3f' % ('$e' or 'default', '$cfg', d['ms_per_step'], r['kernel_ms'], r['frac']))"
done
done
