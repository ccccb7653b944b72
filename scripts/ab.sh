#!/bin/bash
# A/B timing of environment switches on one box: ab.sh CONFIG "ENV1" "ENV2" ...  (use "-" for none;
# several variables in one variant separated by spaces); extra bench flags in $BENCH_FLAGS
cfg=$1; shift
for rep in 1 2; do
for e in "$@"; do
  [ "$e" = "-" ] && e=""
  env $e python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline $BENCH_FLAGS 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('%-44s %s %s  %.3f ms  kernel %.3f ms  frac %.3f' % ('$e' or 'default', '$cfg', '$BENCH_FLAGS', d['ms_per_step'], r['kernel_ms'], r['frac']))"
done
done
