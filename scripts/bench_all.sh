#!/bin/bash
# All five BASELINE configs, both fast modes; one JSON line each into gpurun_out/bench_all_<cfg>_<mode>.log
for cfg in c1 c2 c3 c4 c5; do
  for m in deterministic atomic; do
    timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --mode $m --no-cpu-baseline > gpurun_out/bench_all_${cfg}_${m}.log 2>&1
  done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_all_*.log")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("bench_all_")[1][:-4], "%.1f Melem/s" % d["value"], "%.3f ms" % d["ms_per_step"], "kernel %.3f ms" % d["roofline"]["kernel_ms"], "frac %.3f" % d["roofline"]["frac"], "e2e %.1f" % d["e2e"]["value"])
    except Exception as e:
        print(f, "ERR", open(f).read()[-600:])
PY
