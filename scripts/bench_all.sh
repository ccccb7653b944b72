#!/bin/bash
# All configs (device timing only, no CPU baseline), one JSON line each into gpurun_out/$1_*.json
tag=${1:-bench}
for c in c2 c1 c3 c4 c5; do
  python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_$c.json 2> gpurun_out/${tag}_$c.err
done
python bench.py --config c2 --no-spd --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_c2nospd.json 2> gpurun_out/${tag}_c2nospd.err
python - "$tag" <<'PY'
import json, sys, glob
tag = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/{tag}_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d["roofline"]
    print("%-28s %8.3f ms  %9.1f Melem/s  kernel %.3f ms  frac %.3f (%s)  atomic %s  e2e %.1f  e2eH %.1f" % (
        f.split("/")[-1], d["ms_per_step"], d["value"], r["kernel_ms"], r["frac"], r["bound"],
        "%.3f ms" % d["atomic"]["ms_per_step"] if "atomic" in d else "-", d["e2e"]["value"], d["e2e_host_hessian"]["value"]))
PY
