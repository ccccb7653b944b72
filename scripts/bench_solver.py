"""Device SpMV / PCG measurement on an assembled config. Prints one JSON line:
SpMV effective bandwidth against the HBM roofline (algorithmic bytes: per block 72 B values +
4 B column, per row 4 B row pointer, x read and y written once) and PCG time per iteration."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200.systems import DeviceSystem

p = argparse.ArgumentParser()
p.add_argument("--config", default="c2"); p.add_argument("--reps", type=int, default=20)
p.add_argument("--spd", type=int, default=1); p.add_argument("--pcg-iters", type=int, default=200)
a = p.parse_args()
case = {"c1": C.config1, "c2": C.config2, "c4": C.config4}[a.config]()
ds = DeviceSystem(case, spd=bool(a.spd))
A = ds.asm
A.assemble("deterministic")
b, nr, nb, nd = A.pattern_info()
x = torch.randn(nd, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
stream = torch.cuda.ExternalStream(A.stream())
lib = A.lib
for _ in range(3):
    lib.symel_cuda_matvec(A.h, x.data_ptr(), y.data_ptr(), 1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(a.reps):
    lib.symel_cuda_matvec(A.h, x.data_ptr(), y.data_ptr(), 1)
e1.record(stream); e1.synchronize()
ms = e0.elapsed_time(e1) / a.reps
alg = nb * (b * b * 8 + 4) + (nr + 1) * 4 + 2 * nd * 8
pk = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
hbm = json.load(open(pk))["hbm_gbs"] if os.path.exists(pk) else 6557.4
g = A.gradient()
xs, st = A.pcg(-g, 0.0, 1e-12, a.pcg_iters)
out = {"op": "bsr_spmv", "config": a.config, "spd": bool(a.spd), "n_block_rows": nr, "n_blocks": nb, "ms": ms,
       "algorithmic_bytes": alg, "achieved_GBps": alg / (ms * 1e-3) / 1e9, "peak_GBps": hbm,
       "frac": alg / (ms * 1e-3) / 1e9 / hbm,
       "pcg": {"iters": st["iters"], "solve_ms": st["solve_ms"], "ms_per_iter": st["solve_ms"] / max(1, st["iters"]),
               "converged": st["converged"], "neg_curvature": st["neg_curvature"], "rel_residual": st["rel_residual"]}}
print(json.dumps(out))
