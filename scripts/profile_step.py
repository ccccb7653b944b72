"""Runs a few assembles of a config for ncu captures (no timing output is meaningful here)."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200.systems import DeviceSystem
p = argparse.ArgumentParser()
p.add_argument("--config", default="c2"); p.add_argument("--mode", default="deterministic"); p.add_argument("--steps", type=int, default=3)
p.add_argument("--spd", action="store_true"); p.add_argument("--no-spd", action="store_true")
p.add_argument("--warm", type=int, default=0, help="assembles before the profiled ones (ncu -s skips their kernels)")
p.add_argument("--extras", action="store_true", help="also energy_only, guard_min, matvec, block-Jacobi, PCG")
a = p.parse_args()
case = {"c1": C.config1, "c2": C.config2, "c3": C.config3, "c4": C.config4, "c5": C.config5}[a.config]()
ds = DeviceSystem(case, spd=(a.spd or a.config in ("c2", "c5")) and not a.no_spd)
for _ in range(a.warm):
    ds.asm.assemble(a.mode)
if a.warm:  # ncu --profile-from-start off: only the steady-state assembles below are captured
    import torch
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
for _ in range(a.steps):
    E = ds.asm.assemble(a.mode)
if a.extras:
    import numpy as np
    ds.asm.energy_only()
    ds.asm.guard_min()
    g = ds.asm.gradient()
    ds.asm.matvec(np.ones_like(g))
    ds.asm.block_jacobi(0.0)
    ds.asm.pcg(-g, tau=0.0, rel_tol=1e-6, max_iters=20)
if a.warm:
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
print("E", E, "plan", ds.asm.plan_info())
