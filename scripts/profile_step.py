"""Runs a few assembles of a config for ncu captures (no timing output is meaningful here)."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200.systems import DeviceSystem
p = argparse.ArgumentParser()
p.add_argument("--config", default="c2"); p.add_argument("--mode", default="deterministic"); p.add_argument("--steps", type=int, default=3)
p.add_argument("--spd", action="store_true"); p.add_argument("--no-spd", action="store_true")
a = p.parse_args()
case = {"c1": C.config1, "c2": C.config2, "c3": C.config3, "c4": C.config4, "c5": C.config5}[a.config]()
ds = DeviceSystem(case, spd=(a.spd or a.config in ("c2", "c5")) and not a.no_spd)
for _ in range(a.steps):
    E = ds.asm.assemble(a.mode)
print("E", E, "plan", ds.asm.plan_info())
