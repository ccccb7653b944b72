import os, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from oracle import oracle as O
from paper_2303_02156_b200 import configs as C, systems as S
from paper_2303_02156_b200.device import ENERGY_EXACT
case = C.config4()
ref = O.system_for_case(case, S.golden_tape).energy_gradient()
for exact in ([], ["bending"], ["membrane"], ["bending", "membrane"]):
    ds = S.DeviceSystem(case)
    for n in exact:
        ds.asm.set_energy_flags(ds.energies[n], ENERGY_EXACT)
    for _ in range(3):
        E = ds.asm.assemble()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        E = ds.asm.assemble()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) * 100
    g = ds.asm.gradient()
    print(exact, "ms %.3f" % ms, "errE %.2e" % (abs(E - ref["E"]) / max(1, abs(ref["E"]))), "abs %.2e" % abs(E - ref["E"]),
          "errg %.2e" % O.rel_err(g, ref["grad"]), "eval_ms %.3f" % ds.asm.timings().eval_ms)
