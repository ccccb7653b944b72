"""Prints the SPD-projection parity margin (relative error vs the numpy-eigh oracle) for small
configs -- how far below the 1e-10 tolerance the fused eigen-clamp stays."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200.systems import DeviceSystem, golden_tape
for name, case in [("c2_n10", C.config2(10)), ("c2_n20", C.config2(20)), ("c5_n6", C.config5(6, 2000))]:
    ds = DeviceSystem(case, spd=True)
    E = ds.asm.assemble("deterministic")
    H = ds.asm.hessian()
    ref = O.assemble_spd(O.system_for_case(case, golden_tape))
    print(name, "E %.2e g %.2e H %.2e" % (abs(E - ref["E"]) / max(1, abs(ref["E"])), O.rel_err(ds.asm.gradient(), ref["grad"]),
                                           O.rel_err(H.values, ref["vals"])), flush=True)
