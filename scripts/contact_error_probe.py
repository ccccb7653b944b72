"""Parity margin of the contact barrier (ill-conditioned: d down to 1e-7 with h ~ 1e-2) in the
fast modes, for choosing its arithmetic regime."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200.systems import DeviceSystem, golden_tape
for name, case in [("contact_n3", C.config5(3, 40)), ("c5_n8", C.config5(8, 20000)), ("c5_n20", C.config5(20, 200000))]:
    ref = O.system_for_case(case, golden_tape).assemble()
    refs = O.assemble_spd(O.system_for_case(case, golden_tape))
    for spd in (False, True):
        ds = DeviceSystem(case, spd=spd)
        r = refs if spd else ref
        for mode in ("deterministic", "atomic"):
            E = ds.asm.assemble(mode)
            print(name, "spd" if spd else "raw", mode, "E %.2e g %.2e H %.2e" % (
                abs(E - r["E"]) / max(1, abs(r["E"])), O.rel_err(ds.asm.gradient(), r["grad"]),
                O.rel_err(ds.asm.hessian_values(), r["vals"])), flush=True)
