import sys, numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200.systems import DeviceSystem, golden_tape
seq = [(C.tet4_case(3, name='a'), m) for m in ['ordered', 'deterministic', 'atomic']] + [(C.config2(6), m) for m in ['ordered', 'deterministic', 'atomic', 'ordered']]
for case, mode in seq:
    ref = O.system_for_case(case, golden_tape).assemble()
    ds = DeviceSystem(case, tapes=golden_tape)
    E = ds.asm.assemble(mode)
    print(case.name, mode, E, ref['E'], 'g', O.rel_err(ds.asm.gradient(), ref['grad']), 'H', O.rel_err(ds.asm.hessian_values(), ref['vals']), flush=True)
    del ds
