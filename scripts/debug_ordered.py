import sys, numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200.systems import DeviceSystem, golden_tape
case = C.config2(6)
ref = O.system_for_case(case, golden_tape).assemble()
sysm = O.system_for_case(case, golden_tape)
el = sysm.element_outputs(0, 0, 1296)
print('oracle E', ref['E'], 'sum elem E', el[:, 0].sum())
for mode in ['ordered', 'deterministic', 'ordered', 'atomic', 'ordered']:
    ds = DeviceSystem(case, tapes=golden_tape)
    E = ds.asm.assemble(mode)
    eo = ds.asm.element_outputs(0, 0, 1296, 157, 'ordered')
    print(mode, E, 'elem ordered sum', eo[:, 0].sum(), 'max elem diff', np.abs(eo - el).max(), 'grad err', O.rel_err(ds.asm.gradient(), ref['grad']))
    E2 = ds.asm.assemble(mode)
    print('  again', E2)
