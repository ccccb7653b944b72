import sys, os, numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200.systems import DeviceSystem, golden_tape
keep = sys.argv[1] == 'keep'
a = C.tet4_case(3, name='a'); c2 = C.config2(6)
ds1 = DeviceSystem(a, tapes=golden_tape); ds1.asm.assemble('ordered')
if not keep:
    del ds1
ref = O.system_for_case(c2, golden_tape)
r = ref.assemble()
el = ref.element_outputs(0, 0, 1296)
ds = DeviceSystem(c2, tapes=golden_tape)
eo = ds.asm.element_outputs(0, 0, 1296, 157, 'ordered')
print('elem max diff', np.abs(eo - el).max())
x = ds.asm.get_array(ds.x, c2.x.size); X = ds.asm.get_array(ds.rest, c2.X.size)
print('x ok', np.array_equal(x, c2.x.ravel()), 'X ok', np.array_equal(X, c2.X.ravel()))
E = ds.asm.assemble('ordered')
H = ds.asm.hessian()
print('E', E, r['E'], 'pattern ok', np.array_equal(H.row_ptr, r['row_ptr']), np.array_equal(H.col_idx, r['col_idx']))
print('g err', O.rel_err(ds.asm.gradient(), r['grad']))
