import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from paper_2303_02156_b200 import configs as C, systems as S
from oracle import oracle as O
case = C.config2(6)
ref = O.system_for_case(case, S.golden_tape).assemble()
print("oracle E", ref["E"])
order = sys.argv[1:]
for tag in order:
    env = {"plain": {"SYMEL_NO_QL_LOOKAHEAD": "1"}, "la": {}, "plain_nograph": {"SYMEL_NO_QL_LOOKAHEAD": "1", "SYMEL_NO_GRAPH": "1"}}[tag]
    for k in ("SYMEL_NO_QL_LOOKAHEAD", "SYMEL_NO_GRAPH"):
        os.environ.pop(k, None)
    os.environ.update(env)
    ds = S.DeviceSystem(case, tapes=S.golden_tape, spd=True)
    Es = [ds.asm.assemble("deterministic") for _ in range(3)]
    g = ds.asm.gradient()
    print(tag, Es, "grad err", O.rel_err(g, ref["grad"]))
