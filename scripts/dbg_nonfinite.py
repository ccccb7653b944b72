import os, sys, re
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from test_gpu_edge_cases import _chain_system, _register_chain
from paper_2303_02156_b200.device import SymelError
rng = np.random.default_rng(5)
for trial in range(4):
    x, conn, tape, inputs = _chain_system(4, 2000, 6000, 100 + trial)
    bad = np.sort(rng.choice(2000, 2, replace=False))
    for e in bad:
        x[conn[e, 1]] = x[conn[e, 0]]
    for mode in ("deterministic", "atomic", "ordered"):
        A, sysm = _register_chain(x, conn, tape, inputs, 4, 1.0)
        ref = sysm.assemble()
        try:
            A.assemble(mode)
            msg = "no error"
        except SymelError as ex:
            msg = str(ex)
        outs = A.element_outputs(0, 0, 2000, 1 + 12 + 144, mode=mode)
        nf = np.flatnonzero(~np.isfinite(outs).all(axis=1))
        print(trial, mode, "bad", bad, "ref", ref["bad_element"], "dev:", msg, "| nonfinite elems (element_outputs):", nf[:5])
