"""GPU: registration-time uploads are ordered. add_array zeroes the new array on the context
stream and set_array uploads on the copy stream; an unsynchronised memset could land after the
upload and silently zero the state (seen as an intermittent E = V * psi(F = 0) on config 2 at
n = 6). Many fresh contexts in a row, each checked against the oracle on its first assemble."""
import numpy as np
import pytest

from conftest import golden_tape
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200.systems import DeviceSystem

pytestmark = pytest.mark.gpu


def test_fresh_contexts_see_their_uploaded_state(oracle_mod):
    case = C.config2(6)
    ref = oracle_mod.system_for_case(case, golden_tape).energy_gradient()
    for k in range(60):
        ds = DeviceSystem(case, tapes=golden_tape)
        E = ds.asm.assemble(["deterministic", "atomic", "ordered"][k % 3])
        assert abs(E - ref["E"]) <= 1e-10 * abs(ref["E"]), (k, E)
        assert oracle_mod.rel_err(ds.asm.gradient(), ref["grad"]) <= 1e-10
