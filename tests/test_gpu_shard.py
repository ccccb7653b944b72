"""GPU: the device side of the sharded (owner-computes) assembly, parallel.ShardedTetSystem.

The ranks of a world-3 slab decomposition are assembled one after another on the one GPU
(independent contexts; nothing waits on another rank), their owned rows gathered and compared
with the oracle's assembly of the global grid: pattern bit-exact, E / g / H to the 1e-10
north-star tolerance, for both fast modes and with the SPD projection checked against the
oracle's numpy-eigh projection."""
import numpy as np
import pytest

from conftest import golden_tape
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200 import parallel as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["deterministic", "atomic"])
@pytest.mark.parametrize("spd", [False, True])
def test_sharded_ranks_reassemble_the_global_system(oracle_mod, mode, spd):
    world, n = 3, 4
    parts, E = [], 0.0
    for r in range(world):
        s = C.tet4_slab_case(n, world, r)
        sh = P.ShardedTetSystem(s.case.x, s.case.X, s.case.conn, s.n_own, s.case.params, s.row_lo, s.row_hi,
                                s.global_ids, spd=spd)
        E += sh.assemble(mode)
        parts.append(sh.owned())
    rp, ci, v, g = P.gather_rows(parts)
    sysm = oracle_mod.system_for_case(C.tet4_global_slab_case(n, world), golden_tape)
    ref = oracle_mod.assemble_spd(sysm) if spd else sysm.assemble()
    np.testing.assert_array_equal(rp, ref["row_ptr"])
    np.testing.assert_array_equal(ci, ref["col_idx"])
    assert abs(E - ref["E"]) / max(1.0, abs(ref["E"])) <= 1e-10
    assert oracle_mod.rel_err(g, ref["grad"]) <= 1e-10
    assert oracle_mod.rel_err(v.ravel(), ref["vals"]) <= 1e-10


@pytest.mark.parametrize("spd", [False, True])
def test_sharded_contact_ranks_reassemble_the_global_system(oracle_mod, spd):
    """Config 5 sharded over 3 ranks (run one after another on the one GPU): tets + inertia
    owner-computes, pairs owned by their point node's rank, pair rows exchanged (here routed
    in-process, rank order) and merged; gathered owned rows vs the global oracle."""
    world = 3
    case = C.config5(4, 300)
    ranks = [P.ShardedContactSystem(case, world, r, spd=spd) for r in range(world)]
    outs = [sh.assemble("deterministic") for sh in ranks]
    E = sum(o[0] for o in outs)
    parts = [ranks[r].finish(outs[r][1], [outs[src][2][r] for src in range(world)]) for r in range(world)]
    assert sum(sh.n_owned_elements() for sh in ranks) == case.conn.shape[0] + case.n_nodes + 300
    rp, ci, v, g = P.gather_rows(parts)
    sysm = oracle_mod.system_for_case(case, golden_tape)
    ref = oracle_mod.assemble_spd(sysm, spd_energies=("elastic", "contact")) if spd else sysm.assemble()
    np.testing.assert_array_equal(rp, ref["row_ptr"])
    np.testing.assert_array_equal(ci, ref["col_idx"])
    assert abs(E - ref["E"]) / max(1.0, abs(ref["E"])) <= 1e-10
    assert oracle_mod.rel_err(g, ref["grad"]) <= 1e-10
    assert oracle_mod.rel_err(v.ravel(), ref["vals"]) <= 1e-10
