"""GPU edge cases through the generic C-ABI registration (DeviceAssembler), each against the C
oracle built with the identical registration:

* b = 1: the tet tape bound to a 1-component dof array (12 "nodes" per element), so the
  assembly.hpp:273-276 rule picks scalar blocks -- pattern, gradient and values;
* an energy with no elements next to a populated one; nodes no element touches (their diagonal
  block exists and is zero, assembly.hpp:299-300);
* contact pairs that are all inactive (activation empties the energy) and a second assemble
  after re-activating them (pattern rebuilt).
"""
import numpy as np
import pytest

from conftest import golden_tape
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200 import systems as S
from paper_2303_02156_b200.device import DeviceAssembler, IN_ITEM, SymelError

pytestmark = pytest.mark.gpu
TOL = 1e-10
MODES = ["ordered", "deterministic", "atomic"]


def check(dev, ref, oracle_mod, tol=TOL):
    E, g, H = dev
    assert H.b == ref["b"]
    np.testing.assert_array_equal(H.row_ptr, ref["row_ptr"])
    np.testing.assert_array_equal(H.col_idx, ref["col_idx"])
    assert abs(E - ref["E"]) / max(1.0, abs(ref["E"])) <= tol
    assert oracle_mod.rel_err(g, ref["grad"]) <= tol
    assert oracle_mod.rel_err(H.values, ref["vals"]) <= tol


def device_result(A, mode):
    E = A.assemble(mode)
    return E, A.gradient(), A.hessian()


@pytest.mark.parametrize("mode", MODES)
def test_scalar_blocks_b1(mode, oracle_mod):
    case = C.tet4_case(3, name="b1")
    p = case.params
    n = case.n_nodes
    # every tet "node" dof becomes its own item of a 1-component array
    conn12 = (case.conn[:, :, None] * 3 + np.arange(3)[None, None, :]).reshape(-1, 12)
    x1 = case.x.reshape(-1, 1)
    conn_both = np.concatenate([conn12, case.conn], axis=1)  # slots 0-11: scalar dofs, 12-15: rest nodes
    inputs = [(IN_ITEM, 0, k, 0) for k in range(12)] + [(IN_ITEM, 1, 12 + a, c) for a in range(4) for c in range(3)] \
        + [(S.IN_PARAM, 0, 0, 0)] * 2
    A = DeviceAssembler()
    xa = A.add_array("x", 3 * n, 1, True)
    ra = A.add_array("rest", n, 3)
    A.set_array(xa, x1)
    A.set_array(ra, case.X)
    cid = A.add_connectivity("tets", 16)
    A.set_elements(cid, conn_both)
    A.add_energy("elastic", cid, golden_tape("tet4_elastic"), inputs, range(12), params={24: p["mu"], 25: p["lambda"]})
    from oracle import oracle as O
    sysm = O.System()
    ox = sysm.add_array("x", x1, 1, True)
    orr = sysm.add_array("rest", case.X, 3)
    sysm.add_energy("elastic", conn_both, 16, golden_tape("tet4_elastic"), inputs, range(12),
                    params={24: p["mu"], 25: p["lambda"]})
    ref = sysm.assemble()
    assert ref["b"] == 1
    check(device_result(A, mode), ref, oracle_mod, 1e-13 if mode == "ordered" else TOL)


@pytest.mark.parametrize("mode", MODES)
def test_empty_energy_and_isolated_nodes(mode, oracle_mod):
    case = C.tet4_case(3, name="iso")
    p = case.params
    extra = 7                                  # nodes no element touches
    x = np.concatenate([case.x, np.random.default_rng(3).random((extra, 3))])
    X = np.concatenate([case.X, np.random.default_rng(4).random((extra, 3))])
    A = DeviceAssembler()
    xa = A.add_array("x", x.shape[0], 3, True)
    ra = A.add_array("rest", x.shape[0], 3)
    A.set_array(xa, x)
    A.set_array(ra, X)
    t = A.add_connectivity("tets", 4)
    A.set_elements(t, case.conn)
    A.add_energy("elastic", t, golden_tape("tet4_elastic"), S.solid_tet_inputs(xa, ra), range(12),
                 params={24: p["mu"], 25: p["lambda"]})
    t0 = A.add_connectivity("none", 4)
    A.set_elements(t0, np.zeros((0, 4), np.int64))
    A.add_energy("empty", t0, golden_tape("tet4_elastic"), S.solid_tet_inputs(xa, ra), range(12),
                 params={24: p["mu"], 25: p["lambda"]})
    from oracle import oracle as O
    sysm = O.System()
    ox = sysm.add_array("x", x, 3, True)
    orr = sysm.add_array("rest", X, 3)
    sysm.add_energy("elastic", case.conn, 4, golden_tape("tet4_elastic"), S.solid_tet_inputs(ox, orr), range(12),
                    params={24: p["mu"], 25: p["lambda"]})
    sysm.add_energy("empty", np.zeros((0, 4), np.int64), 4, golden_tape("tet4_elastic"), S.solid_tet_inputs(ox, orr),
                    range(12), params={24: p["mu"], 25: p["lambda"]})
    ref = sysm.assemble()
    E, g, H = device_result(A, mode)
    check((E, g, H), ref, oracle_mod, 1e-13 if mode == "ordered" else TOL)
    n = case.n_nodes
    for r in range(n, n + extra):  # isolated rows: the diagonal block only, zero
        k0, k1 = H.row_ptr[r], H.row_ptr[r + 1]
        assert k1 - k0 == 1 and H.col_idx[k0] == r
        assert not np.any(H.values.reshape(-1, 9)[k0])
    assert not np.any(g[3 * n:])


def test_all_pairs_inactive_then_active(oracle_mod):
    case = C.config5(3, 30)
    off = case.extra["offsets"].reshape(-1, 4, 3).copy()
    q = case.x[case.extra["pairs"]] + off
    nrm = np.cross(q[:, 2] - q[:, 1], q[:, 3] - q[:, 1])
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    far = off.copy()
    far[:, 0] += 5e-3 * nrm                    # every point beyond d_hat: nothing active
    inactive = C.Case(case.name, case.kind, case.x, case.X, case.conn, case.params,
                      dict(case.extra, offsets=far.reshape(-1, 12)))
    ds = S.DeviceSystem(inactive)
    from oracle import oracle as O
    for mode in MODES:
        ref = O.system_for_case(inactive, golden_tape).assemble()
        check(device_result(ds.asm, mode), ref, oracle_mod, 1e-13 if mode == "ordered" else TOL)
        assert ds.asm.active_count(ds.energies["contact"]) == 0
    # back in range: activation refresh rebuilds the pattern with the pairs
    ds.asm.set_array(ds.arrays["pair_offset"], case.extra["offsets"])
    ref = O.system_for_case(case, golden_tape).assemble()
    for mode in MODES:
        check(device_result(ds.asm, mode), ref, oracle_mod, 1e-13 if mode == "ordered" else TOL)
    assert ds.asm.active_count(ds.energies["contact"]) == 30


@pytest.mark.parametrize("mode", ["deterministic", "atomic"])
def test_topology_change(mode, oracle_mod):
    """New connectivity on a live context (the reference's topology stamp, assembly.hpp:207-225):
    the pattern, slot maps and tile plan are rebuilt and results follow the new element set."""
    case = C.tet4_case(4, name="topo")
    p = case.params
    ds = S.DeviceSystem(case)
    ds.asm.assemble(mode)
    from oracle import oracle as O
    for keep in (case.conn[::2], case.conn[1::3], case.conn):
        ds.asm.set_elements(0, keep)  # connectivity 0 = "tets"
        sub = C.Case(case.name, case.kind, case.x, case.X, keep, p)
        ref = O.system_for_case(sub, golden_tape).assemble()
        check(device_result(ds.asm, mode), ref, oracle_mod)


def _assemble_with_env(case, spd, env, mode="deterministic"):
    """A fresh context built while `env` is set (the code generator reads its diagnostic
    switches when it specialises a kernel)."""
    import os
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        ds = S.DeviceSystem(case, tapes=S.default_tapes(), spd=spd)
        E = ds.asm.assemble(mode)
        return E, ds.asm.gradient(), ds.asm.hessian()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_ql_lookahead_is_bitwise_the_plain_ql():
    """The per-lane QL lookahead (codegen sy_ql_la) only reschedules sweeps across a warp; on the
    device too the projected Hessian is bit-identical to the plain QL's (sy_ql)."""
    case = C.config2(6)
    E0, g0, H0 = _assemble_with_env(case, True, {})
    E1, g1, H1 = _assemble_with_env(case, True, {"SYMEL_NO_QL_LOOKAHEAD": "1"})
    assert E0 == E1
    np.testing.assert_array_equal(g0, g1)
    np.testing.assert_array_equal(H0.values, H1.values)


def test_item_lane_reduce_scatter_matches_sequential_item_sum(oracle_mod):
    """tet10's quadrature terms summed by the four-lane reduce-scatter (pairwise order) against
    the per-output shuffle tree (the reference's sequential order): equal to rounding."""
    case = C.config3(3)
    E0, g0, H0 = _assemble_with_env(case, False, {})
    E1, g1, H1 = _assemble_with_env(case, False, {"SYMEL_NO_QUAD_REDUCE": "1"})
    np.testing.assert_array_equal(H0.col_idx, H1.col_idx)
    assert abs(E0 - E1) <= 1e-13 * max(1.0, abs(E1))
    assert oracle_mod.rel_err(g0, g1) <= 1e-13
    assert oracle_mod.rel_err(H0.values, H1.values) <= 1e-13


def test_graph_replay_tracks_params_state_and_modes():
    """The tiled assemble is replayed from a recorded CUDA graph while its launch signature is
    unchanged: a new param value (read at every assemble) and new positions must show up, and
    alternating modes must each replay their own recording."""
    case = C.tet4_case(4)
    ds = S.DeviceSystem(case, tapes=S.default_tapes())
    eid = ds.energies["elastic"]
    ref0 = [ds.asm.assemble(m) for m in ("deterministic", "atomic", "deterministic")]
    assert ref0[0] == ref0[2]
    # param change -> re-record; equal to a fresh context built with that value
    ds.asm.set_param(eid, 24, 2.0 * case.params["mu"])
    E1 = ds.asm.assemble("deterministic")
    H1 = ds.asm.hessian().values.copy()
    case2 = C.tet4_case(4)
    case2.params["mu"] = 2.0 * case.params["mu"]
    ds2 = S.DeviceSystem(case2, tapes=S.default_tapes())
    assert E1 == ds2.asm.assemble("deterministic")
    np.testing.assert_array_equal(H1, ds2.asm.hessian().values)
    # new positions through the same recording (same buffers): equal to the fresh context's
    x = case.x + 1e-3
    ds.asm.set_array(ds.arrays["x"], x)
    ds2.asm.set_array(ds2.arrays["x"], x)
    assert ds.asm.assemble("deterministic") == ds2.asm.assemble("deterministic")
    np.testing.assert_array_equal(ds.asm.gradient(), ds2.asm.gradient())


def _chain_system(nodes, n_elem, n_pts, seed, c=0.0):
    """Random point cloud + elements of `nodes` distinct random points, energy = the hand-built
    chain tape (tests/tapegen.py); device and oracle registered identically."""
    from tapegen import chain_quartic_tape
    from oracle import oracle as O
    rng = np.random.default_rng(seed)
    x = rng.random((n_pts, 3))
    conn = np.stack([rng.choice(n_pts, nodes, replace=False) for _ in range(n_elem)]).astype(np.int64)
    tape = chain_quartic_tape(nodes)
    inputs = [(IN_ITEM, 0, a, k) for a in range(nodes) for k in range(3)] + [(S.IN_PARAM, 0, 0, 0)]
    return x, conn, tape, inputs


def _register_chain(x, conn, tape, inputs, nodes, c):
    from oracle import oracle as O
    A = DeviceAssembler()
    xa = A.add_array("x", x.shape[0], 3, True)
    A.set_array(xa, x)
    cid = A.add_connectivity("chains", nodes)
    A.set_elements(cid, conn)
    A.add_energy("chain", cid, tape, inputs, range(3 * nodes), params={3 * nodes: c})
    sysm = O.System()
    sysm.add_array("x", x, 3, True)
    sysm.add_energy("chain", conn, nodes, tape, inputs, range(3 * nodes), params={3 * nodes: c})
    return A, sysm


@pytest.mark.parametrize("mode", MODES)
def test_large_element_23_nodes(mode, oracle_mod):
    """23-node elements (276 upper local sub-blocks > the tile plan's 8-bit sub-block code):
    the assembler must route them off the tile path and still match the oracle."""
    nodes = 23
    x, conn, tape, inputs = _chain_system(nodes, 300, 900, 11)
    A, sysm = _register_chain(x, conn, tape, inputs, nodes, 0.0)
    ref = sysm.assemble()
    check(device_result(A, mode), ref, oracle_mod, 1e-12 if mode == "ordered" else TOL)


@pytest.mark.parametrize("nodes", [4, 22])
def test_chain_tape_tile_path(nodes, oracle_mod):
    """The same hand-built energy at sizes the tile plan packs (n_lb <= 22)."""
    x, conn, tape, inputs = _chain_system(nodes, 700, 2000, 12)
    A, sysm = _register_chain(x, conn, tape, inputs, nodes, 0.0)
    ref = sysm.assemble()
    for mode in MODES:
        check(device_result(A, mode), ref, oracle_mod, 1e-12 if mode == "ordered" else TOL)


@pytest.mark.parametrize("mode", MODES)
def test_non_finite_names_lowest_element_across_tiles(mode, oracle_mod):
    """check_finite names the lowest (energy, element) (assembly.hpp:426-438), also when the
    non-finite elements sit in different tiles whose spatial (Morton) order differs from the
    element order."""
    import re
    rng = np.random.default_rng(5)
    for trial in range(4):
        x, conn, tape, inputs = _chain_system(4, 2000, 6000, 100 + trial)
        bad = np.sort(rng.choice(2000, 2, replace=False))
        for e in bad:
            x[conn[e, 1]] = x[conn[e, 0]]  # first two nodes coincide: c / (d0.d0) = inf
        A, sysm = _register_chain(x, conn, tape, inputs, 4, 1.0)
        ref = sysm.assemble()
        assert ref["status"] == 4 and ref["bad_energy"] == 0
        assert ref["bad_element"] == min(e for e in range(2000)
                                         if np.all(x[conn[e, 1]] == x[conn[e, 0]]))
        with pytest.raises(SymelError) as ei:
            A.assemble(mode)
        m = re.search(r"element (\d+)", str(ei.value))
        assert m and int(m.group(1)) == ref["bad_element"], (str(ei.value), ref["bad_element"])


@pytest.mark.parametrize("depth", [(2, 1), (4, 4), (12, 6)])
@pytest.mark.parametrize("kind", ["contact", "tet10", "cloth"])
def test_metadata_prefetch_depth(kind, depth, oracle_mod, monkeypatch):
    """The tile reduction's segment-metadata prefetch depth (chosen from the plan: deeper for
    tiles with many short rounds, symel_cuda.cpp Energy::meta_depth) only changes when loads are
    issued: every depth gives the deterministic result of depth 1, bit for bit, and matches the
    oracle. Depths beyond the number of rounds of a tile (predicated-off loads) included."""
    case = {"contact": lambda: C.config5(3, 400), "tet10": lambda: C.config3(3), "cloth": lambda: C.config4(12)}[kind]()
    spd = kind == "contact"
    monkeypatch.setenv("SYMEL_META_DEPTH_H", "1")
    monkeypatch.setenv("SYMEL_META_DEPTH_G", "1")
    base = S.DeviceSystem(case, tapes=golden_tape, spd=spd)
    E0 = base.asm.assemble("deterministic")
    g0, H0 = base.asm.gradient(), base.asm.hessian().values
    monkeypatch.setenv("SYMEL_META_DEPTH_H", str(depth[0]))
    monkeypatch.setenv("SYMEL_META_DEPTH_G", str(depth[1]))
    ds = S.DeviceSystem(case, tapes=golden_tape, spd=spd)
    E = ds.asm.assemble("deterministic")
    assert E == E0
    assert np.array_equal(ds.asm.gradient().view(np.uint64), g0.view(np.uint64))
    assert np.array_equal(ds.asm.hessian().values.view(np.uint64), H0.view(np.uint64))
    if not spd:
        ref = oracle_mod.system_for_case(case, golden_tape).assemble()
        assert abs(E - ref["E"]) <= 1e-10 * max(1.0, abs(ref["E"]))
        assert oracle_mod.rel_err(ds.asm.gradient(), ref["grad"]) <= 1e-10
        assert oracle_mod.rel_err(ds.asm.hessian().values, ref["vals"]) <= 1e-10
    Ea = ds.asm.assemble("atomic")
    assert abs(Ea - E0) <= 1e-12 * max(1.0, abs(E0))
    assert oracle_mod.rel_err(ds.asm.hessian().values, H0) <= 1e-12
