"""CPU tests: the C oracle (oracle/symel_oracle.c) against the reference's own outputs
(golden fixtures made by oracle/make_golden.py from the unmodified reference), plus the
reference's behavioural contracts restated (test_solver.cpp, test_binding.cpp)."""
import hashlib

import numpy as np
import pytest

from conftest import golden, golden_tape
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200 import systems as S

CASES = {
    "tet4_n3": lambda: C.tet4_case(3, name="tet4_n3"),
    "tet4_c1": lambda: C.config1(20),
    "tet4_c2_n6": lambda: C.config2(6),
    "tet10_n2": lambda: C.config3(2),
    "cloth_n8": lambda: C.config4(8),
    "contact_n3": lambda: C.config5(3, 40),
}


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


@pytest.mark.parametrize("name", list(CASES))
def test_generators_are_pinned(name):
    """Seeded synthetic inputs reproduce the ones the golden fixtures were made from."""
    g = golden(name)
    case = CASES[name]()
    assert digest(case.x) == g["x_digest"][0]
    assert digest(case.X) == g["X_digest"][0]
    assert digest(case.conn) == g["conn_digest"][0]


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_matches_reference_bitwise(name, oracle_mod):
    """C restatement == reference Assembler::assemble bit for bit (same op order, IEEE, no FMA)."""
    g = golden(name)
    case = CASES[name]()
    r = oracle_mod.system_for_case(case, golden_tape).assemble()
    assert r["status"] == 0
    assert r["E"] == g["E"][0]
    np.testing.assert_array_equal(r["row_ptr"], g["row_ptr"])
    np.testing.assert_array_equal(r["col_idx"], g["col_idx"])
    np.testing.assert_array_equal(r["grad"], g["grad"])
    if "vals" in g:
        np.testing.assert_array_equal(r["vals"], g["vals"])
    else:
        v = r["vals"].reshape(-1, 9)
        np.testing.assert_array_equal(v[g["vals_sample_blocks"]], g["vals_sample"])
        assert np.abs(r["vals"]).sum() == pytest.approx(g["vals_abs_sum"][0], rel=1e-14)


@pytest.mark.parametrize("name", ["tet4_n3", "tet10_n2", "cloth_n8", "contact_n3"])
def test_oracle_element_outputs_bitwise(name, oracle_mod):
    g = golden(name)
    case = CASES[name]()
    sysm = oracle_mod.system_for_case(case, golden_tape)
    for i, e in enumerate(sysm.energies):
        key = "elem_" + e["name"]
        ref = g[key]
        nd = len(e["dof_slots"])
        stride = 1 + nd + nd * nd
        count = ref.size // stride
        out = sysm.element_outputs(i, 0, count)
        np.testing.assert_array_equal(out.ravel(), ref)


def test_cloth_rest_data_matches_reference():
    """numpy restatements of scene.hpp:783-805, mesh_io.hpp:170-189, energies.hpp:684-736."""
    g = golden("cloth_n8")
    case = C.config4(8)
    np.testing.assert_array_equal(case.extra["flaps"].ravel(), g["ref_flaps"])
    np.testing.assert_array_equal(case.extra["dm2inv"].ravel(), g["ref_dm2inv"])
    np.testing.assert_array_equal(case.extra["area"].ravel(), g["ref_area"])
    np.testing.assert_array_equal(C.bending_Q_for(case).ravel(), g["ref_Q"])


def test_config_counts():
    """element / node counts of the BASELINE configs (small-n generators scale)."""
    X, t = C.kuhn_grid(20)
    assert X.shape[0] == 9261 and t.shape[0] == 48000
    X4, t4 = C.kuhn_grid(4)
    Xq, c10 = C.expand_quadratic(t4, X4)
    assert c10.shape == (6 * 64, 10)
    Xc, tris, _ = C.cloth_grid(1000)
    assert tris.shape[0] == 1_996_002
    flaps = C.interior_edge_flaps(C.cloth_grid(50)[1])
    # interior edges of an N x N grid with one diagonal per quad: 3(N-1)^2 - 2(N-1) ... boundary excluded
    n = 49
    assert flaps.shape[0] == 3 * n * n - 2 * n


def test_quadratic_nodes():
    X4, t = C.kuhn_grid(40)
    Xq, c = C.expand_quadratic(t, X4)
    assert Xq.shape[0] == 531_441 and c.shape[0] == 384_000


def test_contact_pairs_geometry():
    case = C.config5(4, 2000)
    ex = case.extra
    q = case.x[ex["pairs"]] + ex["offsets"].reshape(-1, 4, 3)
    n = np.cross(q[:, 2] - q[:, 1], q[:, 3] - q[:, 1])
    d = np.einsum("ij,ij->i", n, q[:, 0] - q[:, 1]) / np.linalg.norm(n, axis=1)
    assert np.all(d > 0) and np.all(d <= 1e-3)
    assert d.min() >= 1e-7 * 0.999
    e = [np.linalg.norm(q[:, a] - q[:, b], axis=1) for a, b in ((1, 2), (2, 3), (3, 1))]
    longest = np.max(e, axis=0)
    area = 0.5 * np.linalg.norm(n, axis=1)
    assert np.all(longest ** 2 / (2 * area) <= 10.0 + 1e-9)
    assert np.all([len(set(p)) == 4 for p in ex["pairs"][:200]])


def test_tape_interpreter_matches_element_path(oracle_mod):
    case = C.tet4_case(3, name="tet4_n3")
    tape = golden_tape("tet4_elastic")
    p = case.params
    t = case.conn[:5]
    ins = np.concatenate([case.x[t].reshape(5, 12), case.X[t].reshape(5, 12),
                          np.tile([p["mu"], p["lambda"]], (5, 1))], 1)
    out = oracle_mod.tape_eval(tape, ins, 157)
    ref = golden("tet4_n3")["elem_elastic"].reshape(-1, 157)[:5]
    np.testing.assert_array_equal(out, ref)


# ---- reference behavioural contracts restated on the oracle (test_solver.cpp) ------------

def two_tets(oracle_mod, perturb=0.05):
    """TwoTets rig: tets (0,1,2,3) and (0,1,2,4) sharing face (0,1,2)."""
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0.3, 0.3, -1.0]], float)
    rng = np.random.default_rng(1)
    x = X + rng.uniform(-perturb, perturb, X.shape)
    s = oracle_mod.System()
    xa = s.add_array("x", x, 3, True)
    ra = s.add_array("rest", X, 3)
    mu, lam = C.lame_from_young_poisson(1e5, 0.4)
    s.add_energy("elastic", np.array([[0, 1, 2, 3], [0, 2, 1, 4]]), 4, golden_tape("tet4_elastic"),
                 S.solid_tet_inputs(xa, ra), range(12), params={24: mu, 25: lam})
    return s


def test_two_tet_pattern(oracle_mod):
    """test_solver.cpp:126-143: 23 blocks, row 4 = {0,1,2,4}, no (3,4)."""
    r = two_tets(oracle_mod).assemble()
    assert r["b"] == 3 and r["row_ptr"].size == 6 and r["col_idx"].size == 23
    rp, ci = r["row_ptr"], r["col_idx"]
    assert list(ci[rp[4]:rp[5]]) == [0, 1, 2, 4]
    assert 4 not in ci[rp[3]:rp[4]]


def test_pins_contract(oracle_mod):
    """apply_pins: pinned g = 0, rows/cols zeroed, diagonal 1 (assembly.hpp:464-489)."""
    s = two_tets(oracle_mod)
    pins = np.zeros(15, np.uint8)
    pins[0:3] = 1
    pins[5] = 1
    r = s.assemble(pins=pins)
    from paper_2303_02156_b200.device import Bcrs
    D = Bcrs(3, r["row_ptr"], r["col_idx"], r["vals"]).to_dense()
    for i in np.flatnonzero(pins):
        assert r["grad"][i] == 0.0
        assert np.count_nonzero(D[i]) == 1 and D[i, i] == 1.0
        assert np.count_nonzero(D[:, i]) == 1
    assert np.allclose(D, D.T)


def test_non_finite_names_energy_and_element(oracle_mod):
    """test_solver.cpp:236-254: log of a negative coordinate fails at element 1."""
    # a collapsed rest tet (det(Dm) = 0) divides by zero -> non-finite outputs at element 1
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0, 0, 0], [0, 0, 0], [0, 0, 0], [0, 0, 0]], float)
    s2 = oracle_mod.System()
    xa = s2.add_array("x", X + 0.01, 3, True)
    ra = s2.add_array("rest", X, 3)
    mu, lam = C.lame_from_young_poisson(1e5, 0.4)
    s2.add_energy("elastic", np.array([[0, 1, 2, 3], [4, 5, 6, 7]]), 4, golden_tape("tet4_elastic"),
                  S.solid_tet_inputs(xa, ra), range(12), params={24: mu, 25: lam})
    r = s2.assemble()
    assert r["status"] == 4 and r["bad_energy"] == 0 and r["bad_element"] == 1
    assert np.isnan(s2.energy_only()) or not np.isfinite(s2.energy_only())


def test_spd_oracle_properties(oracle_mod):
    rng = np.random.default_rng(3)
    A = rng.normal(size=(50, 12, 12))
    H = A + np.swapaxes(A, 1, 2)
    P = oracle_mod.spd_project(H)
    w = np.linalg.eigvalsh(P)
    assert w.min() > -1e-12 * np.abs(w).max()
    np.testing.assert_allclose(oracle_mod.spd_project(P), P, atol=1e-12)
    B = A @ np.swapaxes(A, 1, 2)
    np.testing.assert_allclose(oracle_mod.spd_project(B), B, atol=1e-10)


@pytest.mark.parametrize("name", ["tet4_n3", "cloth_n8"])
def test_bcrs_dump_matches_reference_text(name):
    """Bcrs.dump() writes the reference's BcrsMatrix::dump text byte for byte (fixture written
    by the reference itself, oracle/make_dump_golden.py)."""
    import gzip
    import os
    from paper_2303_02156_b200.device import Bcrs
    g = golden(name)
    H = Bcrs(b=3, row_ptr=g["row_ptr"], col_idx=g["col_idx"], values=g["vals"])
    with gzip.open(os.path.join(os.path.dirname(__file__), "golden", name + "_dump.txt.gz"), "rt") as f:
        assert H.dump() == f.read()
