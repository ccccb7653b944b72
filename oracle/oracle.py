"""TEST INFRASTRUCTURE ONLY: ctypes front of the C oracle (symel_oracle.c) plus the numpy SPD
projection oracle. Imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
leg only -- never by the product package.

The SPD projection has no reference implementation (the reference regularises with H + tau I,
/root/reference/proj/include/symel/optimizer.hpp:196-221; projection is listed as future
work): its oracle is numpy.linalg.eigh (LAPACK dsyevd) on the element
Hessian, eigenvalues clamped at 0 -- "parity unpinned" by the reference.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REF_DRIVER = os.path.join(HERE, "_ref", "ref_driver")


class OInput(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("array", C.c_uint32), ("tuple_slot", C.c_uint32), ("comp", C.c_uint32)]


class OArray(C.Structure):
    _fields_ = [("data", C.c_void_p), ("items", C.c_uint64), ("comps", C.c_uint32), ("is_dof", C.c_int32)]


class OEnergy(C.Structure):
    _fields_ = [("tape", C.c_void_p), ("tape_len", C.c_uint64), ("act_tape", C.c_void_p), ("act_len", C.c_uint64),
                ("act_kind", C.c_int32), ("guard_tape", C.c_void_p), ("guard_len", C.c_uint64),
                ("inputs", C.c_void_p), ("n_inputs", C.c_uint32), ("dof_slots", C.c_void_p), ("n_dofs", C.c_uint32),
                ("conn", C.c_void_p), ("arity", C.c_uint32), ("n_elems", C.c_uint64), ("sum_items", C.c_void_p),
                ("n_items", C.c_uint32), ("sum_arity", C.c_uint32), ("is_sum", C.c_int32), ("params", C.c_void_p)]


class OResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("bad_energy", C.c_int32), ("bad_element", C.c_int64), ("E", C.c_double),
                ("b", C.c_int32), ("n_rows", C.c_int64), ("n_blocks", C.c_int64), ("n_dofs", C.c_int64),
                ("row_ptr", C.POINTER(C.c_int64)), ("col_idx", C.POINTER(C.c_int64)), ("vals", C.POINTER(C.c_double)),
                ("grad", C.POINTER(C.c_double)), ("active", C.POINTER(C.c_uint8))]


_lib = None


def build() -> None:
    """Compiles liboracle.so (and, when /root/reference is present, _ref/ref_driver)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = C.CDLL(LIB)
        _lib.oracle_tape_eval.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int64]
        _lib.oracle_assemble.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p, C.c_int32,
                                         C.POINTER(OResult)]
        _lib.oracle_element_outputs.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]
        _lib.oracle_energy_only.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p,
                                            C.POINTER(C.c_double)]
        _lib.oracle_guard_min.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.POINTER(C.c_double)]
        _lib.oracle_free_result.argtypes = [C.POINTER(OResult)]
        _lib.oracle_energy_gradient.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.c_int32,
                                                C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p,
                                                C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
        _lib.oracle_bsr_matvec.argtypes = [C.c_int32, C.c_int64] + [C.c_void_p] * 5
        _lib.oracle_block_jacobi_inverse.argtypes = [C.c_int32, C.c_int64] + [C.c_void_p] * 3 + [C.c_double, C.c_void_p]
        _lib.oracle_pcg.argtypes = ([C.c_int32, C.c_int64] + [C.c_void_p] * 3 + [C.c_double, C.c_void_p, C.c_void_p,
                                    C.c_double, C.c_int32] + [C.POINTER(C.c_int32)] * 3 + [C.POINTER(C.c_double)])
    return _lib


class System:
    """Plain description of an energy system, mirroring EnergySystem registration."""

    def __init__(self):
        self.arrays: List[dict] = []
        self.energies: List[dict] = []
        self._keep = []

    def add_array(self, name, data, comps, is_dof=False):
        d = np.ascontiguousarray(data, dtype=np.float64).ravel()
        self.arrays.append({"name": name, "data": d, "items": d.size // comps, "comps": comps, "is_dof": is_dof})
        return len(self.arrays) - 1

    def add_energy(self, name, conn, arity, tape, inputs, dof_slots, params=None, sum_items=None,
                   act_tape=None, act_kind=0, guard_tape=None, is_sum=None):
        c = np.ascontiguousarray(conn, dtype=np.int64).ravel()
        p = np.zeros(len(inputs))
        for k, v in (params or {}).items():
            p[k] = v
        self.energies.append(dict(name=name, conn=c, arity=arity, tape=tape, inputs=list(inputs),
                                  dof_slots=np.asarray(list(dof_slots), np.uint32), params=p, sum_items=sum_items,
                                  act_tape=act_tape, act_kind=act_kind, guard_tape=guard_tape,
                                  is_sum=(sum_items is not None) if is_sum is None else is_sum))
        return len(self.energies) - 1

    def _structs(self):
        keep = []
        arrs = (OArray * max(1, len(self.arrays)))()
        for i, a in enumerate(self.arrays):
            arrs[i] = OArray(a["data"].ctypes.data, a["items"], a["comps"], int(a["is_dof"]))
        ens = (OEnergy * max(1, len(self.energies)))()
        for i, e in enumerate(self.energies):
            ins = (OInput * len(e["inputs"]))(*[OInput(*x) for x in e["inputs"]])
            tb = C.create_string_buffer(e["tape"], len(e["tape"]))
            ab = C.create_string_buffer(e["act_tape"], len(e["act_tape"])) if e["act_tape"] else None
            gb = C.create_string_buffer(e["guard_tape"], len(e["guard_tape"])) if e["guard_tape"] else None
            si = np.ascontiguousarray(e["sum_items"], dtype=np.float64) if e["sum_items"] is not None else None
            keep += [ins, tb, ab, gb, si]
            ens[i] = OEnergy(C.cast(tb, C.c_void_p), len(e["tape"]), C.cast(ab, C.c_void_p) if ab else None,
                             len(e["act_tape"]) if ab else 0, e["act_kind"], C.cast(gb, C.c_void_p) if gb else None,
                             len(e["guard_tape"]) if gb else 0, C.cast(ins, C.c_void_p), len(e["inputs"]),
                             e["dof_slots"].ctypes.data, e["dof_slots"].size, e["conn"].ctypes.data, e["arity"],
                             e["conn"].size // e["arity"], si.ctypes.data if si is not None else None,
                             si.shape[0] if si is not None else 0, si.shape[1] if si is not None else 0,
                             int(e["is_sum"]), e["params"].ctypes.data)
        return arrs, ens, keep

    def assemble(self, pins: Optional[np.ndarray] = None, threads: int = 0) -> dict:
        arrs, ens, keep = self._structs()
        r = OResult()
        pm = np.ascontiguousarray(pins, dtype=np.uint8) if pins is not None else None
        threads = threads or (os.cpu_count() or 1)
        lib().oracle_assemble(arrs, len(self.arrays), ens, len(self.energies),
                              pm.ctypes.data if pm is not None else None, threads, C.byref(r))
        try:
            out = dict(status=r.status, bad_energy=r.bad_energy, bad_element=r.bad_element, E=r.E, b=r.b)
            if r.status in (0, 4):
                out["row_ptr"] = np.ctypeslib.as_array(r.row_ptr, (r.n_rows + 1,)).copy()
                out["col_idx"] = np.ctypeslib.as_array(r.col_idx, (max(1, r.n_blocks),))[:r.n_blocks].copy()
                out["vals"] = np.ctypeslib.as_array(r.vals, (max(1, r.n_blocks * r.b * r.b),))[:r.n_blocks * r.b * r.b].copy()
                out["grad"] = np.ctypeslib.as_array(r.grad, (max(1, r.n_dofs),))[:r.n_dofs].copy()
                ntot = sum(e["conn"].size // e["arity"] for e in self.energies)
                out["active"] = np.ctypeslib.as_array(r.active, (max(1, ntot),))[:ntot].copy()
        finally:
            lib().oracle_free_result(C.byref(r))
        return out

    def energy_gradient(self, threads: int = 0) -> dict:
        """E (reference order and Kahan) and the gradient without the Hessian: full-size checks."""
        arrs, ens, keep = self._structs()
        n_dofs = sum(a["items"] * a["comps"] for a in self.arrays if a["is_dof"])
        g = np.empty(max(1, n_dofs))
        E, Ek = C.c_double(), C.c_double()
        be, bel = C.c_int32(), C.c_int64()
        threads = threads or (os.cpu_count() or 1)
        st = lib().oracle_energy_gradient(arrs, len(self.arrays), ens, len(self.energies), threads, C.byref(E),
                                          C.byref(Ek), g.ctypes.data, C.byref(be), C.byref(bel))
        return dict(status=st, E=E.value, E_kahan=Ek.value, grad=g[:n_dofs], bad_energy=be.value,
                    bad_element=bel.value)

    def element_outputs(self, energy: int, first: int, count: int) -> np.ndarray:
        arrs, ens, keep = self._structs()
        e = self.energies[energy]
        nd = len(e["dof_slots"])
        S = 1 + nd + nd * nd
        out = np.empty(count * S)
        rc = lib().oracle_element_outputs(arrs, len(self.arrays), C.byref(ens[energy]), first, count, out.ctypes.data)
        assert rc == 0
        return out.reshape(count, S)

    def energy_only(self, active: Optional[np.ndarray] = None) -> float:
        arrs, ens, keep = self._structs()
        E = C.c_double()
        am = np.ascontiguousarray(active, dtype=np.uint8) if active is not None else None
        lib().oracle_energy_only(arrs, len(self.arrays), ens, len(self.energies),
                                 am.ctypes.data if am is not None else None, C.byref(E))
        return E.value

    def guard_min(self) -> float:
        arrs, ens, keep = self._structs()
        g = C.c_double()
        lib().oracle_guard_min(arrs, len(self.arrays), ens, len(self.energies), C.byref(g))
        return g.value


def tape_eval(tape: bytes, inputs: np.ndarray, n_out: int) -> np.ndarray:
    """inputs [W, n_in] -> outputs [W, n_out] through the C tape interpreter."""
    W = inputs.shape[0]
    ins = np.ascontiguousarray(inputs.T, dtype=np.float64)
    out = np.empty((n_out, W))
    tb = C.create_string_buffer(tape, len(tape))
    rc = lib().oracle_tape_eval(C.cast(tb, C.c_void_p), len(tape), ins.ctypes.data, out.ctypes.data, W)
    assert rc == 0, "bad tape"
    return out.T.copy()


def system_for_case(case, tapes) -> System:
    """Same registration as paper_2303_02156_b200.systems.DeviceSystem (and ref_driver.cpp)."""
    from paper_2303_02156_b200 import configs, systems as S
    sysm = System()
    p = case.params
    x = sysm.add_array("x", case.x, 3, True)
    rest = sysm.add_array("rest", case.X, 3)
    if case.kind in ("tet4", "contact"):
        sysm.add_energy("elastic", case.conn, 4, tapes("tet4_elastic"), S.solid_tet_inputs(x, rest), range(12),
                        params={24: p["mu"], 25: p["lambda"]})
    elif case.kind == "tet10":
        sysm.add_energy("elastic", case.conn, 10, tapes("tet10_elastic"), S.fem_solid_inputs(x, rest), range(30),
                        params={60: p["mu"], 61: p["lambda"]}, sum_items=S.TET_RULE_QUADRATIC)
    elif case.kind == "cloth":
        dm = sysm.add_array("dm2inv", case.extra["dm2inv"], 4)
        ar = sysm.add_array("area", case.extra["area"], 1)
        sysm.add_energy("membrane", case.conn, 3, tapes("membrane"), S.membrane_inputs(x, dm, ar), range(9),
                        params={14: p["mu"], 15: p["lambda"]})
        q = sysm.add_array("Q", configs.bending_Q_for(case), 144)
        sysm.add_energy("bending", case.extra["flaps"], 4, tapes("bending"), S.bending_inputs(x, q), range(12),
                        params={156: p["kb"]})
    if case.kind == "contact":
        ex = case.extra
        xp = sysm.add_array("x_prev", ex["x_prev"], 3)
        v = sysm.add_array("v", ex["v"], 3)
        m = sysm.add_array("mass", ex["mass"], 1)
        sysm.add_energy("inertia", np.arange(case.n_nodes), 1, tapes("inertia"), S.inertia_inputs(x, xp, v, m), range(3))
        off = sysm.add_array("pair_offset", ex["offsets"], 12)
        sysm.add_energy("contact", ex["pairs"], 4, tapes("contact"), S.contact_inputs(x, off), range(12),
                        params={24: p["kappa"], 25: p["dhat"]}, act_tape=tapes("contact_act"), act_kind=0,
                        guard_tape=tapes("contact_guard"))
    return sysm


# ------------------------------------------------------------------------- SPD projection

def spd_project(H: np.ndarray) -> np.ndarray:
    """Per-element projection of symmetric matrices [..., n, n]: V max(L, 0) V^T (float64 eigh)."""
    Hs = 0.5 * (H + np.swapaxes(H, -1, -2))
    w, V = np.linalg.eigh(Hs)
    return (V * np.maximum(w, 0.0)[..., None, :]) @ np.swapaxes(V, -1, -2)


def assemble_spd(sysm: "System", spd_energies=None) -> dict:
    """Oracle assembly with per-element SPD projection of the element Hessians of the listed
    energies (default: all but inertia-like energies with n_dofs == 3 are projected too; the
    projection of an SPD matrix is itself). E and g are unchanged by the projection; the BSR
    values are re-accumulated from projected element blocks in (energy, element) order."""
    base = sysm.assemble()
    b = base["b"]
    rp, ci = base["row_ptr"], base["col_idx"]
    vals = np.zeros_like(base["vals"]).reshape(-1, b, b)
    off = 0
    layout_off = {}
    o = 0
    for i, a in enumerate(sysm.arrays):
        if a["is_dof"]:
            layout_off[i] = o
            o += a["items"] * a["comps"]
    for ei, e in enumerate(sysm.energies):
        n_el = e["conn"].size // e["arity"]
        act = base["active"][off:off + n_el].astype(bool)
        off += n_el
        idx = np.flatnonzero(act)
        if idx.size == 0:
            continue
        nd = len(e["dof_slots"])
        out = sysm.element_outputs(ei, 0, n_el)[idx]
        H = out[:, 1 + nd:].reshape(-1, nd, nd)
        if spd_energies is None or e["name"] in spd_energies:
            H = spd_project(H)
        conn = e["conn"].reshape(n_el, e["arity"])[idx]
        dofs = np.zeros((idx.size, nd), np.int64)
        for k, s in enumerate(e["dof_slots"]):
            src = e["inputs"][s]
            arr = sysm.arrays[src[1]]
            dofs[:, k] = layout_off[src[1]] + conn[:, src[2]] * arr["comps"] + src[3]
        br = dofs // b
        # block index lookup per (row, col)
        for k in range(nd):
            for l in range(nd):
                r, c = br[:, k], br[:, l]
                blk = np.array([rp[rr] + np.searchsorted(ci[rp[rr]:rp[rr + 1]], cc) for rr, cc in zip(r, c)])
                np.add.at(vals, (blk, dofs[:, k] % b, dofs[:, l] % b), H[:, k, l])
    res = dict(base)
    res["vals"] = vals.ravel()
    return res


def run_ref_driver(case_dir: str, backend: str = "source", threads: int = 0, lanes: int = 8, repeat: int = 1,
                   dump: bool = True, cache: str = "/tmp/symel_ref_cache", timeout: float = 3600,
                   warmup: int = 1) -> dict:
    """Runs the unmodified reference (oracle/_ref/ref_driver) on a case directory."""
    import json
    cmd = [REF_DRIVER, case_dir, "--backend", backend, "--lanes", str(lanes), "--repeat", str(repeat),
           "--cache", cache, "--warmup", str(max(1, warmup))]
    if threads:
        cmd += ["--threads", str(threads)]
    if not dump:
        cmd.append("--no-dump")
    out = subprocess.run(cmd, check=True, capture_output=True, text=True, timeout=timeout)
    return json.loads(out.stdout.strip().splitlines()[-1])


def load_ref_outputs(case_dir: str) -> Dict[str, np.ndarray]:
    f = lambda n, dt: np.fromfile(os.path.join(case_dir, n), dtype=dt)
    return {"E": f("ref_E.f64", np.float64)[0], "grad": f("ref_g.f64", np.float64),
            "row_ptr": f("ref_rowptr.i64", np.int64), "col_idx": f("ref_colidx.i64", np.int64),
            "vals": f("ref_vals.f64", np.float64)}


def rel_err(a: np.ndarray, ref: np.ndarray) -> float:
    """The reference's tolerance measure (acceptance_main.cpp:101-106): max|a-ref| / max(1, |ref|_inf)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - ref)) / max(1.0, float(np.max(np.abs(ref)))))


# ---- consumer of the assembled BCRS: restated in symel_oracle.c ----------

def _bsr_args(b, row_ptr, col_idx, vals):
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int64)
    v = np.ascontiguousarray(vals, dtype=np.float64)
    return rp, ci, v, rp.size - 1


def bsr_matvec(b: int, row_ptr, col_idx, vals, x) -> np.ndarray:
    """BcrsMatrix::matvec (assembly.hpp:43-57), bitwise."""
    rp, ci, v, nr = _bsr_args(b, row_ptr, col_idx, vals)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(nr * b)
    assert lib().oracle_bsr_matvec(b, nr, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, x.ctypes.data,
                                   y.ctypes.data) == 0
    return y


def block_jacobi_inverse(b: int, row_ptr, col_idx, vals, tau: float) -> np.ndarray:
    """detail::block_jacobi_inverse (optimizer.hpp:52-90), bitwise."""
    rp, ci, v, nr = _bsr_args(b, row_ptr, col_idx, vals)
    inv = np.empty(nr * b * b)
    assert lib().oracle_block_jacobi_inverse(b, nr, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, float(tau),
                                             inv.ctypes.data) == 0
    return inv


def pcg(b: int, row_ptr, col_idx, vals, tau: float, rhs, rel_tol: float, max_iters: int):
    """pcg (optimizer.hpp:119-158), bitwise; returns (x, dict(iters, converged, neg_curvature, rel_residual))."""
    rp, ci, v, nr = _bsr_args(b, row_ptr, col_idx, vals)
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    x = np.empty(nr * b)
    it, cv, nc = C.c_int32(), C.c_int32(), C.c_int32()
    rr = C.c_double()
    assert lib().oracle_pcg(b, nr, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, float(tau), rhs.ctypes.data,
                            x.ctypes.data, float(rel_tol), int(max_iters), C.byref(it), C.byref(cv), C.byref(nc),
                            C.byref(rr)) == 0
    return x, {"iters": it.value, "converged": bool(cv.value), "neg_curvature": bool(nc.value),
               "rel_residual": rr.value}
