"""Registers a synthetic Case (configs.py) on a DeviceAssembler with the reference's binding
layout: array registration order and input-slot order follow the reference's energy helpers
(energies.hpp:418-609) exactly, so a tape produced by the reference plugs in unchanged.

Tapes: the derivative / activation / guard kernels of the BASELINE energies as the reference's
own front end produces them (EnergySystem::compile_kernels -> Tape::save, registry.hpp:601-653,
tape.hpp:213-240), stored under paper_2303_02156_b200/tapes/ by oracle/make_golden.py. They are
the IR that crosses the C ABI; the C++ path (include/symel_cuda_assembler.hpp) hands the
reference's in-memory tapes over instead.

Input slots per energy (bind order, registry.hpp:577-594):
  solid_tet  (energies.hpp:435-461): x[a].c (12) | rest[a].c (12) | mu | lambda
  fem_solid  (energies.hpp:465-519): x[a].c (30) | rest[a].c (30) | mu | lambda | item.0..3
  membrane   (energies.hpp:523-543): x[a].c (9) | dm2inv[e].0..3 | area[e] | mu | lambda
  bending    (energies.hpp:594-609): x[a].c (12) | Q[e].0..143 | k_b
  inertia    (energies.hpp:418-430): x | x_prev | v | mass
  contact    (oracle/ref_driver.cpp, point-triangle barrier): x[a].c (12) | off[e].0..11 | k_c | d_hat
"""
from __future__ import annotations

import gzip
import os
from typing import Callable, Dict, Optional

import numpy as np

from . import configs
from .device import (DeviceAssembler, ENERGY_EXACT, ENERGY_SPD, IN_ELEM, IN_ITEM, IN_PARAM, IN_SUM)

_HERE = os.path.dirname(os.path.abspath(__file__))

# tet_rule_quadratic (energies.hpp:42-47)
_QA, _QB, _QW = 0.5854101966249685, 0.1381966011250105, 1.0 / 24.0
TET_RULE_QUADRATIC = np.array([[_QW, _QA, _QB, _QB], [_QW, _QB, _QA, _QB], [_QW, _QB, _QB, _QA],
                               [_QW, _QB, _QB, _QB]])


def _item(arr, nodes, comps=3):
    return [(IN_ITEM, arr, a, c) for a in range(nodes) for c in range(comps)]


def _elem(arr, comps):
    return [(IN_ELEM, arr, 0, c) for c in range(comps)]


def solid_tet_inputs(x, rest):
    return _item(x, 4) + _item(rest, 4) + [(IN_PARAM, 0, 0, 0)] * 2


def fem_solid_inputs(x, rest, nodes=10):
    return _item(x, nodes) + _item(rest, nodes) + [(IN_PARAM, 0, 0, 0)] * 2 + [(IN_SUM, 0, k, 0) for k in range(4)]


def membrane_inputs(x, dm, area):
    return _item(x, 3) + _elem(dm, 4) + _elem(area, 1) + [(IN_PARAM, 0, 0, 0)] * 2


def bending_inputs(x, Q):
    return _item(x, 4) + _elem(Q, 144) + [(IN_PARAM, 0, 0, 0)]


def inertia_inputs(x, xp, v, m):
    return _item(x, 1) + _item(xp, 1) + _item(v, 1) + [(IN_ITEM, m, 0, 0)]


def contact_inputs(x, off):
    return _item(x, 4) + _elem(off, 12) + [(IN_PARAM, 0, 0, 0)] * 2


TapeProvider = Callable[[str], bytes]


def reference_tape(name: str) -> bytes:
    """A tape produced by the reference's front end (see the module docstring)."""
    path = os.path.join(_HERE, "tapes", name + ".sytp.gz")
    with gzip.open(path, "rb") as f:
        return f.read()


golden_tape = reference_tape


def default_tapes() -> TapeProvider:
    return reference_tape


class DeviceSystem:
    """A Case registered on the device; keeps array ids for updates."""

    def __init__(self, case: configs.Case, tapes: Optional[TapeProvider] = None, spd: bool = False,
                 device: int = 0, Q: Optional[np.ndarray] = None, n_own: Optional[int] = None):
        """n_own (tet4 only): the first n_own tets are owned, the rest are ghosts of a sharded
        run (parallel.py): they are registered as a second energy "elastic_ghost" so the owned
        energy is its own part (energy_parts) while the ghosts complete the owned block rows."""
        tapes = tapes or default_tapes()
        self.case = case
        A = self.asm = DeviceAssembler(device)
        n = case.n_nodes
        self.x = A.add_array("x", n, 3, True)
        self.rest = A.add_array("rest", n, 3)
        A.set_array(self.x, case.x)
        A.set_array(self.rest, case.X)
        p = case.params
        self.energies: Dict[str, int] = {}
        self.arrays: Dict[str, int] = {"x": self.x, "rest": self.rest}
        flags = ENERGY_SPD if spd else 0
        if case.kind in ("tet4", "contact"):
            own = case.conn if n_own is None else case.conn[:n_own]
            t = A.add_connectivity("tets", 4)
            A.set_elements(t, own)
            self.energies["elastic"] = A.add_energy("elastic", t, tapes("tet4_elastic"), solid_tet_inputs(self.x, self.rest),
                                                    range(12), params={24: p["mu"], 25: p["lambda"]}, flags=flags)
            if n_own is not None and n_own < case.conn.shape[0]:
                tg = A.add_connectivity("ghost_tets", 4)
                A.set_elements(tg, case.conn[n_own:])
                self.energies["elastic_ghost"] = A.add_energy(
                    "elastic_ghost", tg, tapes("tet4_elastic"), solid_tet_inputs(self.x, self.rest), range(12),
                    params={24: p["mu"], 25: p["lambda"]}, flags=flags)
        elif case.kind == "tet10":
            t = A.add_connectivity("tets", 10)
            A.set_elements(t, case.conn)
            self.energies["elastic"] = A.add_energy("elastic", t, tapes("tet10_elastic"), fem_solid_inputs(self.x, self.rest),
                                                    range(30), sum_items=TET_RULE_QUADRATIC,
                                                    params={60: p["mu"], 61: p["lambda"]}, flags=flags)
        elif case.kind == "cloth":
            ne = case.conn.shape[0]
            nf = case.extra["flaps"].shape[0]
            dm = A.add_array("dm2inv", ne, 4)
            ar = A.add_array("area", ne, 1)
            A.set_array(dm, case.extra["dm2inv"])
            A.set_array(ar, case.extra["area"])
            tc = A.add_connectivity("tris", 3)
            A.set_elements(tc, case.conn)
            self.energies["membrane"] = A.add_energy("membrane", tc, tapes("membrane"), membrane_inputs(self.x, dm, ar),
                                                     range(9), params={14: p["mu"], 15: p["lambda"]}, flags=flags)
            fc = A.add_connectivity("flaps", 4)
            A.set_elements(fc, case.extra["flaps"])
            q = self.arrays["Q"] = A.add_array("Q", nf, 144)
            A.set_array(q, Q if Q is not None else configs.bending_Q_for(case))
            self.energies["bending"] = A.add_energy("bending", fc, tapes("bending"), bending_inputs(self.x, q),
                                                    range(12), params={156: p["kb"]}, flags=flags)
        if case.kind == "contact":
            ex = case.extra
            xp = A.add_array("x_prev", n, 3)
            v = A.add_array("v", n, 3)
            m = A.add_array("mass", n, 1)
            A.set_array(xp, ex["x_prev"])
            A.set_array(v, ex["v"])
            A.set_array(m, ex["mass"])
            vc = A.add_connectivity("verts", 1)
            A.set_elements(vc, np.arange(n, dtype=np.int64))
            self.energies["inertia"] = A.add_energy("inertia", vc, tapes("inertia"), inertia_inputs(self.x, xp, v, m),
                                                    range(3))
            npairs = ex["pairs"].shape[0]
            off = self.arrays["pair_offset"] = A.add_array("pair_offset", npairs, 12)
            A.set_array(off, ex["offsets"])
            pc = A.add_connectivity("pairs", 4)
            A.set_elements(pc, ex["pairs"])
            self.energies["contact"] = A.add_energy(
                "contact", pc, tapes("contact"), contact_inputs(self.x, off), range(12),
                act_tape=tapes("contact_act"), act_kind=0, guard_tape=tapes("contact_guard"),
                params={24: p["kappa"], 25: p["dhat"]}, flags=flags | ENERGY_EXACT)

    def n_elements(self) -> int:
        return sum(self.asm.active_count(e) for e in self.energies.values())
