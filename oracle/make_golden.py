"""TEST INFRASTRUCTURE ONLY: regenerates tests/golden/ from the unmodified reference.

Runs oracle/_ref/ref_driver (reference headers compiled in place) on small seeded cases from
paper_2303_02156_b200/configs.py and stores its outputs as compressed fixtures, plus the
reference's own tapes. Requires /root/reference (this container); the GPU box only reads the
committed fixtures.

    python oracle/make_golden.py
"""
from __future__ import annotations

import gzip
import hashlib
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2303_02156_b200 import configs as C  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
TAPE_DIR = os.path.join(ROOT, "paper_2303_02156_b200", "tapes")  # the reference's own tapes, shipped with the package

# name -> case factory. Small enough to commit; the full configs are checked on the GPU
# against the C oracle (which these fixtures pin) and through size-independent properties.
CASES = {
    "tet4_n3": lambda: C.tet4_case(3, name="tet4_n3"),
    "tet4_c1": lambda: C.config1(20),
    "tet4_c2_n6": lambda: C.config2(6),
    "tet10_n2": lambda: C.config3(2),
    "cloth_n8": lambda: C.config4(8),
    "contact_n3": lambda: C.config5(3, 40),
}
TAPES = {"tet4_elastic": ("tet4_n3", "elastic"), "tet10_elastic": ("tet10_n2", "elastic"),
         "membrane": ("cloth_n8", "membrane"), "bending": ("cloth_n8", "bending"),
         "inertia": ("contact_n3", "inertia"), "contact": ("contact_n3", "contact"),
         "contact_act": ("contact_n3", "contact_act"), "contact_guard": ("contact_n3", "contact_guard")}


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main():
    os.makedirs(TAPE_DIR, exist_ok=True)
    work = tempfile.mkdtemp(prefix="symel_golden_")
    dirs = {}
    for name, make in CASES.items():
        case = make()
        d = os.path.join(work, name)
        case.write_case_dir(d)
        info = O.run_ref_driver(d, backend="interp", threads=4)
        ref = O.load_ref_outputs(d)
        fx = {"E": np.array([ref["E"]]), "grad": ref["grad"], "row_ptr": ref["row_ptr"], "col_idx": ref["col_idx"],
              "x_digest": np.array([digest(case.x)]), "X_digest": np.array([digest(case.X)]),
              "conn_digest": np.array([digest(case.conn)])}
        if ref["vals"].size <= 200_000:
            fx["vals"] = ref["vals"]
        else:  # config-1 size: keep a seeded sample of blocks + a checksum of all values
            rng = np.random.default_rng(7)
            b = 3
            nb = ref["col_idx"].size
            idx = np.sort(rng.choice(nb, 4000, replace=False))
            fx["vals_sample_blocks"] = idx
            fx["vals_sample"] = ref["vals"].reshape(nb, b * b)[idx]
            fx["vals_abs_sum"] = np.array([np.abs(ref["vals"]).sum()])
        for f in os.listdir(d):
            if f.startswith("ref_elem_"):
                fx["elem_" + f[len("ref_elem_"):-4]] = np.fromfile(os.path.join(d, f), np.float64)
        if case.kind == "cloth":
            fx["ref_flaps"] = np.fromfile(os.path.join(d, "ref_flaps.i64"), np.int64)
            fx["ref_dm2inv"] = np.fromfile(os.path.join(d, "ref_dm2inv.f64"), np.float64)
            fx["ref_area"] = np.fromfile(os.path.join(d, "ref_area.f64"), np.float64)
            fx["ref_Q"] = np.fromfile(os.path.join(d, "ref_Q.f64"), np.float64)
        with open(os.path.join(d, "ref_stats.txt")) as f:
            fx["stats"] = np.array([f.read()])
        np.savez_compressed(os.path.join(GOLDEN, name + ".npz"), **fx)
        dirs[name] = d
        print(name, info["E"], info["n_blocks"])
    for tname, (cname, ename) in TAPES.items():
        src = os.path.join(dirs[cname], "ref_tape_%s.sytp" % ename)
        with open(src, "rb") as f, gzip.GzipFile(os.path.join(TAPE_DIR, tname + ".sytp.gz"), "wb", mtime=0) as g:
            g.write(f.read())
    shutil.rmtree(work)


if __name__ == "__main__":
    main()
