"""TEST INFRASTRUCTURE ONLY: solver fixtures from the unmodified reference.

Runs oracle/_ref/ref_driver --solver on small seeded cases: the reference's BcrsMatrix::matvec
on a probe vector, detail::block_jacobi_inverse and pcg (rhs = -g, three shifts tau, loose
1e-4 and tight 1e-10 tolerances) on its own assembled Hessian; stores them with the matrix as
tests/golden/solver_<case>.npz. Requires /root/reference (this container only).

    python oracle/make_golden_solver.py
"""
from __future__ import annotations

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
CASES = {
    "tet4_c2_n6": lambda: C.config2(6),
    "tet4_n3": lambda: C.tet4_case(3, name="tet4_n3"),
    "cloth_n8": lambda: C.config4(8),
}


def main():
    import subprocess
    work = tempfile.mkdtemp(prefix="symel_golden_solver_")
    for name, make in CASES.items():
        case = make()
        d = os.path.join(work, name)
        case.write_case_dir(d)
        subprocess.run([O.REF_DRIVER, d, "--backend", "interp", "--threads", "1", "--solver"], check=True,
                       capture_output=True)
        ref = O.load_ref_outputs(d)
        f = lambda n: np.fromfile(os.path.join(d, n), np.float64)
        fx = {"row_ptr": ref["row_ptr"], "col_idx": ref["col_idx"], "vals": ref["vals"], "grad": ref["grad"],
              "probe": f("ref_probe.f64"), "matvec": f("ref_matvec.f64"), "taus": f("ref_pcg_taus.f64")}
        rows = []
        with open(os.path.join(d, "ref_pcg.txt")) as fh:
            for line in fh:
                tag, it, cv, nc, rr = line.split()
                rows.append((tag, int(it), int(cv), int(nc), float(rr)))
                fx["pcg_x_" + tag] = f("ref_pcg_x_%s.f64" % tag)
        fx["pcg_tags"] = np.array([r[0] for r in rows])
        fx["pcg_stats"] = np.array([[r[1], r[2], r[3]] for r in rows], dtype=np.int64)
        fx["pcg_rel_residual"] = np.array([r[4] for r in rows])
        for t in range(3):
            fx["bjinv_%d" % t] = f("ref_bjinv_%d.f64" % t)
        np.savez_compressed(os.path.join(GOLDEN, "solver_" + name + ".npz"), **fx)
        print(name, [(r[0], r[1], r[2], r[3]) for r in rows])
    shutil.rmtree(work)


if __name__ == "__main__":
    main()
