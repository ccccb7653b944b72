"""CPU: the solver oracle (symel_oracle.c: BcrsMatrix::matvec, block_jacobi_inverse, pcg) pinned
bit for bit to the unmodified reference's outputs (tests/golden/solver_*.npz, made by
oracle/make_golden_solver.py from oracle/_ref/ref_driver --solver)."""
import glob
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "solver_*.npz")))


@pytest.fixture(params=GOLD, ids=[os.path.basename(g)[7:-4] for g in GOLD])
def fx(request):
    return dict(np.load(request.param))


def test_matvec_bitwise(fx):
    y = O.bsr_matvec(3, fx["row_ptr"], fx["col_idx"], fx["vals"], fx["probe"])
    assert np.array_equal(y, fx["matvec"])


def test_block_jacobi_bitwise(fx):
    for t, tau in enumerate(fx["taus"]):
        inv = O.block_jacobi_inverse(3, fx["row_ptr"], fx["col_idx"], fx["vals"], tau)
        assert np.array_equal(inv, fx["bjinv_%d" % t])


def test_pcg_bitwise(fx):
    n = fx["grad"].size
    for k, tag in enumerate(fx["pcg_tags"]):
        t, kind = str(tag).split("_")
        x, st = O.pcg(3, fx["row_ptr"], fx["col_idx"], fx["vals"], fx["taus"][int(t)], -fx["grad"],
                      1e-4 if kind == "loose" else 1e-10, n)
        it, cv, nc = fx["pcg_stats"][k]
        assert (st["iters"], st["converged"], st["neg_curvature"]) == (it, bool(cv), bool(nc)), tag
        assert st["rel_residual"] == fx["pcg_rel_residual"][k]
        assert np.array_equal(x, fx["pcg_x_" + str(tag)])
