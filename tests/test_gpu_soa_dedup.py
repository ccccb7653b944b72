"""GPU: component-row deduplication of wide per-element arrays (the tile kernels' SoA copies).

The reference's bending Q (energies.hpp:684-745) is a 4 x 4 stencil repeated per coordinate:
96 of its 144 components are +0.0 in every flap and the rest repeat 16 values. The device path
keeps one SoA row per distinct non-zero component and reads each once; that must not change a
single output bit, and a later set_array with unstructured data must rebuild kernels and copies."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import golden_tape
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200.systems import DeviceSystem

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SNIPPET = """
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + "/tests")
from conftest import golden_tape
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200.systems import DeviceSystem
ds = DeviceSystem(C.config4(24), tapes=golden_tape)
out = {{}}
for mode in ("deterministic", "atomic"):
    E = ds.asm.assemble(mode)
    out["E_" + mode] = np.float64(E)
    out["g_" + mode] = ds.asm.gradient()
    if mode == "deterministic":
        out["H"] = ds.asm.hessian().values
src = ds.asm.kernel_source(ds.energies["bending"], "deterministic")
out["loads"] = np.int64(src.count("a.soa_n + t)"))
np.savez({path!r}, **out)
"""


def _run(tmp_path, name, env_extra):
    path = str(tmp_path / (name + ".npz"))
    env = dict(os.environ, **env_extra)
    subprocess.run([sys.executable, "-c", _SNIPPET.format(root=ROOT, path=path)], check=True, env=env, timeout=600)
    return np.load(path)


def test_dedup_is_bitwise_neutral(tmp_path):
    a = _run(tmp_path, "dedup", {})
    b = _run(tmp_path, "plain", {"SYMEL_NO_SOA_DEDUP": "1"})
    # the structured Q needs at most 16 row loads (the regular grid repeats some of those too)
    # next to the 4 of the tile-ordered connectivity; the plain copy needs all 144
    assert int(b["loads"]) == 4 + 144 and int(a["loads"]) <= 4 + 16, (int(a["loads"]), int(b["loads"]))
    for k in ("E_deterministic", "g_deterministic", "H"):  # fixed-order mode: every bit
        assert np.array_equal(a[k].view(np.uint64), b[k].view(np.uint64)), k
    assert abs(a["E_atomic"] - b["E_atomic"]) <= 1e-13 * abs(b["E_atomic"])
    assert np.allclose(a["g_atomic"], b["g_atomic"], rtol=0, atol=1e-13 * np.abs(b["g_atomic"]).max())


def test_unstructured_data_after_structured(oracle_mod):
    """set_array with dense, duplicate-free Q on a live context: classes are recomputed, the
    bending kernel and its SoA copy rebuilt; the result follows the new data."""
    case = C.config4(10)
    ds = DeviceSystem(case, tapes=golden_tape)
    ds.asm.assemble("deterministic")
    rng = np.random.default_rng(7)
    nf = case.extra["flaps"].shape[0]
    Q = rng.normal(size=(nf, 144)) * 1e-3  # dense blocks: no zeros, no repeated components
    ds.asm.set_array(ds.arrays["Q"], Q)
    sysm = oracle_mod.system_for_case(case, golden_tape)
    qi = next(i for i, a in enumerate(sysm.arrays) if a["name"] == "Q")
    sysm.arrays[qi]["data"] = np.ascontiguousarray(Q).ravel()
    ref = sysm.assemble()
    for mode in ("deterministic", "atomic"):
        E = ds.asm.assemble(mode)
        assert abs(E - ref["E"]) <= 1e-10 * max(1.0, abs(ref["E"]))
        assert oracle_mod.rel_err(ds.asm.gradient(), ref["grad"]) <= 1e-10
        assert oracle_mod.rel_err(ds.asm.hessian().values, ref["vals"]) <= 1e-10
    src = ds.asm.kernel_source(ds.energies["bending"], "deterministic")
    assert src.count("a.soa_n + t)") == 4 + 144

