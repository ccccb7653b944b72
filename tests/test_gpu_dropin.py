"""GPU: the drop-in boundary, in-process, against the UNMODIFIED reference.

oracle/_ref/ref_cuda_driver is compiled from the reference's own headers
(/root/reference/proj/include/symel, in place) plus include/symel_cuda_assembler.hpp and links
libsymel_cuda.so. For each case it builds one reference EnergySystem with the reference's
energy helpers, assembles it with the reference's CPU `symel::Assembler` and with
`symel::CudaAssembler` (device), and compares pattern (bit-exact), E, gradient and BCRS values
(1e-10, the reference's measure; ordered mode 1e-13) in the three device modes, then
energy_only, guard_min, active sets, pins, a topology change, the check_finite message and the
SPD projection. Every check prints one JSON line; all must pass."""
import json
import os
import subprocess
import tempfile

import pytest

from conftest import ROOT
from paper_2303_02156_b200 import configs as C

pytestmark = pytest.mark.gpu
DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_cuda_driver")

# (case, SPD projection, energies evaluated in the reference's rounding: the barrier at
# d ~ 1e-7 h loses ~6 digits computing d)
CASES = {
    "tet4": (lambda: C.config2(5), True, None),
    "tet10": (lambda: C.config3(2), False, None),
    "cloth": (lambda: C.config4(9), False, None),
    "contact": (lambda: C.config5(3, 40), True, "contact"),
}


@pytest.mark.parametrize("kind", sorted(CASES))
def test_reference_system_through_cuda_assembler(kind):
    assert os.path.exists(DRIVER), "built by oracle/Makefile (needs the reference headers at build time)"
    make, spd, exact = CASES[kind]
    with tempfile.TemporaryDirectory() as d:
        make().write_case_dir(d)
        args = [DRIVER, d] + (["--spd"] if spd else []) + (["--exact", exact] if exact else [])
        out = subprocess.run(args, capture_output=True, text=True, timeout=900)
    lines = [json.loads(s) for s in out.stdout.splitlines() if s.startswith("{")]
    failed = [c for c in lines if not c["ok"]]
    assert out.returncode == 0 and not failed and lines, out.stdout + out.stderr
    names = {c["check"] for c in lines}
    assert {"assemble_deterministic", "assemble_atomic", "assemble_ordered", "energy_only", "guard_min",
            "active_sets", "pins", "non_finite_message"} <= names
    if kind != "cloth":  # the membrane's per-element rest data pins its element count
        assert "topology_change" in names
    if spd:
        assert {"spd_energy_gradient", "spd_symmetric"} <= names
