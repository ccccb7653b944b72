"""GPU: the C++ front end + device Assembler (csrc/host/symel/assembler.hpp) -- the reference's
user flow (declare energy, bind, assemble) -- runs end to end on the device path."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_example_assembles_on_device():
    exe = os.path.join(ROOT, "examples", "assemble_tet")
    assert os.path.exists(exe), "built by __graft_entry__.build()"
    out = subprocess.run([exe, "6"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "blocks" in out.stdout
