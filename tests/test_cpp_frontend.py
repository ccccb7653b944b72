"""CPU: the C++ front end and device Assembler header compile, and the example fails loudly
(no CPU fallback) without a device."""
import os
import subprocess

import pytest

from conftest import ROOT


def test_example_builds_and_refuses_without_device():
    exe = os.path.join(ROOT, "examples", "assemble_tet")
    assert os.path.exists(exe), "built by __graft_entry__.build()"
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    out = subprocess.run([exe, "2"], capture_output=True, text=True, timeout=120)
    assert out.returncode != 0
    assert "no CUDA device" in out.stderr
