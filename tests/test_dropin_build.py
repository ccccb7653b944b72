"""CPU: the reference-side adapter (include/symel_cuda_assembler.hpp) compiles against the
unmodified reference headers into oracle/_ref/ref_cuda_driver, and -- without a device -- the
device path refuses loudly instead of falling back to the CPU."""
import os
import subprocess

import pytest

from conftest import ROOT

DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_cuda_driver")


def test_driver_built_and_refuses_without_device(tmp_path):
    assert os.path.exists(DRIVER), "built by oracle/Makefile"
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2303_02156_b200 import configs as C
    C.config2(2).write_case_dir(str(tmp_path))
    out = subprocess.run([DRIVER, str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert out.returncode != 0
    assert "no CUDA device" in out.stdout + out.stderr
