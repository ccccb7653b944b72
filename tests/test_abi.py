"""CPU tests of the drop-in boundary: libsymel_cuda.so loads, exports every symbol declared in
include/symel_cuda.h, refuses to run without a device (no CPU fallback), and its code generator
emits kernels that NVRTC compiles for sm_100a (device-less codegen context)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_tape
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200 import device as D
from paper_2303_02156_b200.systems import DeviceSystem

HEADER = os.path.join(ROOT, "include", "symel_cuda.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(symel_cuda_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_what_the_binding_uses():
    assert set(declared_symbols()) == set(D.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(D.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.symel_cuda_abi_version() == 1


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = D.load_library()
    h = ctypes.c_void_p()
    assert lib.symel_cuda_create(0, ctypes.byref(h)) == D.E_NODEVICE
    with pytest.raises(D.SymelError):
        D.DeviceAssembler(0)


def test_invalid_tape_is_rejected():
    A = D.DeviceAssembler(-1)
    x = A.add_array("x", 4, 3, True)
    t = A.add_connectivity("tets", 4)
    A.set_elements(t, np.array([[0, 1, 2, 3]]))
    with pytest.raises(D.SymelError) as ei:
        A.add_energy("bad", t, b"SYTX" + b"\0" * 100, [(0, x, 0, 0)], [0])
    assert ei.value.code == D.E_TAPE


def test_binding_errors_match_reference_messages():
    A = D.DeviceAssembler(-1)
    x = A.add_array("x", 4, 3, True)
    with pytest.raises(D.SymelError, match="already registered"):
        A.add_array("x", 4, 3)
    t = A.add_connectivity("tets", 4)
    tape = golden_tape("tet4_elastic")
    from paper_2303_02156_b200.systems import solid_tet_inputs
    bad = solid_tet_inputs(x, x)
    bad[0] = (0, x, 7, 0)   # tuple slot outside arity
    with pytest.raises(D.SymelError, match="tuple slot 7 outside connectivity arity 4"):
        A.add_energy("e", t, tape, bad, range(12))


@pytest.mark.parametrize("mode", ["ordered", "deterministic", "atomic"])
def test_codegen_sources(mode):
    ds = DeviceSystem(C.tet4_case(2), tapes=golden_tape, device=-1)
    src = ds.asm.kernel_source(ds.energies["elastic"], mode)
    assert "__global__" in src and "__launch_bounds__" in src
    if mode == "atomic":  # the tile kernel's per-(tile, block) red.add branch
        assert "atomicAdd(o + q" in src and "a.tile_atomic" in src
    if mode == "deterministic":
        assert "a.partials" in src and "__syncthreads" in src
    body = src.split("__global__")[1]
    if mode == "ordered":
        assert "sy_rcp" not in body   # IEEE division in tape order
    else:
        assert "sy_rcp(" in body


def test_nvrtc_compiles_for_sm100a():
    """Every variant of a small energy compiles (NVRTC, sm_100a) without a GPU."""
    ds = DeviceSystem(C.config5(2, 4), tapes=golden_tape, device=-1)
    for eid in ds.energies.values():
        for mode in ("ordered", "deterministic", "atomic"):
            ds.asm.precompile(eid, mode)
