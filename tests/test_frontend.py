"""CPU: the repo's own C++ symbolic front end (csrc/host/symel) reproduces the reference's tapes
byte for byte -- DAG, CSE plan, register layout, constants and the SHA-256 kernel key."""
import pytest

from conftest import golden_tape
from paper_2303_02156_b200 import frontend

NAMES = ["tet4_elastic", "tet10_elastic", "membrane", "bending", "inertia", "contact", "contact_act", "contact_guard"]


@pytest.mark.parametrize("name", NAMES)
def test_tapes_are_byte_identical_to_reference(name):
    assert frontend.tape(name) == golden_tape(name)


def test_unknown_energy_errors():
    with pytest.raises(RuntimeError, match="unknown standard energy"):
        frontend.tape("nope")
