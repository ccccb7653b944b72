import gzip
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def golden_tape(name):
    """The reference's own tapes (Tape::save of the reference's kernels, oracle/make_golden.py),
    shipped with the package as the data the reference front end hands across the ABI."""
    with gzip.open(os.path.join(ROOT, "paper_2303_02156_b200", "tapes", name + ".sytp.gz"), "rb") as f:
        return f.read()


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle as O
    O.lib()
    return O
