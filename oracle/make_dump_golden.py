"""TEST INFRASTRUCTURE ONLY: the reference's BcrsMatrix::dump text (assembly.hpp:60-74) of two
small golden cases, written by oracle/_ref/ref_driver (reference headers compiled in place) to
tests/golden/<case>_dump.txt.gz. Requires /root/reference (this container).

    python oracle/make_dump_golden.py
"""
import gzip
import os
import shutil
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from oracle.make_golden import CASES, GOLDEN  # noqa: E402

if __name__ == "__main__":
    work = tempfile.mkdtemp(prefix="symel_dump_")
    for name in ("tet4_n3", "cloth_n8"):
        d = os.path.join(work, name)
        CASES[name]().write_case_dir(d)
        O.run_ref_driver(d, backend="interp", threads=4)
        with open(os.path.join(d, "ref_dump.txt"), "rb") as f, \
                gzip.GzipFile(os.path.join(GOLDEN, name + "_dump.txt.gz"), "wb", mtime=0) as g:
            g.write(f.read())
        print(name, "dump written")
    shutil.rmtree(work)
