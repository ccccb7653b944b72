"""CPU: the device kernel cache behaves like the reference's KernelCache (cache.hpp:64-180) on
the cubin side: entries are named by the reference's kernel_key (the tape digest,
registry.hpp:415-428), a warm start rebuilds nothing (acceptance_main.cpp:1113-1151, check11),
and a corrupt entry is a warning plus a rebuild that overwrites it (cache.hpp:119-148).
Device-less contexts (symel_cuda_create(-1)) generate and compile without launching."""
import glob
import os

from conftest import golden_tape
from paper_2303_02156_b200 import configs as C
from paper_2303_02156_b200.systems import DeviceSystem


def _ctx(cache):
    ds = DeviceSystem(C.tet4_case(2), tapes=golden_tape, device=-1)
    ds.asm.lib.symel_cuda_set_cache_dir(ds.asm.h, str(cache).encode())
    return ds


def test_entries_named_by_kernel_key(tmp_path):
    ds = _ctx(tmp_path)
    ds.asm.precompile(ds.energies["elastic"], "deterministic")
    key = golden_tape("tet4_elastic")[8:40].hex()
    cubins = glob.glob(str(tmp_path / "*.sm100a.cubin"))
    assert cubins and all(os.path.basename(p).startswith(key + ".") for p in cubins)
    assert len(glob.glob(str(tmp_path / "*.meta"))) == len(cubins)
    st = ds.asm.cache_stats()
    assert st["builds"] == len(cubins) and st["disk_hits"] == 0 and st["corrupt"] == 0


def test_warm_start_builds_nothing(tmp_path):
    cold = _ctx(tmp_path)
    cold.asm.precompile(cold.energies["elastic"], "deterministic")
    cold.asm.precompile(cold.energies["elastic"], "ordered")
    n = cold.asm.cache_stats()["builds"]
    assert n > 0
    warm = _ctx(tmp_path)
    warm.asm.precompile(warm.energies["elastic"], "deterministic")
    warm.asm.precompile(warm.energies["elastic"], "ordered")
    st = warm.asm.cache_stats()
    assert st["builds"] == 0 and st["disk_hits"] == n and st["corrupt"] == 0
    assert warm.asm.timings().compile_ms == 0.0


def test_corrupt_entry_warns_and_rebuilds(tmp_path, capfd):
    cold = _ctx(tmp_path)
    cold.asm.precompile(cold.energies["elastic"], "deterministic")
    cubins = sorted(glob.glob(str(tmp_path / "*.sm100a.cubin")))
    good = open(cubins[0], "rb").read()
    with open(cubins[0], "wb") as f:
        f.write(b"garbage" * 10)
    capfd.readouterr()
    warm = _ctx(tmp_path)
    warm.asm.precompile(warm.energies["elastic"], "deterministic")
    st = warm.asm.cache_stats()
    assert st["corrupt"] == 1 and st["builds"] == 1 and st["disk_hits"] == len(cubins) - 1
    assert "corrupt cache entry, rebuilding" in capfd.readouterr().err
    assert open(cubins[0], "rb").read() == good  # overwritten with a valid image
    again = _ctx(tmp_path)
    again.asm.precompile(again.energies["elastic"], "deterministic")
    assert again.asm.cache_stats()["corrupt"] == 0 and again.asm.cache_stats()["builds"] == 0
