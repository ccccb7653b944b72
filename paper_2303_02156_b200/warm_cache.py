"""Pre-compiles (NVRTC, sm_100a, no GPU needed) the generated kernels of the BASELINE energies
into the in-tree cubin cache paper_2303_02156_b200/_cache, which travels to the GPU box with
the built library. A cold cache only costs compile time; results never depend on it."""
import os
import sys
import time

from . import configs as C
from .device import DeviceAssembler, load_library
from . import systems as S


def _register(kind, tapes, spd=False):
    """Registers the energies of a config kind on a device-less context (shapes only)."""
    cases = {"tet4": C.tet4_case(2), "tet10": C.config3(1), "cloth": C.config4(4), "contact": C.config5(2, 4)}
    return S.DeviceSystem(cases[kind], tapes=tapes, spd=spd, device=-1)


def main(quick: bool = False):
    load_library()
    tapes = S.default_tapes()
    kinds = ["tet4", "contact"] if quick else ["tet4", "contact", "cloth", "tet10"]
    modes = ["deterministic", "atomic", "ordered"]
    for kind in kinds:
        # configs 2 and 5 (the bench default and the contact config) project to SPD
        for spd in ((False, True) if kind in ("tet4", "contact") else (False,)):
            t0 = time.time()
            ds = _register(kind, tapes, spd)
            for eid in ds.energies.values():
                for m in modes:
                    ds.asm.precompile(eid, m)
            print(f"warm_cache: {kind}{' (SPD)' if spd else ''} kernels ready in {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main(quick="--quick" in sys.argv)
