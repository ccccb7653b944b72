"""Writes the generated CUDA source of a config's tile kernel(s) (for ncu --resolve-source-file /
scripts/ncu_regions.py). usage: dump_kernel_source.py KIND SPD(0|1) OUTDIR
Writes both tile variants: NAME.cu (plan slice in shared memory) and NAME_g.cu (plan from L2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_02156_b200 import warm_cache as W, systems as S
from paper_2303_02156_b200.device import load_library
load_library()
kind, spd, out = sys.argv[1], sys.argv[2] == "1", sys.argv[3]
ds = W._register(kind, S.default_tapes(), spd)
os.makedirs(out, exist_ok=True)
for name, eid in ds.energies.items():
    with open(os.path.join(out, f"{kind}{'_spd' if spd else ''}_{name}.cu"), "w") as f:
        f.write(ds.asm.kernel_source(eid, "deterministic"))
    with open(os.path.join(out, f"{kind}{'_spd' if spd else ''}_{name}_g.cu"), "w") as f:
        f.write(ds.asm.kernel_source(eid, "deterministic", plan_global=True))
