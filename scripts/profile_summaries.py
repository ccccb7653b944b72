"""Turns the reports of scripts/profile_round.sh (gpurun_out/prof_r01_*.ncu-rep) into the
summaries under profiles/ (headline metrics + stall reasons + source regions of the generated
kernel) and profiles/kernel_facts.json (read by bench.py). Run here after the GPU call; the
generated kernel sources are dumped with scripts/dump_kernel_source.py."""
import json, os, re, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/tmp/profile_src"
os.chdir(ROOT)
for k in ("tet4 1", "tet4 0", "contact 1", "cloth 0", "tet10 0"):
    subprocess.run([sys.executable, "scripts/dump_kernel_source.py"] + k.split() + [SRC], check=True,
                   capture_output=True)
JOBS = [  # report, launch index, generated source, command, what, facts key, kernel label
    ("c2_spd_tile", 0, "tet4_spd_elastic.cu", "--config c2 --steps 3",
     "config 2 tile kernel: element tape + reduced 9x9 SPD (lookahead QL) + tile reduction, 2nd launch",
     "c2", "sy_7 (fused tile kernel + reduced-space SPD, lookahead QL)"),
    ("c2_nospd_tile", 0, "tet4_elastic.cu", "--config c2 --no-spd --steps 3",
     "config 2 without SPD: fused tile kernel (factorised tape + tile reduction), 2nd launch",
     "c2_nospd", "sy_6 (fused tile kernel, factorised tape, no SPD)"),
    ("c5_tiles", 0, "contact_spd_elastic.cu", "--config c5 --steps 3",
     "config 5, tets (6M, reduced SPD, lookahead QL), 2nd step", None, None),
    ("c5_tiles", 1, "contact_spd_contact.cu", "--config c5 --steps 3",
     "config 5, point-triangle contact pairs (4M, exact rounding, reduced SPD, plain QL), 2nd step",
     "c5", "sy_7 (contact-pair tile kernel + reduced SPD; the tets' kernel is the other launch)"),
    ("c4_tiles", 0, "cloth_membrane.cu", "--config c4 --steps 3", "config 4, StVK membrane tile kernel, 2nd step",
     None, None),
    ("c4_tiles", 1, "cloth_bending.cu", "--config c4 --steps 3",
     "config 4, hinge-bending tile kernel (144-double Q per flap, SoA), 2nd step",
     "c4", "sy_6 (bending tile kernel; membrane is the other launch)"),
    ("c3_tile", 0, "tet10_elastic.cu", "--config c3 --steps 3",
     "config 3 tet10 tile kernel (item lanes, 4 quadrature points), 2nd launch",
     "c3", "sy_6 (tet10 tile kernel, item lanes, reduce-scatter staging)"),
]


def parse(text):
    d = {}
    for line in text.splitlines():
        m = re.match(r"(\S+)\s+([\d.,]+)\s*(\S*)", line)
        if m:
            try:
                d[m.group(1)] = (float(m.group(2).replace(",", "")), m.group(3))
            except ValueError:
                pass
    return d


def nbytes(v):
    x, u = v
    return int(x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u])


facts = json.load(open("profiles/kernel_facts.json"))
for name, idx, src, cmd, what, key, label in JOBS:
    rep = f"gpurun_out/prof_r01_{name}.ncu-rep"
    shutil.copy(rep, f"profiles/prof_r01_{name}.ncu-rep")
    summ = subprocess.run([sys.executable, "scripts/ncu_summary.py", rep], capture_output=True, text=True).stdout
    body = "Kernel Name" + summ.split("Kernel Name")[1 + idx]
    env = dict(os.environ, NCU_FILTER=f"--launch-skip {idx} --launch-count 1")
    regions = subprocess.run([sys.executable, "scripts/ncu_regions.py", rep, os.path.join(SRC, src)], env=env,
                             capture_output=True, text=True).stdout
    out = f"profiles/r01_{name}{'_' + str(idx) if name in ('c5_tiles', 'c4_tiles') else ''}_ncu_full.txt"
    with open(out, "w") as f:
        f.write(f"# ncu --set full --import-source on --clock-control none: {what}\n"
                f"# command: python scripts/profile_step.py {cmd} (report profiles/prof_r01_{name}.ncu-rep, launch {idx})\n")
        f.write(body.rstrip() + "\n\n# source regions of the generated kernel (scripts/ncu_regions.py)\n" + regions)
    if key:
        d = parse(body)
        facts[key] = {
            "kernel": label,
            "traffic_bytes": nbytes(d["dram__bytes_read.sum"]) + nbytes(d["dram__bytes_write.sum"]),
            "fp64_pipe_active_pct": round(d["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"][0], 2),
            "duration_ms_ncu": round(d["gpu__time_duration.sum"][0], 3),
            "warps_active_pct": round(d["sm__warps_active.avg.pct_of_peak_sustained_active"][0], 1),
            "regs": int(d["launch__registers_per_thread"][0]),
            "capture": out,
        }
    print(out)
json.dump(facts, open("profiles/kernel_facts.json", "w"), indent=1)
shutil.copy("gpurun_out/launches_c2.csv", "profiles/r01_c2_spd_launches.csv")
with open("profiles/r01_c2_spd_launch_summary.txt", "w") as f:
    f.write("# ncu launch list of: python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline (config 2, SPD, deterministic)\n"
            "# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: shares, not absolute times)\n")
    f.write(subprocess.run([sys.executable, "scripts/launch_summary.py", "profiles/r01_c2_spd_launches.csv"],
                           capture_output=True, text=True).stdout)
