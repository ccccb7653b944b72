"""Round-2 profile summaries for profiles/ from the files scripts/profile_r02.sh leaves in
gpurun_out/r02 (raw metric CSVs of every captured kernel, source-region breakdowns of the
generated tile kernels, the launch list of the default bench command):
  profiles/r02_kernel_table.md   every captured kernel: duration, DRAM bytes, HBM GB/s and % of
                                 the measured peak, executed FP64 FLOP/s (DFMA x2 + DMUL + DADD)
                                 and % of the DFMA-probe peak, FP64 pipe %, registers, warps
                                 active, top stall reasons
  profiles/r02_regions_*.txt     source regions of the generated tile kernels
  profiles/r02_c2_launches.csv + r02_c2_launch_summary.txt
  profiles/kernel_facts.json     the dominant kernel per config (read by bench.py)
usage: python scripts/r02_summaries.py DIR [DIR ...]"""
import csv, glob, json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
FP64_PEAK = 37.06e12
try:
    HBM_PEAK = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) * 1e9
except Exception:
    HBM_PEAK = 6550e9
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
CAPTURES = {  # capture name -> what it is
    "c2_first_assemble": "config 2 + SPD, first assemble (pattern, slot map, Morton order, tile plan, copies, "
                         "tile kernel, fix-ups, energy trees) + energy_only, guard_min, SpMV, block-Jacobi, PCG",
    "c2_steady": "config 2 + SPD, one steady-state assemble",
    "c2_nospd_steady": "config 2 without SPD, one steady-state assemble",
    "c3_steady": "config 3 (tet10), one steady-state assemble",
    "c4_steady": "config 4 (cloth: membrane + bending), one steady-state assemble",
    "c5_steady": "config 5 (tets + contact pairs + inertia, SPD), one steady-state assemble",
}
FACTS = {  # facts key -> (capture, kernel name prefix, launch index among matches, label)
    "c2": ("c2_steady", "sy_7", 0, "sy_7 (fused tile kernel + reduced-space SPD, lookahead QL)"),
    "c2_nospd": ("c2_nospd_steady", "sy_6", 0, "sy_6 (fused tile kernel, factorised tape, no SPD)"),
    "c3": ("c3_steady", "sy_6", 0, "sy_6 (tet10 tile kernel, item lanes, reduce-scatter staging)"),
    "c4": ("c4_steady", "sy_6", 1, "sy_6 (bending tile kernel; membrane is the other launch)"),
    "c5": ("c5_steady", "sy_7", 1, "sy_7 (contact-pair tile kernel + reduced SPD; the tets' kernel is the other launch)"),
}


def val(d, u, k):
    v = d.get(k, "")
    try:
        return float(v.replace(",", "")) * SCALE.get(u.get(k, ""), 1.0)
    except ValueError:
        return 0.0


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    return [dict(zip(hdr, r)) for r in rows[2:]], units


def kernel_row(d, u):
    sec = val(d, u, "gpu__time_duration.sum")
    dram = val(d, u, "dram__bytes_read.sum") + val(d, u, "dram__bytes_write.sum")
    cyc = val(d, u, "sm__cycles_elapsed.avg")
    fl = (2 * val(d, u, "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed")
          + val(d, u, "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed")
          + val(d, u, "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed")) * cyc
    st = {k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]: val(d, u, k) for k in d
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    st.pop("selected", None)
    top = ", ".join("%s %.2f" % kv for kv in sorted(st.items(), key=lambda kv: -kv[1])[:3])
    return dict(name=d.get("Kernel Name", "?").split("(")[0].replace("symel_cuda::<unnamed>::", ""), sec=sec,
                dram=dram, gbs=dram / sec if sec else 0, fps=fl / sec if sec else 0,
                pipe=val(d, u, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                regs=d.get("launch__registers_per_thread", "?"),
                warps=val(d, u, "sm__warps_active.avg.pct_of_peak_sustained_active"), stalls=top)


def main():
    dirs = sys.argv[1:]
    lines = ["# Round-2 per-kernel roofline (ncu --set full, --clock-control none; cold-cache replay, so "
             "durations are serialised and slightly pessimistic)", "",
             "Peaks: HBM %.0f GB/s (MEASURED_PEAKS.json), FP64 %.2f TFLOP/s (DFMA probe, symel_cuda_fp64_peak). "
             "FP64 FLOP/s = executed DFMA x2 + DMUL + DADD (SASS thread instructions). Stall columns: warp cycles "
             "per issued instruction, top three (excluding 'selected')." % (HBM_PEAK / 1e9, FP64_PEAK / 1e12), ""]
    facts = json.load(open(os.path.join(PROF, "kernel_facts.json")))
    for cap, what in CAPTURES.items():
        path = next((p for d in dirs for p in [os.path.join(d, "raw_%s.csv" % cap)] if os.path.exists(p)), None)
        if not path:
            continue
        rows, units = load(path)
        lines += ["## %s: %s" % (cap, what), "",
                  "| # | kernel | ms | DRAM GB | HBM GB/s | % HBM | FP64 TFLOP/s | % FP64 | FP64 pipe % | regs | warps % | top stalls |",
                  "|---|---|---|---|---|---|---|---|---|---|---|---|"]
        for i, d in enumerate(rows):
            k = kernel_row(d, units)
            lines.append("| %d | %s | %.4f | %.3f | %.0f | %.1f | %.2f | %.1f | %.1f | %s | %.1f | %s |" % (
                i, k["name"][:44], k["sec"] * 1e3, k["dram"] / 1e9, k["gbs"] / 1e9, 100 * k["gbs"] / HBM_PEAK,
                k["fps"] / 1e12, 100 * k["fps"] / FP64_PEAK, k["pipe"], k["regs"], k["warps"], k["stalls"]))
        lines.append("")
        for key, (fc, prefix, idx, label) in FACTS.items():
            if fc != cap:
                continue
            ms = [d for d in rows if d.get("Kernel Name", "").startswith(prefix)]
            if len(ms) <= idx:
                continue
            k = kernel_row(ms[idx], units)
            facts[key] = {"kernel": label, "traffic_bytes": int(k["dram"]), "fp64_pipe_active_pct": round(k["pipe"], 2),
                          "duration_ms_ncu": round(k["sec"] * 1e3, 3), "warps_active_pct": round(k["warps"], 1),
                          "regs": int(k["regs"]) if str(k["regs"]).isdigit() else k["regs"],
                          "executed_fp64_tflops": round(k["fps"] / 1e12, 2),
                          "capture": "profiles/r02_kernel_table.md (%s)" % cap}
    open(os.path.join(PROF, "r02_kernel_table.md"), "w").write("\n".join(lines) + "\n")
    json.dump(facts, open(os.path.join(PROF, "kernel_facts.json"), "w"), indent=1)
    for d in dirs:
        for f in glob.glob(os.path.join(d, "regions_*.txt")):
            shutil.copy(f, os.path.join(PROF, "r02_" + os.path.basename(f)))
        lc = os.path.join(d, "launches_c2.csv")
        if os.path.exists(lc):
            shutil.copy(lc, os.path.join(PROF, "r02_c2_launches.csv"))
            out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "launch_summary.py"), lc],
                                 capture_output=True, text=True).stdout
            open(os.path.join(PROF, "r02_c2_launch_summary.txt"), "w").write(
                "# ncu launch list of: python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline\n"
                "# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: shares, not "
                "absolute times)\n" + out)
    print("\n".join(lines[:12]))


if __name__ == "__main__":
    main()
