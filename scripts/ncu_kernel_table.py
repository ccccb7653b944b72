"""Per-kernel roofline table from ncu --set full reports (every kernel of the report):
duration, DRAM bytes, achieved HBM GB/s and executed FP64 FLOP/s (DFMA x2 + DMUL + DADD, from
the SASS thread-instruction counters), each against the B200 peaks (measured HBM copy bandwidth
from MEASURED_PEAKS.json; FP64 = the DFMA probe of symel_cuda_fp64_peak).

usage: python scripts/ncu_kernel_table.py OUT.md REPORT.ncu-rep [REPORT ...]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FP64_PEAK = 37.09e12
try:
    HBM_PEAK = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) * 1e9
except Exception:
    HBM_PEAK = 6550e9


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, data = r[0], r[1], r[2:]
    return [dict(zip(hdr, x)) for x in data], dict(zip(hdr, units))


def num(d, k, default=0.0):
    v = d.get(k, "")
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return default


def main():
    out, reps = sys.argv[1], sys.argv[2:]
    lines = ["| report | # | kernel | ms | DRAM GB | HBM GB/s | % HBM | FP64 TFLOP/s | % FP64 | FP64 pipe % | regs | warps active % |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for rep in reps:
        rows, units = rows_of(rep)
        for i, d in enumerate(rows):
            t = num(d, "gpu__time_duration.sum")
            tu = units.get("gpu__time_duration.sum", "ns")
            sec = t * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(tu, 1e-9)
            rb = num(d, "dram__bytes_read.sum") * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(
                units.get("dram__bytes_read.sum", "byte"), 1)
            wb = num(d, "dram__bytes_write.sum") * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(
                units.get("dram__bytes_write.sum", "byte"), 1)
            cyc = num(d, "sm__cycles_elapsed.avg")
            fl_per_cyc = (2 * num(d, "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed")
                          + num(d, "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed")
                          + num(d, "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed"))
            flops = fl_per_cyc * cyc
            fps = flops / sec if sec else 0.0
            gbs = (rb + wb) / sec if sec else 0.0
            lines.append("| %s | %d | %s | %.4f | %.3f | %.0f | %.1f | %.2f | %.1f | %.1f | %s | %.1f |" % (
                os.path.basename(rep).replace(".ncu-rep", ""), i, d.get("Kernel Name", "?")[:48], sec * 1e3,
                (rb + wb) / 1e9, gbs / 1e9, 100 * gbs / HBM_PEAK, fps / 1e12, 100 * fps / FP64_PEAK,
                num(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                d.get("launch__registers_per_thread", "?"),
                num(d, "sm__warps_active.avg.pct_of_peak_sustained_active")))
    hdr = ("# Per-kernel roofline (ncu --set full, --clock-control none; cold-cache replay, so durations are "
           "serialised and slightly pessimistic)\n\nPeaks: HBM %.0f GB/s (MEASURED_PEAKS.json), FP64 %.2f TFLOP/s "
           "(DFMA probe). FP64 FLOP/s = executed DFMA x2 + DMUL + DADD (SASS thread instructions).\n\n"
           % (HBM_PEAK / 1e9, FP64_PEAK / 1e12))
    open(out, "w").write(hdr + "\n".join(lines) + "\n")
    print(hdr + "\n".join(lines))


if __name__ == "__main__":
    main()
