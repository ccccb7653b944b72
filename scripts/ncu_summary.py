"""Prints the headline metrics of an ncu report (first kernel) -- used for profiles/ summaries."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "lts__t_bytes.sum",
        "smsp__pcsamp_sample_count"]
for row in rows[2:]:
    for w in want:
        if w in h:
            print("%-62s %s %s" % (w, row[h.index(w)], u[h.index(w)]))
    stalls = [(int(float(row[i].replace(",", "") or 0)), h[i].replace("smsp__pcsamp_warps_issue_stalled_", ""))
              for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("_not_issued")]
    tot = sum(s for s, _ in stalls) or 1
    print("stall samples:", ", ".join("%s %.1f%%" % (n, 100.0 * s / tot) for s, n in sorted(stalls, reverse=True)[:8]))
