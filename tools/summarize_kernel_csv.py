"""Turn `ncu -i x.ncu-rep --page raw --csv` exports (gpurun_out/*.raw.csv) into a committed markdown table.

    python tools/summarize_kernel_csv.py profiles/r2_deep_kernels_ncu.md "title" gpurun_out/a.raw.csv [gpurun_out/b.raw.csv ...]
"""
import csv, sys
WANT = [
    ("gpu__time_duration.sum", "time"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1/TEX %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instr"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long-scoreboard"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("smsp__average_warps_issue_stalled_membar_per_issue_active.ratio", "stall membar"),
]
out, title, files = sys.argv[1], sys.argv[2], sys.argv[3:]
lines = ["# " + title, ""]
for f in files:
    rr = list(csv.reader(open(f)))
    hdr, units = rr[0], rr[1]
    cols = [(hdr.index(k), label) for k, label in WANT if k in hdr]
    name_i = hdr.index("Kernel Name")
    lines += ["Source: `%s` (`ncu --set full --clock-control none`, raw page)" % f, "",
              "| kernel | " + " | ".join(label for _, label in cols) + " |",
              "|---|" + "---:|" * len(cols)]
    for r in rr[2:]:
        if len(r) <= name_i:
            continue
        cells = []
        for i, _ in cols:
            v = r[i]
            try:
                x = float(v)
                v = ("%.3g" % x) if abs(x) < 1e6 else ("%.4g" % x)
            except ValueError:
                pass
            cells.append("%s %s" % (v, units[i]) if units[i] not in ("", "%") else v)
        lines.append("| `%s` | " % r[name_i].split("(")[0].replace("void ", "") + " | ".join(cells) + " |")
    lines.append("")
open(out, "w").write("\n".join(lines))
print("\n".join(lines))
