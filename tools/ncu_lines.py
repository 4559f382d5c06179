"""Per-source-line hot spots of one kernel launch in an .ncu-rep (dev tool).

    python tools/ncu_lines.py report.ncu-rep LAUNCH_INDEX [TOP]
"""
import csv, subprocess, sys
rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
print(rows[hi - 1][:2] if hi else "")
hdr = rows[hi]
keys = ["stall_long_sb", "stall_wait", "stall_not_selected", "stall_short_sb", "stall_lg", "stall_math",
        "stall_branch_resolving", "stall_no_inst", "stall_dispatch", "stall_mio"]
c = {n: hdr.index(n) for n in ["# Samples", "Instructions Executed", "Thread Instructions Executed"] + keys}
data = []
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or not r[0]:
        continue
    try:
        data.append((int(r[0]), r[1].strip()[:64], int(r[c["# Samples"]]), int(r[c["Instructions Executed"]]),
                     int(r[c["Thread Instructions Executed"]])) + tuple(int(r[c[k]]) for k in keys))
    except ValueError:
        pass
ts = sum(d[2] for d in data) or 1
ti = sum(d[3] for d in data) or 1
print("samples", ts, "warp instructions", ti)
for d in sorted(data, key=lambda d: -d[2])[:top]:
    stalls = " ".join("%s=%d" % (k[6:10], v) for k, v in zip(keys, d[5:]) if v * 20 > d[2])
    print("%4d %-64s smp %5.1f%% ins %5.1f%% act %4.1f | %s"
          % (d[0], d[1], 100 * d[2] / ts, 100 * d[3] / ti, d[4] / max(d[3], 1), stalls))

# instruction / sample share by source region of bc_kernels.cuh (line ranges given as a:b,c:d ...)
if len(sys.argv) > 4:
    for spec in sys.argv[4].split(","):
        a, b = (int(x) for x in spec.split(":"))
        ins = sum(d[3] for d in data if a <= d[0] <= b)
        smp = sum(d[2] for d in data if a <= d[0] <= b)
        print("lines %4d-%4d: ins %5.1f%% samples %5.1f%%" % (a, b, 100 * ins / ti, 100 * smp / ts))
