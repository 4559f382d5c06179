"""Turn the ncu outputs of tools/gpu_round.sh (gpurun_out/) into the committed summaries:

    profiles/<round>_launches.csv          raw launch list (gpu__time_duration per launch)
    profiles/<round>_launches_summary.md   per-kernel totals and shares + first batch in launch order
    profiles/<round>_level_kernel_ncu_full.csv   selected metrics of the --set full capture
    profiles/<round>_traffic.json          DRAM bytes per launch of the forward level kernel
"""
import collections, csv, json, os, shutil, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r1"
out = os.path.join(ROOT, "profiles")
src = os.path.join(ROOT, "gpurun_out")
os.makedirs(out, exist_ok=True)

rows = list(csv.reader(open(os.path.join(src, "launches.csv"))))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
shutil.copy(os.path.join(src, "launches.csv"), os.path.join(out, rnd + "_launches.csv"))
agg = collections.OrderedDict()
order = []
for r in rows[hi + 1:]:
    if len(r) < 15:
        continue
    name = r[4].split("(")[0].replace("void ", "").replace("bcb200::", "")
    us = float(r[-1]) / 1e3
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += us
    order.append((name, r[8], us))
total = sum(a[1] for a in agg.values())
cmd = "ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --steps 1 --warmup 0 --no-cpu --no-extra --relabel 1"
with open(os.path.join(out, rnd + "_launches_summary.md"), "w") as fh:
    fh.write("# ncu launch list, %s (cold-cache, serialised: compare shares, not absolutes)\n\n" % rnd)
    fh.write("Command: `%s`\n(the bench workload: R-MAT scale-20 EF-16, 1024 sources of which 612 have arcs = one batch of 20 lane groups per pass; the command makes four passes -- the untimed byte-model step and the timed step on the graph renumbered by descending degree (`--relabel 1`: the default rule renumbers after 2048 sources, i.e. during the warm-up of a normal run; the renumbering kernels are in the list), then two run_bc calls of the e2e leg, each a fresh handle on the caller's ids; "
             "raw list: `%s_launches.csv`)\n\n" % (cmd, rnd))
    fh.write("| kernel | launches | total us | share |\n|---|---:|---:|---:|\n")
    for name, (cnt, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        fh.write("| `%s` | %d | %.1f | %.1f%% |\n" % (name, cnt, us, 100 * us / total))
    fh.write("\nLaunch order of the first batch (us):\n\n```\n")
    seen_reduce = False
    for name, grid, us in order:
        fh.write("%-40s %-16s %10.1f\n" % (name[:40], grid, us))
        if name.startswith("level_kernel<1") or name.startswith("level_kernel<(bool)1"):
            seen_reduce = True
        if seen_reduce and name.startswith("init_state"):
            break
    fh.write("```\n")

rep = os.path.join(src, "prof_level.ncu-rep")
rawcsv = os.path.join(src, "prof_level.raw.csv")      # exported on the GPU box (the .ncu-rep stays there)
if os.path.exists(rep) or os.path.exists(rawcsv):
    if os.path.exists(rawcsv):
        raw = open(rawcsv).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hdr = rr[0]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "launch__registers_per_thread", "launch__grid_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
    idx = [hdr.index(w) for w in want]
    with open(os.path.join(out, rnd + "_level_kernel_ncu_full.csv"), "w") as fh:
        for r in rr:
            fh.write(",".join('"%s"' % r[i] if "," in r[i] else r[i] for i in idx) + "\n")
    units = rr[1]
    def to_bytes(val, unit):
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]
        return float(val) * mult
    lev = [r for r in rr[2:] if ("level_kernel<" in r[idx[0]] and "advance" not in r[idx[0]]) or "bwd_push" in r[idx[0]] or "bwd_child" in r[idx[0]]]
    # exactly one pass: cut where the forward kernel comes back after the backward sweep
    one, seen_bwd = [], False
    for r in lev:
        fwd = "level_kernel<0" in r[idx[0]] or "level_kernel<(bool)0" in r[idx[0]]
        if fwd and seen_bwd:
            break
        seen_bwd |= not fwd
        one.append(r)
    lev = one
    per = [to_bytes(r[idx[2]], units[idx[2]]) + to_bytes(r[idx[3]], units[idx[3]]) for r in lev]
    # a child-driven backward level (bwd_child_init / bwd_push / bwd_child_apply) counts as ONE level launch, as in the
    # engine's launches_level_timed
    n_levels = sum(1 for r in lev if "level_kernel<" in r[idx[0]] or "bwd_child_apply" in r[idx[0]])
    rec = {"rmat20": sum(per) / n_levels if n_levels else None,
           "note": "dram__bytes_read.sum + dram__bytes_write.sum per level launch: sum over the %d captured kernels of one "
                   "step (level_kernel forward and backward + the bwd_push kernels of the child-driven level) / %d level launches, "
                   "captured with ncu --set full from bench.py --steps 1 --warmup 0 --no-cpu --no-extra --relabel 1"
                   % (len(per), n_levels),
           "per_launch_bytes": per,
           "per_launch_ms": [float(r[idx[1]]) * {"ms": 1.0, "us": 1e-3, "s": 1e3, "ns": 1e-6}.get(units[idx[1]], 1.0)
                             for r in lev],
           "kernels": [r[idx[0]].split("(")[0] for r in lev]}
    json.dump(rec, open(os.path.join(out, rnd + "_traffic.json"), "w"), indent=1)
print(open(os.path.join(out, rnd + "_launches_summary.md")).read()[:3000])
