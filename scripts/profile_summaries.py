"""Write the committed ncu summaries under profiles/ from a gpurun_out capture:
  python scripts/profile_summaries.py <round> <launches.csv> <full.ncu-rep | raw.csv> <bench-cmd>
-> profiles/<round>_launches_C5w.csv, <round>_launches_C5w_summary.md,
   <round>_ncu_full_C5w.md, ncu_traffic.json (DRAM bytes per launch of the
   step kernels).  The third argument may be the report's raw page as CSV
   (`ncu -i rep --page raw --csv`), written on the GPU box when the report
   is too large to copy back."""
import csv, collections, json, os, re, shutil, subprocess, sys

tag, launches, rep, cmd = sys.argv[1:5]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
prof = os.path.join(root, "profiles")
shutil.copy(launches, os.path.join(prof, f"{tag}_launches_C5w.csv"))

# launch list: kernel name, duration
rows = [r for r in csv.reader(open(launches)) if len(r) > 5]
hdr = rows[0]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = collections.OrderedDict()
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*$", "", r[ik]).replace("void ", "")
    name = r[ik].split("(")[0].replace("void ", "") if "<" not in r[ik] else r[ik][: r[ik].index(">") + 1].replace("void ", "")
    v = float(r[iv].replace(",", ""))
    unit_ms = 1e-6 if float(v) > 1e4 else 1e-3   # ncu reports ns or us
    t = tot.setdefault(name, [0, 0.0])
    t[0] += 1
    t[1] += v
# unit: ncu csv gpu__time_duration in nsecond (column "Metric Unit")
iu = hdr.index("Metric Unit")
unit = next(r[iu] for r in rows[1:] if r[im] == "gpu__time_duration.sum")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}[unit]
all_ms = sum(v[1] for v in tot.values()) * scale
step = {k: v for k, v in tot.items() if v[0] >= 5}
step_ms = sum(v[1] / v[0] for v in step.values()) * scale
out = [f"# ncu launch list — `{cmd}` (C5w, n=16M, B=32 fp64)", "",
       "`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised launches; compare shares).",
       "Setup kernels run once; the step kernels 5 times (3 warm-up + 2 timed).", "",
       "| kernel | launches | total ms | share |", "|---|---|---|---|"]
for k, v in sorted(tot.items(), key=lambda x: -x[1][1]):
    out.append(f"| `{k}` | {v[0]} | {v[1] * scale:.3f} | {v[1] * scale / all_ms:.3f} |")
out += ["", "Step kernels only (share of the step; compare with bench.py's `kernels[*].share`):", "",
        "| kernel | ms per launch | share of step |", "|---|---|---|"]
for k, v in sorted(step.items(), key=lambda x: -x[1][1]):
    per = v[1] / v[0] * scale
    out.append(f"| `{k}` | {per:.3f} | {per / step_ms:.3f} |")
open(os.path.join(prof, f"{tag}_launches_C5w_summary.md"), "w").write("\n".join(out) + "\n")

# full capture
metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "l1tex__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "launch__cluster_dim_x", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
raw = (open(rep).read() if rep.endswith(".csv")
       else subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
rr = list(csv.reader(raw.splitlines()))
h, units = rr[0], rr[1]
out = [f"# ncu --set full, C5w full size (n=16M, B=32 fp64), first launch of each step kernel", "",
       f"`ncu --set full --clock-control none --import-source on` (kernels: the step's) on `{cmd}`.", ""]
traffic = {}
keymap = {"k_scan_tiles": "scan", "k_scan_carry_tiles": "scan", "k_gather_r4": "gather", "k_gather_pi": "gather",
          "k_to_rank_major": "perm", "k_moeb_ringcl": "moebius_solve"}
for row in rr[2:]:
    kn = row[h.index("Kernel Name")]
    out.append(f"## {kn}")
    for m in metrics:
        if m in h:
            out.append(f"- {m} = {row[h.index(m)]} {units[h.index(m)]}")
    out.append("")
    for pre, key in keymap.items():
        if re.search(r"\b" + pre + r"\b", kn):
            def gb(m):
                v = float(row[h.index(m)].replace(",", ""))
                u = units[h.index(m)]
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
            traffic[key] = traffic.get(key, 0.0) + gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
open(os.path.join(prof, f"{tag}_ncu_full_C5w.md"), "w").write("\n".join(out) + "\n")
ent = {k: {"bytes": v, "capture": f"profiles/{tag}_ncu_full_C5w.md"} for k, v in traffic.items()}
json.dump({"C5w": ent, "_note": f"dram__bytes_read.sum + dram__bytes_write.sum per launch from profiles/{tag}_ncu_full_C5w.md "
           "(scan = both scan-tile passes + the carry pass)"},
          open(os.path.join(prof, "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(traffic))
