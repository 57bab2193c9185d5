"""Summarise an ncu --set full capture of the sweeps into profiles/.

usage: summarize_ncu.py <report.ncu-rep> <out-prefix>   (writes <prefix>.json/.md)
Per kernel: duration, DRAM bytes, FP64 pipe %, issue %, occupancy, top stalls.
"""
import csv, io, json, subprocess, sys

rep, prefix = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
keys = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "fp64_pipe_active_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "inst_executed": "smsp__inst_executed.sum",
    "shared_ld": "smsp__sass_inst_executed_op_shared_ld.sum",
    "global_ld": "smsp__sass_inst_executed_op_global_ld.sum",
}
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "msecond": 1.0, "usecond": 1e-3, "ms": 1.0}
out = {"report": rep, "kernels": []}
for r in rows[2:]:
    k = {"name": r[hdr.index("Kernel Name")], "grid": r[hdr.index("Grid Size")] if "Grid Size" in hdr else None}
    for nk, m in keys.items():
        if m in hdr:
            v = r[hdr.index(m)].replace(",", "")
            u = units[hdr.index(m)]
            try:
                v = float(v) * scale.get(u, 1.0)
            except ValueError:
                pass
            k[nk] = v
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
            try:
                st.append((float(r[i]), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    k["top_stalls_per_issue"] = {n: round(v, 3) for v, n in sorted(st, reverse=True)[:8]}
    out["kernels"].append(k)
dram = {}
for k in out["kernels"]:
    tag = "phi" if "phi" in k["name"] else ("mu" if "mu_" in k["name"] else k["name"])
    dram[tag] = k.get("dram_read_bytes", 0) + k.get("dram_write_bytes", 0)
out["dram_bytes_per_launch"] = dram
json.dump(out, open(prefix + ".json", "w"), indent=1)
with open(prefix + ".md", "w") as f:
    f.write(f"# ncu --set full summary ({rep})\n\n")
    f.write("| kernel | ms | DRAM read GB | DRAM write GB | DRAM % | FP64 pipe % | issue % | warps % | regs | top stalls |\n")
    f.write("|---|---|---|---|---|---|---|---|---|---|\n")
    for k in out["kernels"]:
        f.write(f"| {k['name'][:40]} | {k.get('duration_ms', 0):.3f} | {k.get('dram_read_bytes', 0)/1e9:.2f} | "
                f"{k.get('dram_write_bytes', 0)/1e9:.2f} | {k.get('dram_throughput_pct', 0):.1f} | "
                f"{k.get('fp64_pipe_active_pct', 0):.1f} | {k.get('issue_active_pct', 0):.1f} | "
                f"{k.get('warps_active_pct', 0):.1f} | {k.get('registers', 0):.0f} | "
                + ", ".join(f"{n} {v}" for n, v in list(k['top_stalls_per_issue'].items())[:5]) + " |\n")
print(json.dumps(dram))
