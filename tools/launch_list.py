"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of
bench.py into a markdown table: launches, total and average device time per
kernel, and each kernel's share of the step kernels.

usage: launch_list.py <launches.csv> <steps>"""
import csv, sys
lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]   # drop ncu's ==WARNING== / ==PROF== lines
rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
agg = {}
for r in rows:
    k = r["Kernel Name"].replace("<unnamed>::", "").split("(")[0]   # anonymous-namespace kernels
    if "<" in k:   # template arguments may contain spaces: keep them, name the kernel by its base
        k = k[:k.index("<")].split()[-1] + k[k.index("<"):]
    n, t = agg.get(k, (0, 0.0))
    agg[k] = (n + 1, t + float(r["Metric Value"].replace(",", "")) / 1e6)
step_k = {k: v for k, v in agg.items() if k.split("<")[0].split()[-1].split("::")[-1] in
          ("phi_tiled_kernel", "mu_tiled_kernel", "fused_kernel", "copy_kernel", "table_kernel")}
tot = sum(t for _, t in step_k.values())
print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none), {sys.argv[1]}\n")
print("| kernel | launches | total ms | avg ms | share of step kernels |\n|---|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    share = f"{100 * t / tot:.1f}%" if k in step_k else "(not in the step)"
    print(f"| {k} | {n} | {t:.3f} | {t / n:.3f} | {share} |")
