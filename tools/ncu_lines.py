"""Aggregate ncu per-SASS-instruction stall samples by CUDA source line.

usage: ncu_lines.py <ncu-rep> <kernel-regex> <cubin> <mangled-function> [top]
Maps SASS offsets to source lines with `nvdisasm -g` (needs -lineinfo)."""
import csv, io, re, subprocess, sys
rep, kre, cubin, fn = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
by_inst = len(sys.argv) > 6 and sys.argv[6] == "inst"   # rank lines by executed instructions
sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
sec = sass.split(f".text.{fn}:")[1].split("//---------------------")[0]
line_of = {}
cur = None
for ln in sec.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}"],
                        capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(csvtxt)))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
hdr = rows[hi]
iA, iW, iI = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
base = None
agg, inst, kinds = {}, {}, {}
for r in rows[hi + 1:]:
    if len(r) <= iW or not r[iA].startswith("0x"):
        continue
    a = int(r[iA], 16)
    if base is None:
        base = a
    key = line_of.get(a - base, ("?", 0))
    agg[key] = agg.get(key, 0) + float(r[iW] or 0)
    inst[key] = inst.get(key, 0) + float(r[iI] or 0)
tot = sum(agg.values())
srcs = {}
for (f, l) in agg:
    if f not in srcs:
        for root in ["paper_1506_01684_b200/csrc/"]:
            try:
                srcs[f] = open(root + f).read().splitlines()
            except OSError:
                srcs[f] = []
order = sorted(agg.items(), key=(lambda kv: -inst[kv[0]]) if by_inst else (lambda kv: -kv[1]))
for key, w in order[:top]:
    f, l = key
    txt = srcs.get(f, [])[l - 1].strip() if 0 < l <= len(srcs.get(f, [])) else ""
    print(f"{100 * w / tot:5.1f}%  inst {inst[key]:12.0f}  {f}:{l:<4d} {txt[:90]}")
by_file = {}
for (f, l), w in agg.items():
    by_file[f] = by_file.get(f, 0) + w
print({f: round(100 * w / tot, 1) for f, w in by_file.items()})
