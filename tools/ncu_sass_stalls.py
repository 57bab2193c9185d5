"""Per-SASS-instruction stall breakdown of one kernel in an ncu report: the top
instructions by warp-stall samples, with their dominant stall reasons and the
CUDA source line (nvdisasm -g of the cubin).

usage: ncu_sass_stalls.py <ncu-rep> <kernel-regex> <cubin> <mangled-function> [top]"""
import csv, io, re, subprocess, sys
rep, kre, cubin, fn = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
sec = sass.split(f".text.{fn}:")[1].split("//---------------------")[0]
line_of, text_of, cur = {}, {}, None
for ln in sec.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        off = int(m.group(1), 16)
        line_of[off] = cur
        text_of[off] = m.group(2).strip()
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if "Address" in r)
hdr = rows[hi]
iA, iW = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
st = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
recs = []
base = None
for r in rows[hi + 1:]:
    if len(r) <= iW or not r[iA].startswith("0x"):
        continue
    a = int(r[iA], 16)
    base = a if base is None else min(base, a)
    try:
        w = float(r[iW] or 0)
    except ValueError:
        continue
    reasons = sorted(((float(r[i] or 0), h[6:]) for i, h in st), reverse=True)[:3]
    recs.append((w, a, reasons))
tot = sum(w for w, _, _ in recs) or 1
for w, a, reasons in sorted(recs, reverse=True)[:top]:
    off = a - base
    src = line_of.get(off)
    print(f"{100 * w / tot:5.1f}%  {off:05x}  {text_of.get(off, '?')[:40]:40s} {src}  " +
          ", ".join(f"{n} {v:.0f}" for v, n in reasons if v > 0))
