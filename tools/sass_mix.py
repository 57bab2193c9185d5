"""Dynamic SASS opcode mix of one kernel from an ncu report (source page, SASS view).

usage: sass_mix.py <ncu-rep> <kernel-regex> [cells]
Prints warp-level executed instructions per opcode, and per cell if `cells` is given
(thread instructions / cells), plus the warp-stall samples attributed to each opcode."""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
cells = float(sys.argv[3]) if len(sys.argv) > 3 else None
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
hdr = rows[hi]
iS, iI, iT, iW = (hdr.index(h) for h in ("Source", "Instructions Executed", "Thread Instructions Executed",
                                          "Warp Stall Sampling (All Samples)"))
mix, thr, stall = {}, {}, {}
for r in rows[hi + 1:]:
    if len(r) <= iW or not r[0].startswith("0x"):
        continue
    toks = r[iS].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    mix[op] = mix.get(op, 0) + float(r[iI] or 0)
    thr[op] = thr.get(op, 0) + float(r[iT] or 0)
    stall[op] = stall.get(op, 0) + float(r[iW] or 0)
tot, tst = sum(mix.values()), sum(stall.values())
print(f"total warp instructions {tot:.4g}" + (f"  thread-instr/cell {sum(thr.values()) / cells:.1f}" if cells else ""))
for op, v in sorted(mix.items(), key=lambda kv: -kv[1])[:40]:
    per = f"  {thr[op] / cells:7.1f}/cell" if cells else ""
    print(f"{op:10s} {v:14.0f} {100 * v / tot:5.1f}%{per}  stall {100 * stall[op] / tst:5.1f}%")
