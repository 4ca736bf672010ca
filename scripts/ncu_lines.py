"""Warp-stall samples per CUDA source line of an ncu report (source page, cuda+sass):
python scripts/ncu_lines.py rep.ncu-rep [top]"""
import collections
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = collections.Counter()
txt = {}
fname = "?"
si = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        si = r.index("Warp Stall Sampling (All Samples)")
        continue
    if si is None or len(r) <= si:
        continue
    if r[0].isdigit():  # a source line row (its samples are the sum of its SASS rows)
        key = (fname, int(r[0]))
        txt[key] = r[1][:90]
        if r[si].isdigit():
            agg[key] += int(r[si])
tot = sum(agg.values())
print("total samples", tot)
for (f, ln), c in agg.most_common(top):
    print(f"{c:6d} {100.0 * c / max(tot, 1):5.1f}%  {f}:{ln}  {txt[(f, ln)]}")
