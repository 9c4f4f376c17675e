"""Summarise an ncu --set full --import-source capture's SASS source page:
instruction runs (consecutive instructions with equal execution counts)
with their stall samples, and the hottest instructions.  Tool."""
import csv, subprocess, sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
kern = None; data = {}; hdr = None
for r in rows:
    if r and r[0] == "Kernel Name":
        kern = r[1]; data[kern] = []; hdr = None; continue
    if r and r[0] == "Address":
        hdr = r; continue
    if kern and hdr and len(r) > 5:
        data[kern].append(r)
h = hdr
ie = h.index("Instructions Executed"); st = h.index("Warp Stall Sampling (All Samples)")
at = h.index("Avg. Threads Executed")
for k, v in data.items():
    if kfilter not in k:
        continue
    tot = sum(int(r[ie] or 0) for r in v); sam = sum(int(r[st] or 0) for r in v)
    print(k[:90], "instructions", tot, "samples", sam)
    runs = []
    for r in v:
        n = int(r[ie] or 0); s = int(r[st] or 0)
        if runs and runs[-1][1] == n:
            runs[-1][2] += 1; runs[-1][3] += s; runs[-1][5] = r[1][:44]
        else:
            runs.append([r[0][-5:], n, 1, s, r[1][:44], r[1][:44], r[at]])
    thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
    for x in runs:
        if x[1] * x[2] > thr * tot or x[3] > thr * sam:
            print(f"{x[0]} exec {x[1]:7d} x{x[2]:4d} = {x[1]*x[2]:8d}  stall {x[3]:5d}  thr {x[6]:>5}  | {x[4]} ... {x[5]}")
