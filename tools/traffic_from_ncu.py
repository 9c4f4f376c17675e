"""Writes profiles/traffic.json from committed `ncu --set full` raw CSVs:
DRAM bytes (read + write) per launch of each product kernel, next to the
launch's size, so bench.py can report roofline.traffic per launch and the
per-frame device traffic against the algorithmic 2F.  Tool.

Usage: python tools/traffic_from_ncu.py profiles/r02b_ncu_full_raw.csv ..."""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def rows(path):
    r = list(csv.reader(open(path)))
    h, units = r[0], r[1]
    for v in r[2:]:
        yield {k: (x, u) for k, x, u in zip(h, v, units)}


def num(cell):
    x, u = cell
    return float(x.replace(",", "")) * UNIT.get(u, 1)


out = {"source": [os.path.relpath(p, ROOT) for p in sys.argv[1:]],
       "method": "dram__bytes_read.sum + dram__bytes_write.sum of one launch, ncu --set full "
                 "--clock-control none (cache flushed before each replayed kernel: cold L2); "
                 "writes still dirty in L2 at kernel end are not in dram__bytes_write"}
for p in sys.argv[1:]:
    for r in rows(p):
        name = re.sub(r"<.*>", "", r["Kernel Name"][0].split("(")[0].split("::")[-1]).strip()
        rec = {"dram_bytes": num(r["dram__bytes_read.sum"]) + num(r["dram__bytes_write.sum"]),
               "dram_read": num(r["dram__bytes_read.sum"]),
               "dram_write": num(r["dram__bytes_write.sum"]),
               "duration_us": float(r["gpu__time_duration.sum"][0].replace(",", "")) *
               {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r["gpu__time_duration.sum"][1]],
               "grid": r["launch__grid_size"][0], "block": r["launch__block_size"][0]}
        out.setdefault(name, rec)  # first launch of each kernel
# the generator launches of tools/ncu_capture.py: one C4 launch of 131072
# iterations x 128 lanes (k_prbg_chain_walk writes one 8-byte checkpoint per lane
# per 8 iterations: 2.1 MB, consumed from L2 by k_prbg_verify_emit)
for k in ("k_prbg_chain", "k_prbg_chain_walk", "k_prbg_verify_emit"):
    if k in out:
        out[k].update({"iterations": 131072, "lanes": 128,
                       "checkpoint_bytes_written": 131072 // 8 * 128 * 8})
json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
