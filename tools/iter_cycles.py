"""Static cycles per unrolled loop iteration of a SASS function: sum of stall
counts between consecutive instructions matching a marker regex.
usage: python tools/iter_cycles.py <binary> <function-substring> <marker-regex>"""
import re, subprocess, sys
binary, fn, marker = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["cuobjdump", "-sass", binary], capture_output=True, text=True).stdout
for b in out.split("Function : ")[1:]:
    name = b.split("\n", 1)[0]
    if fn not in name:
        continue
    lines = b.split("\n")
    rows = []
    for i, ln in enumerate(lines):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", ln)
        if m:
            hi = int(re.search(r"/\* (0x[0-9a-f]+) \*/", lines[i + 1]).group(1), 16)
            rows.append((m.group(2), (hi >> 41) & 0xF))
    sums, cur, started = [], 0, False
    for ins, st in rows:
        if re.search(marker, ins):
            if started:
                sums.append(cur)
            cur, started = 0, True
        cur += st
    print(name[-40:], "per-iteration static cycles:", sums[:12])
