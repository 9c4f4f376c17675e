"""Decode Volta+ SASS control bits (stall/yield/scoreboards) from cuobjdump.
usage: python tools/sass_ctrl.py <binary> <function-substring> [start] [count]"""
import re, subprocess, sys
binary, fn = sys.argv[1], sys.argv[2]
start = int(sys.argv[3]) if len(sys.argv) > 3 else 0
count = int(sys.argv[4]) if len(sys.argv) > 4 else 80
out = subprocess.run(["cuobjdump", "-sass", binary], capture_output=True, text=True).stdout
blocks = out.split("Function : ")
for b in blocks[1:]:
    name = b.split("\n", 1)[0]
    if fn not in name:
        continue
    lines = b.split("\n")
    rows = []
    for i, ln in enumerate(lines):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", ln)
        if m:
            hi_m = re.search(r"/\* (0x[0-9a-f]+) \*/", lines[i + 1])
            hi = int(hi_m.group(1), 16)
            rows.append((m.group(1), m.group(2).strip(), hi))
    print(name)
    for off, ins, hi in rows[start:start + count]:
        stall = (hi >> 41) & 0xF
        yld = (hi >> 45) & 1
        wb = (hi >> 46) & 7
        rb = (hi >> 49) & 7
        wait = (hi >> 52) & 0x3F
        w = "".join(str(k) for k in range(6) if wait >> k & 1)
        print(f"{off} S{stall:2d} {'Y' if yld else ' '} W{wb if wb != 7 else '-'} R{rb if rb != 7 else '-'} "
              f"wait[{w:6s}] {ins}")
    break


def iteration_stalls(binary, fn, marker="STG", n=4):
    """Sum of stall counts between consecutive `marker` instructions."""
    import io, contextlib
    buf = io.StringIO()
    saved = sys.argv
    sys.argv = ["x", binary, fn, "0", "100000"]
    with contextlib.redirect_stdout(buf):
        exec(compile(open(__file__).read().split("\n\ndef iteration_stalls")[0], __file__, "exec"),
             {"__name__": "sub"})
    sys.argv = saved
    sums, cur, started = [], 0, False
    for ln in buf.getvalue().splitlines()[1:]:
        st = int(ln.split()[1][1:] or ln.split()[2]) if ln.split()[1] != "S" else int(ln.split()[2])
        if marker in ln:
            if started:
                sums.append(cur)
            cur, started = 0, True
        cur += st
    return sums[:n]
