"""Search equivalent source formulations of the speculative PLCM step for the
fewest static cycles per iteration (ptxas stall counts).  Tool, CPU-only."""
import itertools, os, random, re, subprocess, sys, tempfile

HDR = r'''
#include <cstdint>
struct LaneConst { double p, q, yh_p, yl_p, yh_q, yl_q, cthr, a_b, a_d, hp, hq; uint32_t plo, pad; };
__device__ __forceinline__ double step(double x, const LaneConst& c) {
%s
}
__global__ void __launch_bounds__(128, 1) k(double* state, const LaneConst* lcs, double* orbit, uint32_t iters, uint32_t nl) {
  const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nl) return;
  const LaneConst c = lcs[l];
  double x = state[l];
  double* o = orbit + l;
  for (uint32_t i = 0; i < iters; i += 8) {
#pragma unroll
    for (int t = 0; t < 8; ++t) { x = step(x, c); o[size_t(t) * nl] = x; }
    o += size_t(8) * nl;
  }
  state[l] = x;
}
'''

STMTS = {
    "c1": "const bool c1 = x > 0.5;",
    "low": "const bool low = (x < c.p) | (x > c.cthr);",
    "t1": "const double t1 = __dsub_rn(1.0, x);",
    "nd": "const double nd = __dsub_rn(t1, c.p);",
    "nb": "const double nb = __dsub_rn(x, c.p);",
    "f": "const double f = c1 ? t1 : x;",
    "g": "const double g = low ? c.yl_p : c.yl_q;",
    "a": "const double a = low ? 0.0 : c.a_b;",
    "corr": "const double corr = __fma_rn(f, g, a);",
    "num": "const double num = low ? f : (c1 ? nd : nb);",
    "yh": "const double yh = low ? c.yh_p : c.yh_q;",
}
DEPS = {"nd": ["t1"], "f": ["c1", "t1"], "g": ["low"], "a": ["low"],
        "corr": ["f", "g", "a"], "num": ["low", "f", "c1", "nd", "nb"], "yh": ["low"]}
ALT = {
    "low": ["const bool low = (x < c.p) | (x > c.cthr);",
            "const bool low = (x > c.cthr) | (x < c.p);",
            "const bool low = c1 ? (x > c.cthr) : (x < c.p);"],
    "nd": ["const double nd = __dsub_rn(t1, c.p);", "const double nd = __dadd_rn(t1, -c.p);"],
    "num": ["const double num = low ? f : (c1 ? nd : nb);",
            "const double num = !low ? (c1 ? nd : nb) : f;",
            "const double num = low ? (c1 ? t1 : x) : (c1 ? nd : nb);"],
    "corr": ["const double corr = __fma_rn(f, g, a);", "const double corr = __fma_rn(g, f, a);"],
}


def topo_orders(rng, n):
    names = list(STMTS)
    out = set()
    tries = 0
    while len(out) < n and tries < 10000:
        tries += 1
        placed, order = set(), []
        rem = names[:]
        while rem:
            ready = [s for s in rem if all(d in placed for d in DEPS.get(s, []))]
            s = rng.choice(ready)
            order.append(s); placed.add(s); rem.remove(s)
        out.add(tuple(order))
    return list(out)


def cycles(cubin):
    out = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True).stdout
    lines = out.split("\n")
    rows = []
    for i, ln in enumerate(lines):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", ln)
        if m:
            hi = int(re.search(r"/\* (0x[0-9a-f]+) \*/", lines[i + 1]).group(1), 16)
            rows.append((m.group(2), (hi >> 41) & 0xF))
    sums, cur, st = [], 0, False
    for ins, s in rows:
        if re.search(r"^DADD R\d+, -R\d+(\.reuse)?, 1", ins):
            if st:
                sums.append(cur)
            cur, st = 0, True
        cur += s
    return sums


def main(n=40, seed=1):
    rng = random.Random(seed)
    results = []
    for order in topo_orders(rng, n):
        body = []
        choice = {}
        for s in order:
            stmt = rng.choice(ALT[s]) if s in ALT else STMTS[s]
            choice[s] = stmt
            body.append("  " + stmt)
        body.append("  return __fma_rn(num, yh, corr);")
        src = HDR % "\n".join(body)
        with tempfile.TemporaryDirectory() as d:
            cu, cb = os.path.join(d, "k.cu"), os.path.join(d, "k.cubin")
            open(cu, "w").write(src)
            r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                                "-fmad=false", "-cubin", cu, "-o", cb], capture_output=True)
            if r.returncode:
                continue
            cs = cycles(cb)
        if cs:
            steady = sorted(cs)[len(cs) // 2]
            results.append((steady, cs, "\n".join(body)))
    results.sort(key=lambda t: t[0])
    for steady, cs, body in results[:3]:
        print("static cycles", steady, cs)
        print(body)
        print()
    print("distribution:", sorted(r[0] for r in results))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 40)
