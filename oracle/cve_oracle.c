/*
 * cve_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, deliberately naive restatement of the reference cipher path
 * (arXiv 2302.07411 reference, /root/reference/proj).  It is the CHECKER for
 * the CUDA product path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.  Nothing in paper_2302_07411_b200/ links or
 * calls it, and the product path never falls back to it.
 *
 * Parity pin: tests/test_oracle.py checks this file against (a) the golden
 * constants of the reference's own unit tests (test_chaos.cpp:96-109,
 * test_keying.cpp:160-179, test_engine.cpp:61-70/117-120; LASM:
 * test_chaos.cpp:36-45/111-123, test_keying.cpp:181-195) and (b) the
 * compiled reference itself (oracle/_ref/libcve_ref.so, built from the
 * reference sources in place by oracle/Makefile) on whole frames.
 *
 * Every function cites the reference file:line whose behaviour it restates
 * (paths relative to /root/reference/proj).  Arithmetic is IEEE binary64 with
 * FP contraction off (see Makefile: -ffp-contract=off), like the reference's
 * x86-64 Release build (no -march, so no FMA).  The LASM map calls the host
 * libm `sin`, exactly as the reference does (chaos.cpp:34-38).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_INVALID 1
#define ORC_BAD_KEY 2
#define ORC_MISMATCH 5

/* ---- L0: PLCM map ------------------------------------------------------ */

/* src/chaos.cpp:28-32 */
static double orc_plcm_step(double x, double p) {
  if (x > 0.5) x = 1.0 - x;
  if (x < p) return x / p;
  return (x - p) / (0.5 - p);
}

/* src/chaos.cpp:15-24 (kGuardEps = 2^-52) */
static double orc_plcm_guard(double x, double p) {
  if (x == 0.0 || x == p || x == 0.5 || x == 1.0) {
    x += 0x1p-52;
    if (x > 1.0) x -= 1.0;
  }
  return x;
}

double orc_plcm_iterate(double x, double p) {
  return orc_plcm_guard(orc_plcm_step(x, p), p);
}

/* src/chaos.cpp:34-38 (std::numbers::pi, evaluated left to right, glibc sin) */
static void orc_lasm_step(double* x, double* y, double mu) {
  const double pi = 3.14159265358979323846;
  double xn = sin(pi * mu * (*y + 3.0) * *x * (1.0 - *x));
  double yn = sin(pi * mu * (xn + 3.0) * *y * (1.0 - *y));
  *x = xn;
  *y = yn;
}

/* src/chaos.cpp:40-44 */
static int orc_lasm_mu_valid(double mu) {
  return (mu >= 0.37 && mu <= 0.38) || (mu >= 0.40 && mu <= 0.42) ||
         (mu >= 0.44 && mu <= 0.93) || mu == 1.0;
}

/* Two-lane byte generator, src/chaos.cpp:79-107 (ctors), 109-117 (step_lane),
 * 119-141 (refill: 6 bytes per PLCM iteration, 12 per LASM iteration, x bytes
 * then y bytes), 143-153 (fill), 46-56 (extract_bytes).  Lane q = p (PLCM) or
 * mu (LASM). */
typedef struct {
  int lasm;
  double xa, ya, qa, xb, yb, qb;
  uint8_t buf[12];
  int pos, len; /* pos == len: empty */
  uint64_t emitted;
} orc_prbg;

static int orc_plcm_valid(double x0, double p) { /* src/chaos.cpp:58-65 */
  if (!(isfinite(x0) && x0 >= 0.0 && x0 <= 1.0)) return 0;
  if (!(isfinite(p) && p > 0.0 && p < 0.5)) return 0;
  return 1;
}

static int orc_lasm_valid(double x0, double y0, double mu) { /* src/chaos.cpp:67-77 */
  if (!(isfinite(x0) && x0 >= 0.0 && x0 <= 1.0)) return 0;
  if (!(isfinite(y0) && y0 >= 0.0 && y0 <= 1.0)) return 0;
  return isfinite(mu) && orc_lasm_mu_valid(mu);
}

static void orc_step_lanes(orc_prbg* g) { /* src/chaos.cpp:109-117 */
  if (g->lasm) {
    orc_lasm_step(&g->xa, &g->ya, g->qa);
    orc_lasm_step(&g->xb, &g->yb, g->qb);
  } else {
    g->xa = orc_plcm_iterate(g->xa, g->qa);
    g->xb = orc_plcm_iterate(g->xb, g->qb);
  }
}

static void orc_prbg_init(orc_prbg* g, double xa, double pa, double xb,
                          double pb) {
  memset(g, 0, sizeof *g);
  g->qa = pa;
  g->qb = pb;
  g->xa = orc_plcm_guard(xa, pa);
  g->xb = orc_plcm_guard(xb, pb);
  for (int i = 0; i < 256; ++i) orc_step_lanes(g); /* kWarmupSteps, chaos.hpp:14 */
}

static void orc_lasm_init(orc_prbg* g, const double a[3], const double b[3]) {
  memset(g, 0, sizeof *g); /* src/chaos.cpp:93-107: no guard */
  g->lasm = 1;
  g->xa = a[0], g->ya = a[1], g->qa = a[2];
  g->xb = b[0], g->yb = b[1], g->qb = b[2];
  for (int i = 0; i < 256; ++i) orc_step_lanes(g);
}

static void orc_xor48(uint8_t* out, double a, double b) {
  uint64_t ua, ub;
  memcpy(&ua, &a, 8);
  memcpy(&ub, &b, 8);
  for (int k = 0; k < 6; ++k) out[k] = (uint8_t)((ua ^ ub) >> (8 * k));
}

static void orc_prbg_fill(orc_prbg* g, uint8_t* out, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    if (g->pos == g->len) {
      orc_step_lanes(g);
      orc_xor48(g->buf, g->xa, g->xb);
      if (g->lasm) orc_xor48(g->buf + 6, g->ya, g->yb);
      g->len = g->lasm ? 12 : 6;
      g->pos = 0;
    }
    out[i] = g->buf[g->pos++];
  }
  g->emitted += n;
}

/* Raw stream of a generator seeded with explicit lanes (test_chaos golden). */
int orc_plcm_stream(double xa, double pa, double xb, double pb, uint8_t* out,
                    size_t n) {
  orc_prbg g;
  if (!orc_plcm_valid(xa, pa) || !orc_plcm_valid(xb, pb)) return ORC_BAD_KEY;
  orc_prbg_init(&g, xa, pa, xb, pb);
  orc_prbg_fill(&g, out, n);
  return ORC_OK;
}

/* lanes = {x0a, y0a, mua, x0b, y0b, mub} */
int orc_lasm_stream(const double lanes[6], uint8_t* out, size_t n) {
  orc_prbg g;
  if (!orc_lasm_valid(lanes[0], lanes[1], lanes[2]) ||
      !orc_lasm_valid(lanes[3], lanes[4], lanes[5]))
    return ORC_BAD_KEY;
  orc_lasm_init(&g, lanes, lanes + 3);
  orc_prbg_fill(&g, out, n);
  return ORC_OK;
}

/* One LASM iteration (x, y) -> (x', y'), for the frozen examples. */
void orc_lasm_iterate(double* x, double* y, double mu) { orc_lasm_step(x, y, mu); }

/* ---- L1: key + coordinator -------------------------------------------- */

static int orc_nibble(char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  if (c >= 'A' && c <= 'F') return c - 'A' + 10;
  return -1;
}

/* src/keying.cpp:77-107.  Returns the map kind in *lasm; PLCM keys fill
 * k[0..3] = {x0a, pa, x0b, pb}, LASM keys k[0..2] = {x0, y0, mu}. */
int orc_parse_key(const char* hex, double k[4], int* lasm) {
  size_t len = strlen(hex);
  uint8_t bytes[33];
  while (len > 0 && (hex[len - 1] == '\n' || hex[len - 1] == '\r' ||
                     hex[len - 1] == ' ' || hex[len - 1] == '\t'))
    --len;
  if (len != 66 && len != 50) return ORC_BAD_KEY;
  for (size_t i = 0; i < len / 2; ++i) {
    int hi = orc_nibble(hex[2 * i]), lo = orc_nibble(hex[2 * i + 1]);
    if (hi < 0 || lo < 0) return ORC_BAD_KEY;
    bytes[i] = (uint8_t)(hi << 4 | lo);
  }
  if (bytes[0] == 0x00 && len == 66) {
    *lasm = 0;
  } else if (bytes[0] == 0x01 && len == 50) {
    *lasm = 1;
  } else {
    return ORC_BAD_KEY; /* unknown tag, or a tag with the other map's length */
  }
  for (int j = 0; j < (*lasm ? 3 : 4); ++j) {
    uint64_t bits = 0;
    for (int i = 0; i < 8; ++i) bits |= (uint64_t)bytes[1 + 8 * j + i] << (8 * i);
    memcpy(&k[j], &bits, 8);
  }
  if (*lasm ? !orc_lasm_valid(k[0], k[1], k[2])
            : (!orc_plcm_valid(k[0], k[1]) || !orc_plcm_valid(k[2], k[3])))
    return ORC_BAD_KEY;
  return ORC_OK;
}

int orc_parse_plcm_key(const char* hex, double lanes[4]) {
  int lasm = 0;
  int st = orc_parse_key(hex, lanes, &lasm);
  return st ? st : (lasm ? ORC_BAD_KEY : ORC_OK);
}

/* src/keying.cpp:67-73 */
static double orc_rotate_half(double v) {
  v += 0.5;
  if (v >= 1.0) v -= 1.0;
  return v;
}

/* src/keying.cpp:61-65 */
static double orc_clamp_inside(double v, double lo, double hi) {
  if (v <= lo) return nextafter(lo, hi);
  if (v >= hi) return nextafter(hi, lo);
  return v;
}

/* src/keying.cpp:172-178 */
static double orc_next_unit(orc_prbg* coord) {
  uint8_t b[6];
  uint64_t v = 0;
  orc_prbg_fill(coord, b, 6);
  for (int i = 0; i < 6; ++i) v |= (uint64_t)b[i] << (8 * i);
  return (double)v / (double)((UINT64_C(1) << 48) - 1);
}

/* src/keying.cpp:209-218 */
static uint32_t orc_next_seed(orc_prbg* coord) {
  uint8_t b[4];
  orc_prbg_fill(coord, b, 4);
  uint64_t u = (uint64_t)b[0] | (uint64_t)b[1] << 8 | (uint64_t)b[2] << 16 |
               (uint64_t)b[3] << 24;
  return (uint32_t)(u % UINT64_C(0xFFFFFFFF)) + 1;
}

/* ---- L2: engine --------------------------------------------------------- */

/* src/engine.cpp:14-17 */
static uint32_t orc_euclid(int64_t v, uint32_t m) {
  int64_t r = v % (int64_t)m;
  return (uint32_t)(r < 0 ? r + (int64_t)m : r);
}

/* src/engine.cpp:19-22 */
int64_t orc_confusion_shift(uint32_t alpha, uint32_t side, uint32_t seed) {
  const double pi = 3.14159265358979323846;
  double angle = 2.0 * pi * (double)alpha / (double)side;
  return (int64_t)floor((double)seed * sin(angle));
}

typedef struct {
  uint32_t n, r;
  int lasm;
  orc_prbg coord;
  orc_prbg* workers;
  double* params; /* PLCM: n x (x0a, pa, x0b, pb); LASM: n x (x0a, y0a, mua, x0b, y0b, mub) */
  uint64_t seeds;
} orc_cipher;

/* src/engine.cpp:168-179, src/keying.cpp:164-207, 154-162 */
int orc_cipher_create(const char* key_hex, uint32_t n, uint32_t r,
                      orc_cipher** out) {
  double k[4];
  int st, lasm = 0;
  if (!key_hex || !out) return ORC_INVALID;
  st = orc_parse_key(key_hex, k, &lasm);
  if (st) return st;
  if (n == 0 || r == 0 || r > 255) return ORC_INVALID;
  orc_cipher* c = (orc_cipher*)calloc(1, sizeof *c);
  const size_t per = lasm ? 6 : 4;
  c->n = n;
  c->r = r;
  c->lasm = lasm;
  if (lasm) { /* keying.cpp:164-170: lane b = key rotated by one half */
    double b[3] = {orc_rotate_half(k[0]), orc_rotate_half(k[1]), k[2]};
    orc_lasm_init(&c->coord, k, b);
  } else {
    orc_prbg_init(&c->coord, k[0], k[1], k[2], k[3]);
  }
  c->workers = (orc_prbg*)calloc(n, sizeof(orc_prbg));
  c->params = (double*)calloc((size_t)n * per, sizeof(double));
  for (uint32_t i = 0; i < n; ++i) { /* keying.cpp:180-207 */
    double* q = c->params + per * (size_t)i;
    for (int lane = 0; lane < 2; ++lane) {
      if (lasm) {
        q[3 * lane + 0] = orc_clamp_inside(orc_next_unit(&c->coord), 0.0, 1.0);
        q[3 * lane + 1] = orc_clamp_inside(orc_next_unit(&c->coord), 0.0, 1.0);
        q[3 * lane + 2] = orc_clamp_inside(
            0.44 + orc_next_unit(&c->coord) * (0.93 - 0.44), 0.44, 0.93);
      } else {
        q[2 * lane + 0] = orc_clamp_inside(orc_next_unit(&c->coord), 0.0, 1.0);
        q[2 * lane + 1] =
            orc_clamp_inside(orc_next_unit(&c->coord) * 0.5, 0.0, 0.5);
      }
    }
  }
  for (uint32_t i = 0; i < n; ++i) {
    double* q = c->params + per * (size_t)i;
    if (lasm)
      orc_lasm_init(&c->workers[i], q, q + 3);
    else
      orc_prbg_init(&c->workers[i], q[0], q[1], q[2], q[3]);
  }
  *out = c;
  return ORC_OK;
}

void orc_cipher_destroy(orc_cipher* c) {
  if (!c) return;
  free(c->workers);
  free(c->params);
  free(c);
}

uint64_t orc_cipher_seeds_drawn(const orc_cipher* c) { return c->seeds; }

const double* orc_cipher_params(const orc_cipher* c) { return c->params; }

int orc_cipher_is_lasm(const orc_cipher* c) { return c->lasm; }

/* Draw `len` more keystream bytes of worker i (for PRBG kernel parity). */
void orc_cipher_worker_stream(orc_cipher* c, uint32_t i, uint8_t* out,
                              size_t len) {
  orc_prbg_fill(&c->workers[i], out, len);
}

uint32_t orc_cipher_next_seed(orc_cipher* c) {
  ++c->seeds;
  return orc_next_seed(&c->coord);
}

/* One frame, forward (src/engine.cpp:207-250) or inverse (252-284).
 * Scatter-form confusion exactly as confuse_rows (engine.cpp:32-47). */
static int orc_run_frame(orc_cipher* c, uint8_t* px, uint32_t side,
                         int decrypt) {
  if (!c || !px || side == 0) return ORC_INVALID; /* capi.cpp:169-171 */
  uint32_t seed = orc_cipher_next_seed(c);       /* engine.cpp:294/299 */
  if (side % c->n != 0) return ORC_MISMATCH;      /* engine.cpp:189-196 */
  const uint32_t n = c->n, r = c->r, w = side, rows = side / n;
  const size_t region = (size_t)rows * w * 3, bytes = (size_t)w * w * 3;
  uint8_t* ks = (uint8_t*)malloc((size_t)n * r * region);
  uint8_t* a = (uint8_t*)malloc(bytes);
  uint8_t* b = (uint8_t*)malloc(bytes);
  int64_t* shift = (int64_t*)malloc(sizeof(int64_t) * w);
  for (uint32_t i = 0; i < n; ++i) /* draw_streams, engine.cpp:198-205 */
    orc_prbg_fill(&c->workers[i], ks + (size_t)i * r * region, r * region);
  for (uint32_t al = 0; al < w; ++al) shift[al] = orc_confusion_shift(al, w, seed);
  memcpy(a, px, bytes);
  if (!decrypt) {
    for (uint32_t k = 0; k < r; ++k) {
      /* confusion: source (row, o) -> (alpha, beta), engine.cpp:32-47 */
      for (uint32_t row = 0; row < w; ++row)
        for (uint32_t o = 0; o < w; ++o) {
          uint32_t al = (row + o) % w;
          uint32_t be = orc_euclid((int64_t)o + shift[al], w);
          memcpy(b + ((size_t)al * w + be) * 3, a + ((size_t)row * w + o) * 3, 3);
        }
      { uint8_t* t = a; a = b; b = t; }
      /* diffusion per band, engine.cpp:66-73 (chain), 231-246 (seed byte) */
      for (uint32_t i = 0; i < n; ++i) {
        const uint8_t* s = ks + (size_t)i * r * region + (size_t)k * region;
        uint8_t prev = a[((size_t)((i + 1) % n) + 1) * region - 1];
        for (size_t j = 0; j < region; ++j) {
          uint8_t v = a[(size_t)i * region + j];
          prev = (uint8_t)(s[j] ^ (uint8_t)(v + s[j]) ^ prev); /* engine.hpp:32-34 */
          b[(size_t)i * region + j] = prev;
        }
      }
      { uint8_t* t = a; a = b; b = t; }
    }
  } else {
    for (uint32_t k = r; k-- > 0;) {
      /* inverse diffusion, engine.hpp:36-38, engine.cpp:75-83 */
      for (uint32_t i = 0; i < n; ++i) {
        const uint8_t* s = ks + (size_t)i * r * region + (size_t)k * region;
        const size_t base = (size_t)i * region;
        for (size_t j = 1; j < region; ++j)
          b[base + j] = (uint8_t)((s[j] ^ a[base + j] ^ a[base + j - 1]) - s[j]);
      }
      /* heads against the neighbour's recovered last byte, engine.cpp:271-276 */
      for (uint32_t i = 0; i < n; ++i) {
        const uint8_t* s = ks + (size_t)i * r * region + (size_t)k * region;
        uint8_t sd = b[((size_t)((i + 1) % n) + 1) * region - 1];
        b[(size_t)i * region] =
            (uint8_t)((s[0] ^ a[(size_t)i * region] ^ sd) - s[0]);
      }
      { uint8_t* t = a; a = b; b = t; }
      /* inverse confusion, engine.cpp:49-64 */
      for (uint32_t al = 0; al < w; ++al)
        for (uint32_t be = 0; be < w; ++be) {
          uint32_t o = orc_euclid((int64_t)be - shift[al], w);
          uint32_t row = orc_euclid((int64_t)al - (int64_t)o, w);
          memcpy(b + ((size_t)row * w + o) * 3, a + ((size_t)al * w + be) * 3, 3);
        }
      { uint8_t* t = a; a = b; b = t; }
    }
  }
  memcpy(px, a, bytes);
  free(ks);
  free(a);
  free(b);
  free(shift);
  return ORC_OK;
}

/* Engine::transform (src/engine.cpp:302-307 -> forward, 207-250): one seed,
 * the streams only when diffusion is on (rounds * region bytes per worker),
 * then per round the confusion half and / or the diffusion half.  states
 * (optional): rounds * side*side*3 bytes, the frame after each round (the
 * per_round callback, engine.cpp:247). */
int orc_cipher_transform_frame(orc_cipher* c, uint8_t* px, uint32_t side, uint32_t rounds,
                               int confusion, int diffusion, uint8_t* states) {
  if (!c || !px || side == 0) return ORC_INVALID;
  uint32_t seed = orc_cipher_next_seed(c);
  if (side % c->n != 0) return ORC_MISMATCH;
  const uint32_t n = c->n, w = side, rows = side / n;
  const size_t region = (size_t)rows * w * 3, bytes = (size_t)w * w * 3;
  uint8_t* ks = diffusion ? (uint8_t*)malloc((size_t)n * rounds * region + 1) : NULL;
  uint8_t* a = (uint8_t*)malloc(bytes);
  uint8_t* b = (uint8_t*)malloc(bytes);
  int64_t* shift = (int64_t*)malloc(sizeof(int64_t) * w);
  if (diffusion)
    for (uint32_t i = 0; i < n; ++i)
      orc_prbg_fill(&c->workers[i], ks + (size_t)i * rounds * region, rounds * region);
  if (confusion)
    for (uint32_t al = 0; al < w; ++al) shift[al] = orc_confusion_shift(al, w, seed);
  memcpy(a, px, bytes);
  for (uint32_t k = 0; k < rounds; ++k) {
    if (confusion) { /* engine.cpp:32-47 */
      for (uint32_t row = 0; row < w; ++row)
        for (uint32_t o = 0; o < w; ++o) {
          uint32_t al = (row + o) % w;
          uint32_t be = orc_euclid((int64_t)o + shift[al], w);
          memcpy(b + ((size_t)al * w + be) * 3, a + ((size_t)row * w + o) * 3, 3);
        }
      { uint8_t* t = a; a = b; b = t; }
    }
    if (diffusion) { /* engine.cpp:66-73, 231-246 */
      for (uint32_t i = 0; i < n; ++i) {
        const uint8_t* s = ks + (size_t)i * rounds * region + (size_t)k * region;
        uint8_t prev = a[((size_t)((i + 1) % n) + 1) * region - 1];
        for (size_t j = 0; j < region; ++j) {
          uint8_t v = a[(size_t)i * region + j];
          prev = (uint8_t)(s[j] ^ (uint8_t)(v + s[j]) ^ prev);
          b[(size_t)i * region + j] = prev;
        }
      }
      { uint8_t* t = a; a = b; b = t; }
    }
    if (states) memcpy(states + (size_t)k * bytes, a, bytes);
  }
  memcpy(px, a, bytes);
  free(ks);
  free(a);
  free(b);
  free(shift);
  return ORC_OK;
}

int orc_cipher_encrypt_frame(orc_cipher* c, uint8_t* px, uint32_t side) {
  return orc_run_frame(c, px, side, 0);
}

int orc_cipher_decrypt_frame(orc_cipher* c, uint8_t* px, uint32_t side) {
  return orc_run_frame(c, px, side, 1);
}

/* src/frame.cpp:19-26 */
uint32_t orc_padded_side(uint32_t w, uint32_t h, uint32_t n) {
  uint32_t m = w > h ? w : h;
  return (m + n - 1) / n * n;
}

/* engine.hpp:32-34 / 36-38, exported for the unit goldens */
uint8_t orc_diffuse_byte(uint8_t v, uint8_t b, uint8_t prev) {
  return (uint8_t)(b ^ (uint8_t)(v + b) ^ prev);
}
uint8_t orc_inverse_diffuse_byte(uint8_t c, uint8_t b, uint8_t prev) {
  return (uint8_t)((b ^ c ^ prev) - b);
}
