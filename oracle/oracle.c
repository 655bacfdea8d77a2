/* TEST INFRASTRUCTURE — CPU oracle (see oracle.h). Not part of the product.
 *
 * Repair semantics, restated from the reference:
 *   - predicates H(u)=(u&0xFC00)==0xD800, L(u)=(u&0xFC00)==0xDC00:
 *       SPEC.md:31-33 (SurrogateClass invariant); exhaustive pin
 *       proj/tests/test_surrogate.cpp:24-33.
 *   - or_fix_scalar: the sequential consuming scan, SPEC.md:67-77 and the
 *       pair-consumption rule SPEC.md:99; call sites
 *       proj/src/bitmask_kernel_avx512.cpp:67, proj/src/driver.cpp:116.
 *   - or_stencil: the per-unit formulation, proj/tests/test_helpers.hpp:42-53
 *       (reference_fix), checked equal to fix_scalar at
 *       proj/tests/test_surrogate.cpp:106.
 *   - or_unpaired_offsets: proj/tests/test_surrogate.cpp:122-128,
 *       proj/bindings/module.cpp:72-78.
 *   - or_ref_generate: proj/src/datagen.cpp:10-74 (mt19937_64 with the
 *       reference's own bounded-draw mapping; the RNG identity is a contract,
 *       proj/include/utf16mend/datagen.hpp:21-22). mt19937_64 itself is the
 *       standard published algorithm (Matsumoto & Nishimura, 64-bit variant).
 * Config generators (or_gen_*) are NEW (BASELINE.json configs 0-4 have no
 * reference generator); their spec is DESIGN.md §Inputs and the device
 * generator in paper_2601_06349_b200/csrc/datagen.cu is an independent
 * implementation checked bit-exact against this one.
 */
#include "oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define REPL 0xFFFDu

static inline int is_h(uint32_t u) { return (u & 0xFC00u) == 0xD800u; }
static inline int is_l(uint32_t u) { return (u & 0xFC00u) == 0xDC00u; }
static inline int is_sur(uint32_t u) { return (u & 0xF800u) == 0xD800u; }

void or_fix_scalar(uint16_t* out, const uint16_t* in, size_t n) {
  size_t i = 0;
  while (i < n) {
    const uint16_t u = in[i];
    if (is_h(u) && i + 1 < n && is_l(in[i + 1])) {
      const uint16_t l = in[i + 1];
      out[i] = u;
      out[i + 1] = l;
      i += 2;
    } else {
      out[i] = is_sur(u) ? (uint16_t)REPL : u;
      i += 1;
    }
  }
}

void or_stencil_halo(const uint16_t* in, size_t n, uint16_t* out, int32_t left, int32_t right) {
  for (size_t i = 0; i < n; i++) {
    const uint32_t u = in[i];
    const int prev_h = i >= 1 ? is_h(in[i - 1]) : (left >= 0 && is_h((uint32_t)left));
    const int next_l = i + 1 < n ? is_l(in[i + 1]) : (right >= 0 && is_l((uint32_t)right));
    uint16_t r = (uint16_t)u;
    if (is_h(u) && !next_l) r = (uint16_t)REPL;
    if (is_l(u) && !prev_h) r = (uint16_t)REPL;
    out[i] = r;
  }
}

void or_stencil(const uint16_t* in, size_t n, uint16_t* out) { or_stencil_halo(in, n, out, -1, -1); }

int or_fix_batched(const uint16_t* in, const int64_t* offsets, size_t num_strings, uint16_t* out) {
  for (size_t s = 0; s < num_strings; s++) {
    const int64_t a = offsets[s], b = offsets[s + 1];
    if (a < 0 || b < a) return -1;
    or_fix_scalar(out + a, in + a, (size_t)(b - a));
  }
  return 0;
}

size_t or_unpaired_offsets(const uint16_t* in, size_t n, size_t limit, uint64_t* out) {
  size_t k = 0, i = 0;
  while (i < n && k < limit) {
    if (is_h(in[i]) && i + 1 < n && is_l(in[i + 1])) {
      i += 2;
      continue;
    }
    if (is_sur(in[i])) {
      if (out) out[k] = i;
      k++;
    }
    i += 1;
  }
  return k;
}

int or_is_well_formed(const uint16_t* in, size_t n) { return or_unpaired_offsets(in, n, 1, NULL) == 0; }

typedef struct {
  const uint16_t* in;
  uint16_t* out;
  size_t n, a, b;
} mt_job;

static void* mt_worker(void* p) {
  const mt_job* j = (const mt_job*)p;
  const int32_t left = j->a > 0 ? (int32_t)j->in[j->a - 1] : -1;
  const int32_t right = j->b < j->n ? (int32_t)j->in[j->b] : -1;
  or_stencil_halo(j->in + j->a, j->b - j->a, j->out + j->a, left, right);
  return NULL;
}

void or_stencil_mt(const uint16_t* in, size_t n, uint16_t* out, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (n < (size_t)threads * 4096) threads = 1;
  pthread_t tid[256];
  mt_job jobs[256];
  for (int t = 0; t < threads; t++) {
    jobs[t].in = in;
    jobs[t].out = out;
    jobs[t].n = n;
    jobs[t].a = n * (size_t)t / (size_t)threads;
    jobs[t].b = n * (size_t)(t + 1) / (size_t)threads;
  }
  for (int t = 1; t < threads; t++) pthread_create(&tid[t], NULL, mt_worker, &jobs[t]);
  mt_worker(&jobs[0]);
  for (int t = 1; t < threads; t++) pthread_join(tid[t], NULL);
}

/* ---- mt19937_64 (standard algorithm) + reference sampler --------------- */
#define MT_NN 312
#define MT_MM 156
typedef struct {
  uint64_t mt[MT_NN];
  int idx;
} mt64;

static void mt64_seed(mt64* m, uint64_t seed) {
  m->mt[0] = seed;
  for (int i = 1; i < MT_NN; i++)
    m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
  m->idx = MT_NN;
}

static uint64_t mt64_next(mt64* m) {
  static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (m->idx >= MT_NN) {
    int i;
    uint64_t x;
    for (i = 0; i < MT_NN - MT_MM; i++) {
      x = (m->mt[i] & UM) | (m->mt[i + 1] & LM);
      m->mt[i] = m->mt[i + MT_MM] ^ (x >> 1) ^ mag[x & 1ULL];
    }
    for (; i < MT_NN - 1; i++) {
      x = (m->mt[i] & UM) | (m->mt[i + 1] & LM);
      m->mt[i] = m->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ mag[x & 1ULL];
    }
    x = (m->mt[MT_NN - 1] & UM) | (m->mt[0] & LM);
    m->mt[MT_NN - 1] = m->mt[MT_MM - 1] ^ (x >> 1) ^ mag[x & 1ULL];
    m->idx = 0;
  }
  uint64_t x = m->mt[m->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* proj/src/datagen.cpp:19-21 */
static uint32_t ref_below(mt64* m, uint32_t n) {
  return (uint32_t)(((unsigned __int128)mt64_next(m) * n) >> 64);
}
/* proj/src/datagen.cpp:23-27 */
static int ref_chance(mt64* m, double p) {
  if (p <= 0.0) return 0;
  if (p >= 1.0) return 1;
  return mt64_next(m) < (uint64_t)(p * 18446744073709551616.0);
}
/* proj/src/datagen.cpp:33-40 */
static uint16_t ref_filler(mt64* m) {
  const uint32_t low_span = 0xD7FF, high_span = 0xFFFD - 0xE000 + 1;
  const uint32_t r = ref_below(m, low_span + high_span);
  return (uint16_t)(r < low_span ? 1 + r : 0xE000 + (r - low_span));
}

/* proj/src/datagen.cpp:44-74 */
void or_ref_generate(size_t n, double pair_pct, double mismatch_pct, uint64_t seed, uint16_t* out) {
  mt64* m = (mt64*)malloc(sizeof(mt64));
  mt64_seed(m, seed);
  const double q = pair_pct / (2.0 - pair_pct);
  size_t k = 0;
  while (k < n) {
    if (ref_chance(m, q)) {
      if (k + 2 <= n) {
        out[k++] = (uint16_t)(0xD800 + ref_below(m, 0x400));
        out[k++] = (uint16_t)(0xDC00 + ref_below(m, 0x400));
      } else {
        out[k++] = ref_filler(m);
      }
    } else if (ref_chance(m, mismatch_pct)) {
      const uint32_t base = ref_chance(m, 0.5) ? 0xD800 : 0xDC00;
      out[k++] = (uint16_t)(base + ref_below(m, 0x400));
    } else {
      out[k++] = ref_filler(m);
    }
  }
  free(m);
}

/* ---- counter-based generators (spec: DESIGN.md §Inputs) ----------------- */
#define GEN_CHUNK 4096u
#define GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t or_rng_key(uint64_t seed, uint64_t stream, uint64_t index) {
  return mix64(seed * GOLDEN + stream * 0xD1B54A32D192ED03ULL + index * 0x8CB92BA72F3D8DD7ULL);
}

uint64_t or_rng_next(uint64_t* s) {
  *s += GOLDEN;
  return mix64(*s);
}

uint32_t or_rng_below(uint64_t* s, uint32_t bound) {
  return (uint32_t)(((unsigned __int128)or_rng_next(s) * bound) >> 64);
}

/* BMP non-surrogate from 0x0080: [0x0080,0xD7FF] u [0xE000,0xFFFF] */
static uint16_t bmp80(uint64_t* s) {
  const uint32_t r = or_rng_below(s, 0xD780u + 0x2000u);
  return (uint16_t)(r < 0xD780u ? 0x80u + r : 0xE000u + (r - 0xD780u));
}
/* BMP non-surrogate from 0x0020: [0x0020,0xD7FF] u [0xE000,0xFFFF] */
static uint16_t bmp20(uint64_t* s) {
  const uint32_t r = or_rng_below(s, 0xD7E0u + 0x2000u);
  return (uint16_t)(r < 0xD7E0u ? 0x20u + r : 0xE000u + (r - 0xD7E0u));
}

/* Config-0 character at pos with `room` slots left in the chunk; returns units written. */
static int c0_char(uint64_t* s, uint16_t* dst, uint64_t room, int allow_lone) {
  const uint32_t d = or_rng_below(s, allow_lone ? 1000u : 990u);
  if (d < 700u) {
    dst[0] = (uint16_t)(0x20u + or_rng_below(s, 95u));
    return 1;
  }
  if (d < 940u) {
    dst[0] = bmp80(s);
    return 1;
  }
  if (d < 990u) {
    if (room >= 2) {
      dst[0] = (uint16_t)(0xD800u + or_rng_below(s, 1024u));
      dst[1] = (uint16_t)(0xDC00u + or_rng_below(s, 1024u));
      return 2;
    }
    dst[0] = bmp80(s);
    return 1;
  }
  if (d < 995u) {
    dst[0] = (uint16_t)(0xD800u + or_rng_below(s, 1024u));
    return 1;
  }
  dst[0] = (uint16_t)(0xDC00u + or_rng_below(s, 1024u));
  return 1;
}

static int c2_char(uint64_t* s, uint16_t* dst, uint64_t room) {
  const uint32_t d = or_rng_below(s, 100000u);
  if (d < 5u) {
    dst[0] = (uint16_t)(0xD800u + or_rng_below(s, 1024u));
    return 1;
  }
  if (d < 10u) {
    dst[0] = (uint16_t)(0xDC00u + or_rng_below(s, 1024u));
    return 1;
  }
  if (d < 50005u && room >= 2) {
    const uint32_t cp = 0x1F300u + or_rng_below(s, 0x800u) - 0x10000u;
    dst[0] = (uint16_t)(0xD800u + (cp >> 10));
    dst[1] = (uint16_t)(0xDC00u + (cp & 0x3FFu));
    return 2;
  }
  dst[0] = bmp20(s);
  return 1;
}

/* Base content of one 4096-unit chunk c of a logical buffer of `total` units. */
static void gen_chunk(int cfg, uint64_t seed, uint64_t total, uint64_t c, uint16_t* chunk) {
  const uint64_t a = c * GEN_CHUNK;
  const uint64_t len = total - a < GEN_CHUNK ? total - a : GEN_CHUNK;
  uint64_t s = or_rng_key(seed, 1, c);
  uint64_t k = 0;
  if (cfg == 1) {
    while (k < len) {
      const uint64_t v = or_rng_next(&s);
      for (int j = 0; j < 4 && k < len; j++, k++) chunk[k] = (uint16_t)(v >> (16 * j));
    }
    return;
  }
  while (k < len) {
    if (cfg == 2)
      k += (uint64_t)c2_char(&s, chunk + k, len - k);
    else
      k += (uint64_t)c0_char(&s, chunk + k, len - k, 1);
  }
}

/* Adversarial pattern `kind` at boundary b: writes up to 3 units (b-1, b, b+1).
 * vals are drawn from key(seed, stream, tag). Returns count, fills pos/val. */
static int boundary_pattern(uint64_t seed, uint64_t stream, uint64_t tag, uint64_t b, int kind,
                            uint64_t* pos, uint16_t* val) {
  uint64_t s = or_rng_key(seed, stream, tag);
  const uint16_t h = (uint16_t)(0xD800u + or_rng_below(&s, 1024u));
  const uint16_t l = (uint16_t)(0xDC00u + or_rng_below(&s, 1024u));
  const uint16_t h2 = (uint16_t)(0xD800u + or_rng_below(&s, 1024u));
  const uint16_t l2 = (uint16_t)(0xDC00u + or_rng_below(&s, 1024u));
  pos[0] = b - 1;
  pos[1] = b;
  pos[2] = b + 1;
  switch (kind) {
    case 0: val[0] = h; val[1] = l; return 2;          /* H|L straddling pair  */
    case 1: val[0] = h; val[1] = 0x0041; return 2;     /* H|x lone high        */
    case 2: val[0] = 0x0042; val[1] = l; return 2;     /* x|L lone low         */
    case 3: val[0] = h; val[1] = h2; val[2] = l; return 3; /* H|H L            */
    default: val[0] = l; val[1] = l2; return 2;        /* L|L                  */
  }
}

#define C2_TILE 256u
#define C4_REGION (1u << 20)

int or_gen_config(int cfg, uint64_t seed, uint64_t total, uint64_t shard_len, uint64_t first,
                  uint64_t count, uint16_t* out) {
  if (cfg != 0 && cfg != 1 && cfg != 2 && cfg != 4) return -1;
  if (first + count > total) return -1;
  if (count == 0) return 0;
  const uint64_t end = first + count;
  uint16_t chunk[GEN_CHUNK];
  for (uint64_t c = first / GEN_CHUNK; c * GEN_CHUNK < end; c++) {
    gen_chunk(cfg, seed, total, c, chunk);
    const uint64_t a = c * GEN_CHUNK;
    const uint64_t lo = a > first ? a : first;
    const uint64_t hi = a + GEN_CHUNK < end ? a + GEN_CHUNK : end;
    memcpy(out + (lo - first), chunk + (lo - a), (size_t)(hi - lo) * 2);
  }
  uint64_t pos[3];
  uint16_t val[3];
  if (cfg == 2) {
    /* every multiple of 256 units (subsumes 4 KiB = 2048 and 64 KiB = 32768) */
    uint64_t t0 = first / C2_TILE;
    if (t0 < 1) t0 = 1;
    for (uint64_t t = t0; t * C2_TILE <= end; t++) {
      const uint64_t b = t * C2_TILE;
      const int m = boundary_pattern(seed, 2, t, b, (int)(t % 5), pos, val);
      for (int j = 0; j < m; j++)
        if (pos[j] >= first && pos[j] < end && pos[j] < total) out[pos[j] - first] = val[j];
    }
  }
  if (cfg == 4) {
    for (uint64_t r = first / C4_REGION; r * C4_REGION < end; r++) {
      uint64_t s = or_rng_key(seed, 5, r);
      const uint32_t d = or_rng_below(&s, 100u);
      if (d < 90u) continue;
      const uint64_t ra = r * C4_REGION;
      const uint64_t rlen = total - ra < C4_REGION ? total - ra : C4_REGION;
      const uint64_t len = 1u + or_rng_below(&s, (uint32_t)rlen);
      const uint64_t st = ra + or_rng_below(&s, (uint32_t)(rlen - len + 1));
      const uint32_t phase = or_rng_below(&s, 2u);
      const uint64_t lo = st > first ? st : first;
      const uint64_t hi = st + len < end ? st + len : end;
      for (uint64_t p = lo; p < hi; p++) {
        uint16_t v = 0xD800;
        if (d >= 95u) v = ((p - st + phase) & 1u) ? 0xDC00 : 0xD800;
        out[p - first] = v;
      }
    }
    if (shard_len > 0) {
      for (uint64_t k = 1; k * shard_len < total; k++) {
        const uint64_t b = k * shard_len;
        const int m = boundary_pattern(seed, 6, k, b, (int)(k % 5), pos, val);
        for (int j = 0; j < m; j++)
          if (pos[j] >= first && pos[j] < end && pos[j] < total) out[pos[j] - first] = val[j];
      }
    }
  }
  return 0;
}

void or_gen_c3_offsets(uint64_t seed, size_t num_strings, int64_t* offsets) {
  offsets[0] = 0;
  for (size_t i = 0; i < num_strings; i++) {
    uint64_t s = or_rng_key(seed, 3, i);
    const uint32_t e = or_rng_below(&s, 12u);
    const uint32_t len = (1u << e) + or_rng_below(&s, 1u << e);
    offsets[i + 1] = offsets[i] + (int64_t)len;
  }
}

void or_gen_c3_content(uint64_t seed, size_t num_strings, const int64_t* offsets, uint16_t* out) {
  for (size_t i = 0; i < num_strings; i++) {
    uint16_t* x = out + offsets[i];
    const uint64_t len = (uint64_t)(offsets[i + 1] - offsets[i]);
    uint64_t s = or_rng_key(seed, 4, i);
    const int has_err = or_rng_below(&s, 100u) < 20u;
    uint64_t k = 0;
    while (k < len) k += (uint64_t)c0_char(&s, x + k, len - k, 0);
    if (has_err) {
      const uint32_t m = 1u + or_rng_below(&s, 8u);
      for (uint32_t j = 0; j < m; j++) {
        const uint64_t p = or_rng_below(&s, (uint32_t)len);
        const uint32_t hl = or_rng_below(&s, 2u);
        x[p] = (uint16_t)((hl ? 0xD800u : 0xDC00u) + or_rng_below(&s, 1024u));
      }
    }
    if (or_rng_below(&s, 100u) < 3u) x[0] = (uint16_t)(0xDC00u + or_rng_below(&s, 1024u));
    if (or_rng_below(&s, 100u) < 3u) x[len - 1] = (uint16_t)(0xD800u + or_rng_below(&s, 1024u));
  }
}
