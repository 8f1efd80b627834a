/*
 * go_world.c -- oracle restatement of rng.py, perlin.py and worldgen.py.
 * TEST INFRASTRUCTURE ONLY (see gr_oracle.h).
 *
 * Every function names the reference lines it restates.  Float semantics
 * follow numpy: f32 arithmetic is separately rounded (-ffp-contract=off),
 * comparisons against Python float literals happen in f32 (NEP 50), the
 * overworld noise uses numpy's own float32 SIMD sin/cos, the cave noise uses
 * libm double cos/sin exactly like numpy's float64 path.
 */
#include "gr_oracle.h"
#include "go_tables.h"

#include <math.h>
#include <string.h>
#include <stdlib.h>

/* ---------------------------------------------------------------- rng.py */

#define GOLDEN64 0x9E3779B97F4A7C15ULL

/* rng.py:23-27 */
uint64_t go_mix(uint64_t z) {
  z += GOLDEN64;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* rng.py:30-32 */
uint64_t go_hash2(uint64_t key, uint64_t n) { return go_mix(key ^ go_mix(n)); }

/* rng.py:75-80 */
uint32_t go_vmix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  return x ^ (x >> 16);
}

/* rng.py:83-88 */
float go_vuniform32(uint32_t key, uint32_t n) {
  uint32_t h = go_vmix32(key ^ (n * 0x9E3779B9u + 0x9E3779B9u));
  return (float)(h >> 8) * (1.0f / 16777216.0f);
}

/* rng.py:58-61 */
double go_vuniform(uint64_t key, uint64_t n) {
  return (double)(go_hash2(key, n) >> 11) * (1.0 / 9007199254740992.0);
}

/* RngStream (rng.py:91-141) as a (key, counter) pair */
typedef struct { uint64_t key, ctr; } stream_t;

static stream_t st_make(uint64_t seed) { stream_t s = {go_mix(seed), 0}; return s; }
static stream_t st_raw(uint64_t key) { stream_t s = {key, 0}; return s; }
/* rng.py:109-112 */
static stream_t st_split(stream_t p, uint64_t id) {
  stream_t s = {go_hash2(p.key, go_hash2(id, p.ctr)), 0};
  return s;
}
/* rng.py:115-116 */
static uint64_t st_next(stream_t *s) { return go_hash2(s->key, s->ctr++); }
/* rng.py:127-132 */
static int64_t st_randint(stream_t *s, int64_t lo, int64_t hi) {
  uint64_t raw = st_next(s);
  return lo + (int64_t)(raw % (uint64_t)(hi - lo));
}
/* rng.py:119-124 (lo=0, hi=1) */
static double st_uniform01(stream_t *s) {
  uint64_t raw = st_next(s);
  double u = (double)(raw >> 11) * (1.0 / 9007199254740992.0);
  return 0.0 + (1.0 - 0.0) * u;
}
/* rng.py:135-140 */
static void st_uniform_array(stream_t *s, int n, double *out) {
  for (int i = 0; i < n; ++i) out[i] = go_vuniform(s->key, s->ctr + (uint64_t)i);
  s->ctr += (uint64_t)n;
}

/* ------------------------------------------- numpy float32 sin/cos (H1) */
/* numpy loops_trigonometric.dispatch: Cody-Waite reduction by pi/2 with the
 * quadrant rounded to nearest, then minimax polynomials; all muladds are
 * fused. */
static float np_sincosf(float x, int is_cos) {
  float q = x * 0x1.45f306p-1f;
  q = rintf(q);
  float r = fmaf(q, -0x1.921fb0p+0f, x);
  r = fmaf(q, -0x1.5110b4p-22f, r);
  r = fmaf(q, -0x1.846988p-48f, r);
  float r2 = r * r;
  int iq = (int)q + (is_cos ? 1 : 0);
  float c = fmaf(0x1.98e616p-16f, r2, -0x1.6c06dcp-10f);
  c = fmaf(c, r2, 0x1.55553cp-5f);
  c = fmaf(c, r2, -0x1.000000p-1f);
  c = fmaf(c, r2, 0x1.000000p+0f);
  float sn = fmaf(0x1.7d3bbcp-19f, r2, -0x1.a06bbap-13f);
  sn = fmaf(sn, r2, 0x1.11119ap-07f);
  sn = fmaf(sn, r2, -0x1.555556p-03f);
  sn = sn * r2;
  sn = fmaf(sn, r, r);
  float v = ((iq & 1) == 0) ? sn : c;
  if (iq & 2) v = -v;
  return v;
}
float go_np_sinf(float x) { return np_sincosf(x, 0); }
float go_np_cosf(float x) { return np_sincosf(x, 1); }

/* np.argsort of 6 float32 (worldgen.py:647-649) as numpy >= 2 runs it on
   AVX-512 hosts: x86-simd-sort's key/index bitonic network over one 8-lane
   register (lanes 6-7 = +inf, inert), compare-exchange on a strict '>' with
   each lane keeping its index on ties -- 15 comparators on the live lanes.
   Not stable; pinned against np.argsort on all 6^6 value patterns. */
void go_np_argsort6(const float *v, uint8_t *idx) {
  static const int P[15][2] = {{0, 1}, {2, 3}, {4, 5}, {0, 3}, {1, 2}, {0, 1}, {2, 3}, {4, 5},
                               {2, 5}, {3, 4}, {0, 2}, {1, 3}, {0, 1}, {2, 3}, {4, 5}};
  float k[6];
  for (int i = 0; i < 6; ++i) { k[i] = v[i]; idx[i] = (uint8_t)i; }
  for (int c = 0; c < 15; ++c) {
    int a = P[c][0], b = P[c][1];
    if (k[a] > k[b]) {
      float tk = k[a]; k[a] = k[b]; k[b] = tk;
      uint8_t ti = idx[a]; idx[a] = idx[b]; idx[b] = ti;
    }
  }
}

/* -------------------------------------------------------------- perlin.py */

/* perlin.py:22-23, evaluated left to right in the working precision */
static float fadef(float t) { return ((t * t) * t) * ((t * ((t * 6.0f) - 15.0f)) + 10.0f); }
static double fade_d(double t) { return ((t * t) * t) * ((t * ((t * 6.0) - 15.0)) + 10.0); }

/* perlin.py:54-92, float32: angles (res+1)x(res+1), square dims */
static void octave_f32(int h, int w, const float *ang, int res, float *out) {
  int dr = h / res, dc = w / res;
  float gx[17 * 17], gy[17 * 17];
  for (int i = 0; i < (res + 1) * (res + 1); ++i) {
    gx[i] = go_np_cosf(ang[i]);
    gy[i] = go_np_sinf(ang[i]);
  }
  /* perlin.py:36-51 */
  float a1[64], a2[64], a3[64], a4[64], b0[64], b1[64], b2[64], b3[64];
  const float one = 1.0f, root2 = (float)1.4142135623730951;
  for (int i = 0; i < dr; ++i) {
    float fr = (float)i / (float)dr;
    float u = fadef(fr);
    a1[i] = one - u;
    a2[i] = (one - u) * fr;
    a3[i] = u;
    a4[i] = u * (fr - one);
  }
  for (int j = 0; j < dc; ++j) {
    float fc = (float)j / (float)dc;
    float v = fadef(fc);
    b0[j] = ((one - v) * fc) * root2;
    b1[j] = (one - v) * root2;
    b2[j] = (v * (fc - one)) * root2;
    b3[j] = v * root2;
  }
  int n = res + 1;
  for (int R = 0; R < res; ++R)
    for (int i = 0; i < dr; ++i)
      for (int C = 0; C < res; ++C) {
        float t0 = gx[R * n + C] * a1[i] + gx[(R + 1) * n + C] * a3[i];
        float t1 = gy[R * n + C] * a2[i] + gy[(R + 1) * n + C] * a4[i];
        float t2 = gx[R * n + C + 1] * a1[i] + gx[(R + 1) * n + C + 1] * a3[i];
        float t3 = gy[R * n + C + 1] * a2[i] + gy[(R + 1) * n + C + 1] * a4[i];
        for (int j = 0; j < dc; ++j) {
          float p0 = t0 * b0[j], p1 = t1 * b1[j], p2 = t2 * b2[j], p3 = t3 * b3[j];
          out[(R * dr + i) * w + C * dc + j] = ((p0 + p1) + p2) + p3;
        }
      }
}

/* same octave in float64 (caves): theta = f64(angle f32), libm cos/sin */
static void octave_f64(int h, int w, const float *ang, int res, double *out) {
  int dr = h / res, dc = w / res;
  double gx[17 * 17], gy[17 * 17];
  for (int i = 0; i < (res + 1) * (res + 1); ++i) {
    gx[i] = cos((double)ang[i]);
    gy[i] = sin((double)ang[i]);
  }
  double a1[64], a2[64], a3[64], a4[64], b0[64], b1[64], b2[64], b3[64];
  const double one = 1.0, root2 = 1.4142135623730951;
  for (int i = 0; i < dr; ++i) {
    double fr = (double)i / (double)dr;
    double u = fade_d(fr);
    a1[i] = one - u; a2[i] = (one - u) * fr; a3[i] = u; a4[i] = u * (fr - one);
  }
  for (int j = 0; j < dc; ++j) {
    double fc = (double)j / (double)dc;
    double v = fade_d(fc);
    b0[j] = ((one - v) * fc) * root2; b1[j] = (one - v) * root2;
    b2[j] = (v * (fc - one)) * root2; b3[j] = v * root2;
  }
  int n = res + 1;
  for (int R = 0; R < res; ++R)
    for (int i = 0; i < dr; ++i)
      for (int C = 0; C < res; ++C) {
        double t0 = gx[R * n + C] * a1[i] + gx[(R + 1) * n + C] * a3[i];
        double t1 = gy[R * n + C] * a2[i] + gy[(R + 1) * n + C] * a4[i];
        double t2 = gx[R * n + C + 1] * a1[i] + gx[(R + 1) * n + C + 1] * a3[i];
        double t3 = gy[R * n + C + 1] * a2[i] + gy[(R + 1) * n + C + 1] * a4[i];
        for (int j = 0; j < dc; ++j) {
          double p0 = t0 * b0[j], p1 = t1 * b1[j], p2 = t2 * b2[j], p3 = t3 * b3[j];
          out[(R * dr + i) * w + C * dc + j] = ((p0 + p1) + p2) + p3;
        }
      }
}

/* perlin.py:95-114 with CAVE_OCTAVES [(4,1.0),(8,0.5)], dtype float64 */
void go_perlin_cave(const float *a25, const float *a81, int h, int w, double *field) {
  double *o2 = (double *)malloc(sizeof(double) * h * w);
  octave_f64(h, w, a25, 4, field);
  octave_f64(h, w, a81, 8, o2);
  for (int i = 0; i < h * w; ++i) {
    double total = 1.0 * field[i];
    total = total + 0.5 * o2[i];
    field[i] = total / 1.5;
  }
  free(o2);
}

/* worldgen.py:181-196 (angles252 = 3x3 | 9x9 | 9x9 | 9x9) */
void go_overworld_fields(const float *angles252, int h, int w,
                         float *height, float *forest, float *special) {
  float *fine = (float *)malloc(sizeof(float) * h * w);
  octave_f32(h, w, angles252, 2, height);
  octave_f32(h, w, angles252 + 9, 8, fine);
  for (int i = 0; i < h * w; ++i)
    height[i] = (height[i] + 0.35f * fine[i]) / 1.35f;
  octave_f32(h, w, angles252 + 90, 8, forest);
  octave_f32(h, w, angles252 + 171, 8, special);
  free(fine);
}

/* ----------------------------------------------------------- worldgen.py */

/* worldgen.py:75-87 */
void go_level_angles(uint64_t seed, float *angles252, uint64_t *floor_seeds9) {
  stream_t base = st_make(seed);
  stream_t s1 = st_split(base, 1);
  double flat[252];
  st_uniform_array(&s1, 252, flat);
  for (int i = 0; i < 252; ++i) {
    double t = flat[i] * 2.0;
    t = t * 3.141592653589793;
    angles252[i] = (float)t;
  }
  for (int f = 0; f < 9; ++f) floor_seeds9[f] = st_split(base, 100 + f).key;
}

typedef struct { int h, w; } dims_t;

/* worldgen.py:124-131 */
static void tile_uniform(uint64_t key, int n, uint64_t salt, float *u) {
  uint32_t k32 = (uint32_t)(go_hash2(key, salt) & 0xFFFFFFFFu);
  for (int i = 0; i < n; ++i) u[i] = go_vuniform32(k32, (uint32_t)i);
}

static int cheb(int r0, int c0, int r1, int c1) {
  int a = abs(r0 - r1), b = abs(c0 - c1);
  return a > b ? a : b;
}

/* worldgen.py:146-156: argmax(where(mask, u, -1)) -> flat idx or -1 */
static int pick_tile_f32(int n, const uint8_t *mask, const float *u) {
  int best = -1;
  float bv = 0;
  for (int i = 0; i < n; ++i)
    if (mask[i] && (best < 0 || u[i] > bv)) { best = i; bv = u[i]; }
  return best;
}
static int pick_tile_f64(int n, const uint8_t *mask, const double *u) {
  int best = -1;
  double bv = 0;
  for (int i = 0; i < n; ++i)
    if (mask[i] && (best < 0 || u[i] > bv)) { best = i; bv = u[i]; }
  return best;
}

/* worldgen.py:159-171 */
static void carve_line(uint8_t *blk, int w, int r, int c, int tr, int tc, uint8_t fill) {
  while (c != tc) { c += tc > c ? 1 : -1; blk[r * w + c] = fill; }
  while (r != tr) { r += tr > r ? 1 : -1; blk[r * w + c] = fill; }
}

#define DEGENERATE (-1)

/* worldgen.py:340-364 for a float32 score (overworld / realm).
 * score_sign: +1 uses score, -1 uses -score.  Returns DEGENERATE or 0. */
static int ensure_block_f32(uint8_t *blk, int n, uint8_t block, const float *hsrc,
                            int neg, int low, const uint8_t *near) {
  for (int i = 0; i < n; ++i) if (blk[i] == block) return 0;
  /* score = -height if low else height ; with hsrc possibly pre-negated */
  int sneg = neg ^ (low ? 1 : 0);
#define SCORE(i) (sneg ? -hsrc[i] : hsrc[i])
  if (!low) {
    int best = -1; float bv = 0;
    for (int i = 0; i < n; ++i)
      if (blk[i] == B_STONE && (best < 0 || SCORE(i) > bv)) { best = i; bv = SCORE(i); }
    if (best >= 0) { blk[best] = block; return 0; }
  }
  int use_near = 0;
  if (near) for (int i = 0; i < n; ++i) if (blk[i] == B_GRASS && near[i]) { use_near = 1; break; }
  int any = 0;
  for (int i = 0; i < n; ++i) if (blk[i] == B_GRASS && (!use_near || near[i])) { any = 1; break; }
  int best = -1; float bv = 0;
  if (any) {
    for (int i = 0; i < n; ++i)
      if (blk[i] == B_GRASS && (!use_near || near[i]) && (best < 0 || SCORE(i) > bv)) { best = i; bv = SCORE(i); }
  } else {
    for (int i = 0; i < n; ++i)
      if ((blk[i] == B_GRASS || blk[i] == B_TREE) && (best < 0 || SCORE(i) > bv)) { best = i; bv = SCORE(i); }
  }
#undef SCORE
  if (best < 0) return DEGENERATE;
  blk[best] = block;
  return 0;
}

/* f64 score variant used by caves: score = -field, low=False, near=None */
static int ensure_block_cave(uint8_t *blk, int n, uint8_t block, const double *field) {
  for (int i = 0; i < n; ++i) if (blk[i] == block) return 0;
  int best = -1; double bv = 0;
  for (int i = 0; i < n; ++i)
    if (blk[i] == B_STONE && (best < 0 || -field[i] > bv)) { best = i; bv = -field[i]; }
  if (best >= 0) { blk[best] = block; return 0; }
  for (int i = 0; i < n; ++i)
    if ((blk[i] == B_GRASS || blk[i] == B_TREE) && (best < 0 || -field[i] > bv)) { best = i; bv = -field[i]; }
  if (best < 0) return DEGENERATE;
  blk[best] = block;
  return 0;
}

/* worldgen.py:222-244 */
static uint8_t overworld_tile(float h, float forest, float special, float u) {
  uint8_t b = B_GRASS;
  if (h < -0.28f) b = B_WATER;
  if (h >= -0.28f && h < -0.22f) b = B_SAND;
  int mountain = h > 0.28f;
  if (mountain) b = B_STONE;
  if (b == B_GRASS && forest > 0.18f && u < 0.55f) b = B_TREE;
  if (mountain && fabsf(special) < 0.06f) b = B_PATH;
  if (mountain && special < -0.5f) b = B_LAVA;
  if (b == B_STONE) {
    if (u < 0.035f) b = B_COAL;
    if (u >= 0.94f && h > 0.34f) b = B_IRON;
    if (u >= 0.91f && u < 0.94f && h > 0.45f) b = B_DIAMOND;
  }
  return b;
}

typedef struct {
  uint8_t *blocks, *items;
  int spawn_r, spawn_c;
  int ld_r, ld_c, lu_r, lu_c; /* -1 when absent */
} floor_out;

/* worldgen.py:247-327 (the non-batched path; generate_worlds' batched
 * census/spawn is bit-identical to it) */
static int gen_overworld(const float *height, const float *forest, const float *special,
                         uint64_t seed0, int h, int w, int extended, int attempt,
                         floor_out *o) {
  int n = h * w;
  uint64_t key = go_hash2(seed0, (uint64_t)attempt);
  float *u = (float *)malloc(sizeof(float) * n);
  uint8_t *near = (uint8_t *)malloc(n);
  uint8_t *mask = (uint8_t *)malloc(n);
  int rc = 0;
  tile_uniform(key, n, 1, u);
  uint8_t *blk = o->blocks;
  for (int i = 0; i < n; ++i) blk[i] = overworld_tile(height[i], forest[i], special[i], u[i]);
  /* spawn: argmin of where(walk, center chebyshev f32, 1e9) */
  int spawn = -1, bestd = 0;
  for (int i = 0; i < n; ++i) {
    if (!WALKABLE_T[blk[i]]) continue;
    int d = cheb(i / w, i % w, h / 2, w / 2);
    if (spawn < 0 || d < bestd) { spawn = i; bestd = d; }
  }
  if (spawn < 0) { rc = DEGENERATE; goto out; }
  int sr = spawn / w, sc = spawn % w;
  blk[spawn] = B_GRASS;
  for (int i = 0; i < n; ++i) near[i] = cheb(i / w, i % w, sr, sc) <= 8 && i != spawn;
  /* census after the spawn fix (worldgen.py:289-294) */
  int census[64] = {0};
  for (int i = 0; i < n; ++i) census[blk[i]] = 1;
  int fixed_any = 0;
  static const struct { uint8_t b; int low; } order[6] = {
      {B_COAL, 0}, {B_IRON, 0}, {B_DIAMOND, 0}, {B_LAVA, 0}, {B_WATER, 1}, {B_SAND, 1}};
  for (int k = 0; k < 6; ++k) {
    if (!census[order[k].b]) {
      if (ensure_block_f32(blk, n, order[k].b, height, 0, order[k].low, near)) { rc = DEGENERATE; goto out; }
      fixed_any = 1;
    }
  }
  int stone_now = 0;
  for (int i = 0; i < n; ++i) if (blk[i] == B_STONE) { stone_now = 1; break; }
  if (!census[B_STONE] || (fixed_any && !stone_now)) {
    if (ensure_block_f32(blk, n, B_STONE, height, 0, 0, near)) { rc = DEGENERATE; goto out; }
  }
  if (!census[B_TREE]) {
    for (int i = 0; i < n; ++i) mask[i] = blk[i] == B_GRASS && near[i];
    int pos = pick_tile_f32(n, mask, u);
    if (pos < 0) {
      for (int i = 0; i < n; ++i) mask[i] = blk[i] == B_GRASS;
      pos = pick_tile_f32(n, mask, u);
    }
    if (pos < 0) { rc = DEGENERATE; goto out; }
    blk[pos] = B_TREE;
  }
  memset(o->items, 0, n);
  o->ld_r = o->ld_c = o->lu_r = o->lu_c = -1;
  if (extended) {
    for (int i = 0; i < n; ++i) mask[i] = WALKABLE_T[blk[i]] && cheb(i / w, i % w, sr, sc) >= 10;
    int pos = pick_tile_f32(n, mask, u);
    if (pos < 0) {
      for (int i = 0; i < n; ++i) mask[i] = WALKABLE_T[blk[i]];
      pos = pick_tile_f32(n, mask, u);
    }
    if (pos < 0 || pos == spawn) { rc = DEGENERATE; goto out; }
    o->items[pos] = I_LADDER_DOWN;
    o->ld_r = pos / w; o->ld_c = pos % w;
  }
  o->spawn_r = sr; o->spawn_c = sc;
out:
  free(u); free(near); free(mask);
  return rc;
}

/* worldgen.py:367-406 */
static int gen_dungeon(uint64_t seed, int h, int w, int floor, int attempt, floor_out *o) {
  int n = h * w;
  stream_t s = st_split(st_raw(seed), 1000 + (uint64_t)attempt);
  uint8_t *blk = o->blocks;
  memset(blk, B_WALL, n);
  int n_rooms = (int)st_randint(&s, 4, 8);
  int cr[8], cc[8];
  for (int k = 0; k < n_rooms; ++k) {
    int rh = (int)st_randint(&s, 5, 10);
    int rw = (int)st_randint(&s, 5, 10);
    int r0 = (int)st_randint(&s, 2, h - rh - 2);
    int c0 = (int)st_randint(&s, 2, w - rw - 2);
    for (int r = r0; r < r0 + rh; ++r)
      for (int c = c0; c < c0 + rw; ++c) blk[r * w + c] = B_PATH;
    cr[k] = r0 + rh / 2; cc[k] = c0 + rw / 2;
  }
  for (int k = 0; k + 1 < n_rooms; ++k) carve_line(blk, w, cr[k], cc[k], cr[k + 1], cc[k + 1], B_PATH);
  float *u = (float *)malloc(sizeof(float) * n);
  uint8_t *path = (uint8_t *)malloc(n);
  tile_uniform(go_hash2(seed, 7 + (uint64_t)attempt), n, 4, u);
  for (int i = 0; i < n; ++i) path[i] = blk[i] == B_PATH;
  for (int r = 0; r < h; ++r)
    for (int c = 0; c < w; ++c) {
      int i = r * w + c;
      int np_ = path[i] || (r > 0 && path[i - w]) || (r < h - 1 && path[i + w]) ||
                (c > 0 && path[i - 1]) || (c < w - 1 && path[i + 1]);
      if (blk[i] == B_WALL && np_ && u[i] < 0.25f) blk[i] = B_WALL_MOSS;
    }
  if (floor == 3)
    for (int i = 0; i < n; ++i) if (path[i] && u[i] > 0.82f) blk[i] = B_WATER;
  if (floor == 4)
    for (int i = 0; i < n; ++i) if (path[i] && u[i] > 0.85f) blk[i] = B_GRAVEL;
  for (int i = 0; i < n; ++i) path[i] = blk[i] == B_PATH;
  int fountain = pick_tile_f32(n, path, u);
  if (fountain >= 0) blk[fountain] = B_FOUNTAIN;
  free(u); free(path);
  int up = cr[0] * w + cc[0], down = cr[n_rooms - 1] * w + cc[n_rooms - 1];
  if (blk[up] != B_PATH || blk[down] != B_PATH || up == down) return DEGENERATE;
  memset(o->items, 0, n);
  o->items[up] = I_LADDER_UP;
  o->items[down] = I_LADDER_DOWN;
  o->spawn_r = o->lu_r = cr[0]; o->spawn_c = o->lu_c = cc[0];
  o->ld_r = cr[n_rooms - 1]; o->ld_c = cc[n_rooms - 1];
  return 0;
}

/* worldgen.py:418-468 */
static int gen_cave(uint64_t seed, int h, int w, int floor, int attempt, floor_out *o) {
  int n = h * w, rc = 0;
  stream_t s = st_split(st_raw(seed), 2000 + (uint64_t)attempt);
  double g25[25], g81[81];
  float a25[25], a81[81];
  st_uniform_array(&s, 25, g25);
  for (int i = 0; i < 25; ++i) a25[i] = (float)((g25[i] * 2.0) * 3.141592653589793);
  st_uniform_array(&s, 81, g81);
  for (int i = 0; i < 81; ++i) a81[i] = (float)((g81[i] * 2.0) * 3.141592653589793);
  double *field = (double *)malloc(sizeof(double) * n);
  double *dist = (double *)malloc(sizeof(double) * n);
  float *u = (float *)malloc(sizeof(float) * n);
  uint8_t *open = (uint8_t *)malloc(n);
  go_perlin_cave(a25, a81, h, w, field);
  uint8_t *blk = o->blocks;
  for (int i = 0; i < n; ++i) { open[i] = field[i] > -0.02; blk[i] = open[i] ? B_PATH : B_STONE; }
  tile_uniform(go_hash2(seed, 11 + (uint64_t)attempt), n, 5, u);
  for (int i = 0; i < n; ++i) if (open[i] && u[i] < 0.04f) blk[i] = B_STALAGMITE;
  for (int i = 0; i < n; ++i) {
    if (blk[i] != B_STONE) continue;
    float v = u[i];
    if (floor == 2) {
      if (v < 0.06f) blk[i] = B_COAL;
      if (v >= 0.90f && v < 0.93f) blk[i] = B_IRON;
      if (v >= 0.975f) blk[i] = B_SAPPHIRE;
    } else {
      if (v < 0.05f) blk[i] = B_COAL;
      if (v >= 0.90f && v < 0.93f) blk[i] = B_IRON;
      if (v >= 0.96f && v < 0.975f) blk[i] = B_DIAMOND;
      if (v >= 0.985f) blk[i] = B_RUBY;
    }
  }
  if (floor != 2)
    for (int i = 0; i < n; ++i) if (field[i] < -0.62) blk[i] = B_LAVA;
  {
    static const uint8_t must2[3] = {B_COAL, B_IRON, B_SAPPHIRE};
    static const uint8_t must5[4] = {B_COAL, B_IRON, B_DIAMOND, B_RUBY};
    const uint8_t *must = floor == 2 ? must2 : must5;
    int nm = floor == 2 ? 3 : 4;
    for (int k = 0; k < nm; ++k)
      if (ensure_block_cave(blk, n, must[k], field)) { rc = DEGENERATE; goto out; }
  }
  int cnt = 0;
  for (int i = 0; i < n; ++i) { open[i] = blk[i] == B_PATH; cnt += open[i]; }
  if (cnt < 40) { rc = DEGENERATE; goto out; }
  int up = pick_tile_f32(n, open, u);
  if (up < 0) { rc = DEGENERATE; goto out; }
  int ur = up / w, uc = up % w;
  double dmax = 0;
  for (int i = 0; i < n; ++i) {
    dist[i] = (double)cheb(i / w, i % w, ur, uc);
    if (dist[i] > dmax) dmax = dist[i];
  }
  for (int i = 0; i < n; ++i) dist[i] = dist[i] / dmax;
  int down = pick_tile_f64(n, open, dist);
  if (down < 0 || down == up) { rc = DEGENERATE; goto out; }
  int dr_ = down / w, dc_ = down % w;
  carve_line(blk, w, ur, uc, dr_, dc_, B_PATH);
  blk[up] = B_PATH;
  blk[down] = B_PATH;
  memset(o->items, 0, n);
  o->items[up] = I_LADDER_UP;
  o->items[down] = I_LADDER_DOWN;
  o->spawn_r = o->lu_r = ur; o->spawn_c = o->lu_c = uc;
  o->ld_r = dr_; o->ld_c = dc_;
out:
  free(field); free(dist); free(u); free(open);
  return rc;
}

/* worldgen.py:479-520 */
static int gen_realm(uint64_t seed, int h, int w, int floor, int attempt, floor_out *o) {
  int n = h * w, rc = 0;
  stream_t s = st_split(st_raw(seed), 3000 + (uint64_t)attempt);
  double g[252];
  float ang[252];
  st_uniform_array(&s, 9, g);
  st_uniform_array(&s, 81, g + 9);
  st_uniform_array(&s, 81, g + 90);
  st_uniform_array(&s, 81, g + 171);
  for (int i = 0; i < 252; ++i) ang[i] = (float)((g[i] * 2.0) * 3.141592653589793);
  float *height = (float *)malloc(sizeof(float) * n * 4);
  float *forest = height + n, *special = height + 2 * n, *u = height + 3 * n;
  uint8_t *base = (uint8_t *)malloc(n * 3);
  uint8_t *walk = base + n, *mask = base + 2 * n;
  go_overworld_fields(ang, h, w, height, forest, special);
  floor_out bo;
  bo.blocks = base;
  bo.items = o->items;
  if (gen_overworld(height, forest, special, go_hash2(seed, 4000 + (uint64_t)attempt), h, w, 0,
                    attempt, &bo)) { rc = DEGENERATE; goto out; }
  uint8_t *out = o->blocks;
  for (int i = 0; i < n; ++i) {
    uint8_t b = base[i], d = b;
    if (floor == 6) {
      if (b == B_GRASS) d = B_FIRE_GRASS;
      else if (b == B_TREE) d = B_FIRE_TREE;
      else if (b == B_WATER) d = B_LAVA;
      else if (b == B_SAND) d = B_GRAVEL;
    } else {
      if (b == B_GRASS) d = B_ICE_GRASS;
      else if (b == B_TREE) d = B_ICE_SHRUB;
      else if (b == B_SAND) d = B_GRAVEL;
      else if (b == B_LAVA) d = B_WATER;
    }
    out[i] = d;
  }
  uint8_t gem = floor == 6 ? B_RUBY : B_SAPPHIRE;
  tile_uniform(go_hash2(seed, 13 + (uint64_t)attempt), n, 6, u);
  for (int i = 0; i < n; ++i) if (out[i] == B_STONE && u[i] > 0.975f) out[i] = gem;
  if (ensure_block_f32(out, n, gem, u, 0, 0, NULL)) { rc = DEGENERATE; goto out; }
  /* _nearest_walkable: first row-major tile of min chebyshev to centre */
  int spawn = -1, bestd = 0;
  for (int i = 0; i < n; ++i) {
    if (!WALKABLE_T[out[i]]) continue;
    int d = cheb(i / w, i % w, h / 2, w / 2);
    if (spawn < 0 || d < bestd) { spawn = i; bestd = d; }
  }
  if (spawn < 0) { rc = DEGENERATE; goto out; }
  int sr = spawn / w, sc = spawn % w;
  for (int i = 0; i < n; ++i) mask[i] = WALKABLE_T[out[i]] && cheb(i / w, i % w, sr, sc) <= 8;
  int tpos = pick_tile_f32(n, mask, u);
  if (tpos < 0 || tpos == spawn) { rc = DEGENERATE; goto out; }
  out[tpos] = floor == 6 ? B_ENCHANT_TABLE_FIRE : B_ENCHANT_TABLE_ICE;
  for (int i = 0; i < n; ++i) {
    walk[i] = WALKABLE_T[out[i]];
    mask[i] = walk[i] && cheb(i / w, i % w, sr, sc) >= 10;
  }
  int down = pick_tile_f32(n, mask, u);
  if (down < 0) {
    float *inv = forest; /* reuse as 1 - u */
    for (int i = 0; i < n; ++i) inv[i] = 1.0f - u[i];
    down = pick_tile_f32(n, walk, inv);
  }
  if (down < 0 || down == spawn) { rc = DEGENERATE; goto out; }
  memset(o->items, 0, n);
  o->items[spawn] = I_LADDER_UP;
  o->items[down] = I_LADDER_DOWN;
  o->spawn_r = o->lu_r = sr; o->spawn_c = o->lu_c = sc;
  o->ld_r = down / w; o->ld_c = down % w;
out:
  free(height); free(base);
  return rc;
}

/* worldgen.py:523-546 */
static void gen_graveyard(int h, int w, floor_out *o) {
  int n = h * w;
  uint8_t *blk = o->blocks;
  memset(blk, B_DARKNESS, n);
  int cr = h / 2, cc = w / 2;
  int r0 = cr - 10, r1 = cr + 10, c0 = cc - 10, c1 = cc + 10;
  for (int r = r0; r <= r1; ++r) for (int c = c0; c <= c1; ++c) blk[r * w + c] = B_WALL;
  for (int r = r0 + 1; r < r1; ++r) for (int c = c0 + 1; c < c1; ++c) blk[r * w + c] = B_PATH;
  static const int go_[12][2] = {{-3, -5}, {-3, 5}, {0, -7}, {0, 7}, {3, -4}, {3, 4},
                                 {5, 0}, {-5, -2}, {-5, 2}, {6, -6}, {6, 6}, {2, 0}};
  static const uint8_t graves[3] = {B_GRAVE, B_GRAVE2, B_GRAVE3};
  for (int i = 0; i < 12; ++i) blk[(cr + go_[i][0]) * w + cc + go_[i][1]] = graves[i % 3];
  int pr = cr + 4, pc = cc - 5;
  for (int r = pr; r < pr + 3; ++r) for (int c = pc; c < pc + 3; ++c) blk[r * w + c] = B_WATER;
  blk[(cr - 6) * w + cc] = B_NECROMANCER;
  memset(o->items, 0, n);
  int ur = r1 - 2, uc = cc;
  blk[ur * w + uc] = B_PATH;
  o->items[ur * w + uc] = I_LADDER_UP;
  o->spawn_r = o->lu_r = ur; o->spawn_c = o->lu_c = uc;
  o->ld_r = o->ld_c = -1;
}

/* worldgen.py:549-575 */
static void template_floor(int floor, int h, int w, floor_out *o) {
  int n = h * w;
  uint8_t *blk = o->blocks;
  memset(blk, floor == 0 ? B_GRASS : B_PATH, n);
  if (floor != 0) {
    for (int c = 0; c < w; ++c) { blk[c] = B_WALL; blk[(h - 1) * w + c] = B_WALL; }
    for (int r = 0; r < h; ++r) { blk[r * w] = B_WALL; blk[r * w + w - 1] = B_WALL; }
  }
  int cr = h / 2, cc = w / 2;
  if (floor == 0) {
    for (int r = 2; r < 5; ++r) for (int c = 2; c < 5; ++c) blk[r * w + c] = B_WATER;
    for (int r = 6; r < 8; ++r) for (int c = 2; c < 6; ++c) blk[r * w + c] = B_SAND;
    blk[(cr - 4) * w + cc] = B_TREE;
    for (int r = h - 6; r < h - 2; ++r) for (int c = w - 6; c < w - 2; ++c) blk[r * w + c] = B_STONE;
    blk[(h - 5) * w + w - 5] = B_COAL;
    blk[(h - 4) * w + w - 4] = B_IRON;
    blk[(h - 3) * w + w - 3] = B_DIAMOND;
    blk[(h - 6) * w + w - 3] = B_LAVA;
  }
  memset(o->items, 0, n);
  o->spawn_r = cr; o->spawn_c = cc;
  o->lu_r = o->lu_c = o->ld_r = o->ld_c = -1;
  if (floor != 0) { o->lu_r = cr; o->lu_c = cc - 5; o->items[cr * w + cc - 5] = I_LADDER_UP; }
  if (floor != 8) { o->ld_r = cr; o->ld_c = cc + 5; o->items[cr * w + cc + 5] = I_LADDER_DOWN; }
}

/* worldgen.py:626-633 */
static void weighted_loot(double u, int *kind, int *qty) {
  static const int kinds[4] = {LOOT_POTION, LOOT_ARROWS, LOOT_TORCHES, LOOT_BOOK};
  static const int qtys[4] = {1, 3, 4, 1};
  static const double wts[4] = {0.40, 0.25, 0.20, 0.15};
  double acc = 0.0;
  for (int k = 0; k < 4; ++k) {
    acc += wts[k];
    if (u < acc) { *kind = kinds[k]; *qty = qtys[k]; return; }
  }
  *kind = kinds[3]; *qty = qtys[3];
}

/* worldgen.MAX_GEN_RETRIES (worldgen.py:36); settable so tests can force the
   _template_floor fallback (worldgen.py:549-595) */
static int max_gen_retries = 16;
void go_set_max_gen_retries(int n) { max_gen_retries = n; }

/* worldgen.py:636-651 + 578-633 */
void go_generate_world(uint64_t seed, int classic, go_world *W) {
  int h = classic ? 64 : 48, w = h, n = h * w;
  int F = classic ? 1 : 9;
  float angles[252];
  uint64_t fs[9];
  memset(W, 0, sizeof(*W));
  go_level_angles(seed, angles, fs);
  W->seed = seed;
  float *fields = (float *)malloc(sizeof(float) * n * 3);
  go_overworld_fields(angles, h, w, fields, fields + n, fields + 2 * n);
  for (int f = 0; f < F; ++f) {
    floor_out o;
    o.blocks = W->blocks[f];
    o.items = W->items[f];
    int ok = 0, attempt;
    for (attempt = 0; attempt < max_gen_retries && !ok; ++attempt) {
      int rc;
      if (f == 0) rc = gen_overworld(fields, fields + n, fields + 2 * n, fs[0], h, w, !classic, attempt, &o);
      else if (f == 1 || f == 3 || f == 4) rc = gen_dungeon(fs[f], h, w, f, attempt, &o);
      else if (f == 2 || f == 5) rc = gen_cave(fs[f], h, w, f, attempt, &o);
      else if (f == 6 || f == 7) rc = gen_realm(fs[f], h, w, f, attempt, &o);
      else { gen_graveyard(h, w, &o); rc = 0; }
      ok = rc == 0;
    }
    W->attempts[f] = attempt;
    if (!ok) template_floor(f, h, w, &o);
    if (f == 0) { W->spawn[0] = (int16_t)o.spawn_r; W->spawn[1] = (int16_t)o.spawn_c; }
    W->ladder_down[f][0] = (int16_t)o.ld_r; W->ladder_down[f][1] = (int16_t)o.ld_c;
    W->ladder_up[f][0] = (int16_t)o.lu_r; W->ladder_up[f][1] = (int16_t)o.lu_c;
  }
  free(fields);
  /* potion permutation: np.argsort of six hashed f32 draws (worldgen.py:647-649) */
  {
    uint32_t k32 = (uint32_t)(go_hash2(seed, 42) & 0xFFFFFFFFu);
    float v[6];
    for (int i = 0; i < 6; ++i) v[i] = go_vuniform32(k32, (uint32_t)i);
    go_np_argsort6(v, W->potion);
    for (int i = 0; i < 6; ++i)
      for (int j = i + 1; j < 6; ++j) if (v[i] == v[j]) W->potion_tie = 1;
  }
  /* chests (worldgen.py:598-623) */
  static const int per_floor[9] = {0, 4, 2, 3, 3, 2, 2, 2, 0};
  for (int f = 0; f < F; ++f) {
    int nc = per_floor[f];
    W->n_chests[f] = 0;
    if (!nc) continue;
    stream_t s = st_split(st_raw(seed), 5000 + (uint64_t)f);
    uint8_t *blk = W->blocks[f], *itm = W->items[f];
    int *list = (int *)malloc(sizeof(int) * n);
    int len = 0;
    for (int i = 0; i < n; ++i) if (blk[i] == B_PATH) list[len++] = i;
    if (len) {
      int lim = nc < 6 ? nc : 6;
      if (len < lim) lim = len;
      for (int i = 0; i < lim; ++i) {
        int j = (int)st_randint(&s, 0, len);
        int t = list[j];
        if (blk[t] != B_PATH || itm[t] != I_EMPTY) continue;
        blk[t] = B_CHEST;
        int kind, qty;
        int nl = W->n_chests[f];
        if (f == 1 && nl == 0) { kind = LOOT_BOW; qty = 1; }
        else if (f == 1 && nl == 1) { kind = LOOT_BOOK; qty = 1; }
        else weighted_loot(st_uniform01(&s), &kind, &qty);
        W->chest[f][nl][0] = (int16_t)(t / w);
        W->chest[f][nl][1] = (int16_t)(t % w);
        W->chest[f][nl][2] = (int16_t)kind;
        W->chest[f][nl][3] = (int16_t)qty;
        W->n_chests[f] = nl + 1;
      }
    }
    free(list);
  }
}
