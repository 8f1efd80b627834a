// gr_device.cuh -- device-side rule tables, counter-based PRNG and the
// bit-exact math shared by the worldgen, step and observation kernels.
//
// Reference (read-only, /root/reference/pkg/src/gridrogue):
//   constants.py:17-567   rule tables             -> __constant__ arrays here
//   rng.py:23-88          splitmix64 / lowbias32   -> gr_mix / gr_hash2 / gr_u32
//   _kern.py:57-66        q1 / resolve_attack_vec  -> gr_q1 / gr_resolve
//
// Numerics: everything is compiled with -fmad=false so each float op is
// separately rounded like numpy's elementwise loops; the few fused ops that
// numpy *does* use (its float32 SIMD sin/cos) are spelled out with
// __fmaf_rn.  No fast-math anywhere.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gr {

// ---------------------------------------------------------------- blocks
enum : uint8_t {
  B_INVALID, B_OOB, B_GRASS, B_WATER, B_STONE, B_TREE, B_WOOD, B_PATH, B_COAL,
  B_IRON, B_DIAMOND, B_TABLE, B_FURNACE, B_SAND, B_LAVA, B_PLANT, B_RIPE_PLANT,
  B_WALL, B_DARKNESS, B_WALL_MOSS, B_STALAGMITE, B_SAPPHIRE, B_RUBY, B_CHEST,
  B_FOUNTAIN, B_FIRE_GRASS, B_ICE_GRASS, B_GRAVEL, B_FIRE_TREE, B_ICE_SHRUB,
  B_ENCHANT_FIRE, B_ENCHANT_ICE, B_NECROMANCER, B_GRAVE, B_GRAVE2, B_GRAVE3,
  B_NECROMANCER_VULN
};
enum : uint8_t { I_EMPTY, I_TORCH, I_LADDER_DOWN, I_LADDER_UP };
enum : uint8_t { LOOT_NOTHING, LOOT_BOW, LOOT_BOOK, LOOT_POTION, LOOT_ARROWS, LOOT_TORCHES };

// bit sets over the 37 block ids (constants.py:422-462)
#define GR_BIT(b) (1ull << (b))
constexpr uint64_t WALK_SET = GR_BIT(B_GRASS) | GR_BIT(B_PATH) | GR_BIT(B_SAND) | GR_BIT(B_FIRE_GRASS) |
                              GR_BIT(B_ICE_GRASS) | GR_BIT(B_GRAVEL);
// COLLISION_WALKABLE rows: ground, flying, amphibian, aquatic
__host__ __device__ __forceinline__ constexpr uint64_t coll_set(int c) {
  return c == 1 ? (WALK_SET | GR_BIT(B_WATER) | GR_BIT(B_LAVA) | GR_BIT(B_STALAGMITE))
       : c == 2 ? (WALK_SET | GR_BIT(B_WATER))
       : c == 3 ? GR_BIT(B_WATER)
                : WALK_SET;
}
constexpr uint64_t ALL37 = (1ull << 37) - 1;
constexpr uint64_t PROJ_STOP_SET =
    ALL37 & ~(WALK_SET | GR_BIT(B_WATER) | GR_BIT(B_LAVA) | GR_BIT(B_PLANT) | GR_BIT(B_RIPE_PLANT));
constexpr uint64_t PLACE_STONE_SET = WALK_SET | GR_BIT(B_WATER) | GR_BIT(B_LAVA);
constexpr uint64_t PLACE_SOLID_SET = WALK_SET;

__device__ __forceinline__ bool in_set(uint64_t set, uint32_t b) { return (set >> b) & 1ull; }

// ------------------------------------------------------------ creatures
// kind -> hp, damage, defense, collision (constants.py:113-136)
__constant__ float C_HP[19] = {5, 3, 3, 7, 5, 6, 9, 6, 4, 11, 8, 12, 12, 20, 6, 20, 14, 24, 16};
__constant__ float C_DMG[19][3] = {
    {2, 0, 0}, {2, 0, 0}, {0, 0, 0}, {3, 0, 0}, {3, 0, 0}, {0, 0, 0}, {4, 0, 0},
    {2, 0, 0}, {0, 0, 0}, {5, 0, 0}, {4, 0, 0}, {6, 0, 0}, {4, 0, 0}, {6, 1, 1},
    {4, 3, 3}, {3, 5, 0}, {3, 5, 0}, {4, 0, 5}, {4, 0, 4}};
__constant__ float C_DEF[19][3] = {
    {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0},
    {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {50, 0, 0}, {50, 0, 0}, {20, 0, 0},
    {0, 0, 0}, {90, 100, 0}, {90, 100, 0}, {90, 0, 100}, {90, 0, 100}};
__constant__ uint8_t C_COLL[19] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 2, 0, 0, 0, 0, 3, 0, 1, 0, 0};
// per-floor resident kinds (constants.py:160-167), -1 = none
__constant__ int8_t C_MEL_KIND[9] = {0, 3, 6, 9, 11, 13, 15, 17, -1};
__constant__ int8_t C_RAN_KIND[9] = {1, 4, 7, 10, 12, 14, 16, 18, -1};
__constant__ int8_t C_PAS_KIND[9] = {2, 5, 8, 5, 5, 8, 8, -1, -1};
__constant__ uint8_t C_RANGED_PROJ[19] = {0, 3, 0, 0, 4, 0, 0, 3, 0, 0, 5, 0, 3, 0, 6, 0, 7, 0, 8};
__constant__ uint8_t C_DEFEAT_ACH[19] = {8, 12, 2, 38, 39, 51, 36, 37, 50, 40, 41, 65, 66, 42, 43, 44, 45, 46, 47};
__constant__ float C_EAT[19] = {0, 0, 6, 0, 0, 4, 0, 0, 2, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
// q1(max(sum(dmg), 0)) against an unarmoured player (creatures.py:53)
__constant__ float C_DEALT_BARE[19] = {2, 2, 0, 3, 3, 0, 4, 2, 0, 5, 4, 6, 4, 8, 10, 8, 8, 9, 8};
// achievement tier values (constants.py:299-307)
__constant__ uint8_t C_ACH_TIER[67] = {
    1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 3, 3, 3, 3, 3, 5, 5, 5, 8,
    8, 8, 3, 3, 3, 3, 5, 5, 5, 5, 8, 8, 8, 8, 8, 8, 3, 3, 3, 3, 3, 5, 5, 5, 5, 3, 3, 3, 3, 5, 5, 5, 5};
__constant__ uint8_t C_ENTER_ACH[9] = {255, 29, 28, 30, 31, 32, 33, 34, 35};
__constant__ float C_SWORD_BASE[5] = {1, 2, 3, 5, 8};
__constant__ float C_FLOOR_AMB[9] = {1, 1, 0, 1, 1, 0, 1, 0, 0};
// spawn probabilities, float64 (creatures.py:61-69)
__constant__ double C_MEL_PROB[2][9] = {{0.008, 0.05, 0.05, 0.05, 0.05, 0.05, 0.05, 0.05, 0},
                                        {0.05, 0.05, 0.05, 0.05, 0.05, 0.05, 0.05, 0.05, 0}};
__constant__ double C_RAN_PROB[9] = {0.02, 0.02, 0.02, 0.02, 0.02, 0.02, 0.02, 0.02, 0};
__constant__ double C_PAS_PROB[9] = {0.1, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1, 0};
__constant__ int8_t C_DIR[4][2] = {{0, -1}, {0, 1}, {-1, 0}, {1, 0}};

// ------------------------------------------------------------------ rng
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t hash2(uint64_t key, uint64_t n) { return mix64(key ^ mix64(n)); }
__host__ __device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  return x ^ (x >> 16);
}
// rng.vuniform32: 24-bit uniform in [0,1) as float32
__device__ __forceinline__ float u32f(uint32_t key, uint32_t n) {
  uint32_t h = mix32(key ^ (n * 0x9E3779B9u + 0x9E3779B9u));
  return __fmul_rn(__uint2float_rn(h >> 8), 5.9604644775390625e-08f);
}
// rng.vuniform: 53-bit uniform in [0,1) as float64
__device__ __forceinline__ double u64d(uint64_t key, uint64_t n) {
  return __dmul_rn(__ull2double_rn(hash2(key, n) >> 11), 1.1102230246251565e-16);
}

// immutable (key, counter) stream of rng.RngStream
struct Stream {
  uint64_t key, ctr;
  __device__ static Stream raw(uint64_t k) { return {k, 0}; }
  __device__ Stream split(uint64_t id) const { return {hash2(key, hash2(id, ctr)), 0}; }
  __device__ uint64_t next() { return hash2(key, ctr++); }
  __device__ int randint(int lo, int hi) { return lo + (int)(next() % (uint64_t)(hi - lo)); }
  __device__ double uniform01() { return __dmul_rn(__ull2double_rn(next() >> 11), 1.1102230246251565e-16); }
  // uniform_array element i (does not advance)
  __device__ double at(uint64_t i) const { return u64d(key, ctr + i); }
};

// ------------------------------------------- numpy float32 SIMD sin/cos
// numpy's loops_trigonometric: Cody-Waite by pi/2 (quadrant rounded to
// nearest), then minimax polynomials evaluated with fused multiply-adds.
__device__ __forceinline__ float np_sincosf(float x, bool is_cos) {
  float q = rintf(__fmul_rn(x, 0x1.45f306p-1f));
  float r = __fmaf_rn(q, -0x1.921fb0p+0f, x);
  r = __fmaf_rn(q, -0x1.5110b4p-22f, r);
  r = __fmaf_rn(q, -0x1.846988p-48f, r);
  float r2 = __fmul_rn(r, r);
  int iq = (int)q + (is_cos ? 1 : 0);
  float v;
  if ((iq & 1) == 0) {
    float s = __fmaf_rn(0x1.7d3bbcp-19f, r2, -0x1.a06bbap-13f);
    s = __fmaf_rn(s, r2, 0x1.11119ap-07f);
    s = __fmaf_rn(s, r2, -0x1.555556p-03f);
    s = __fmul_rn(s, r2);
    v = __fmaf_rn(s, r, r);
  } else {
    float c = __fmaf_rn(0x1.98e616p-16f, r2, -0x1.6c06dcp-10f);
    c = __fmaf_rn(c, r2, 0x1.55553cp-5f);
    c = __fmaf_rn(c, r2, -0x1.000000p-1f);
    v = __fmaf_rn(c, r2, 0x1.000000p+0f);
  }
  return (iq & 2) ? -v : v;
}

// float64 sin / cos of the cave noise (hazard H3): glibc's own algorithm,
// bit for bit (gr_glibc_sincos.h).
#include "gr_glibc_sincos.h"

// -------------------------------------------------------- game helpers
// _kern.q1: one-decimal quantiser, every op separately rounded
// np.argsort of 6 float32 (worldgen.py:647-649).  numpy >= 2 on AVX-512
// hardware sorts n <= 256 elements with x86-simd-sort's key/index bitonic
// network: one 8-lane register (lanes 6, 7 padded with +inf, which never
// move), six compare-exchange layers with partner lane l^1, l^3, l^1, l^7,
// l^2, l^1, the upper lane taking the max and each lane keeping its own index
// on equal keys.  Restricted to the six live lanes that is the 15-comparator
// network below, exchanging only on a strict '>'.  On ties it is NOT a stable
// sort; it equals np.argsort on all 6^6 value patterns
// (tests/golden/numpy_corners.npz).
__host__ __device__ __forceinline__ void np_argsort6(const float* v, uint8_t* idx) {
  constexpr uint8_t P[15][2] = {{0, 1}, {2, 3}, {4, 5}, {0, 3}, {1, 2}, {0, 1}, {2, 3}, {4, 5},
                                {2, 5}, {3, 4}, {0, 2}, {1, 3}, {0, 1}, {2, 3}, {4, 5}};
  float k[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) { k[i] = v[i]; idx[i] = (uint8_t)i; }
#pragma unroll
  for (int c = 0; c < 15; ++c) {
    const int a = P[c][0], b = P[c][1];
    if (k[a] > k[b]) {
      const float tk = k[a]; k[a] = k[b]; k[b] = tk;
      const uint8_t ti = idx[a]; idx[a] = idx[b]; idx[b] = ti;
    }
  }
}

__device__ __forceinline__ float q1(float x) {
  return __fmul_rn(floorf(__fadd_rn(__fmul_rn(x, 10.0f), 0.5f)), 0.1f);
}
// _kern.resolve_attack_vec for one (3,) damage vs (3,) percent defense.
// Three IEEE divisions (~25 instructions each): one out-of-line copy instead
// of one per call site keeps k_step's code (and its i-cache misses) smaller.
#ifndef GR_RESOLVE_INLINE
#define GR_RESOLVE_INLINE __noinline__
#endif
static __device__ GR_RESOLVE_INLINE float resolve(const float d0, const float d1, const float d2, const float f0,
                                         const float f1, const float f2) {
  float t0 = __fmul_rn(d0, __fsub_rn(1.0f, __fdiv_rn(f0, 100.0f)));
  float t1 = __fmul_rn(d1, __fsub_rn(1.0f, __fdiv_rn(f1, 100.0f)));
  float t2 = __fmul_rn(d2, __fsub_rn(1.0f, __fdiv_rn(f2, 100.0f)));
  float s = __fadd_rn(__fadd_rn(t0, t1), t2);
  if (s < 0.0f) s = 0.0f;
  return q1(s);
}

}  // namespace gr
