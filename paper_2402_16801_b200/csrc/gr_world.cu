// gr_world.cu -- procedural world generation on device, one CTA per
// (world, floor), the floor staged in shared memory.
//
// Restates worldgen.py (and perlin.py) per floor:
//   floor 0   overworld  worldgen.py:181-327  (+ make_level_params :75-87)
//   1, 3, 4   dungeon    worldgen.py:367-406
//   2, 5      cave       worldgen.py:418-468  (float64 noise)
//   6, 7      realm      worldgen.py:479-520
//   8         graveyard  worldgen.py:523-546
//   fallback  template   worldgen.py:549-575 after 16 failed attempts (:578-595)
//   chests    worldgen.py:598-633, potion permutation :647-649
// The per-tile work (noise, thresholds, sprinkles) is spread over the
// threads; every argmax/argmin of the reference becomes a block reduction
// with numpy's first-index tie-break; the sequential RNG parts are spread
// over threads where the counter-based streams allow it.
//
// Shared memory holds only the floor's blocks/items and small tables: the
// per-tile uniforms and noise values are recomputed where needed (hashing
// is cheaper than the occupancy that storing them costs), so ~5 CTAs fit
// per SM next to the observation writer.
#include <cstdint>
#include <climits>
#include <algorithm>
#include "gr_device.cuh"
#include "gr_state.cuh"
#include "gr_kernels.cuh"

#ifndef GR_WG_EXT_THREADS
#define GR_WG_EXT_THREADS 128
#endif
namespace gr {
#if GR_WG_WIDE
// gr_world_wide.cu: this file again with 512-thread extended-tier CTAs, for
// small batches where the reset chain's latency (one floor per CTA) is the
// step's critical path
namespace wide {
#else
namespace wide {
void launch_worldgen(bool ext, const WorldJob& j, cudaStream_t st);
}
#endif

constexpr double PI_D = 3.141592653589793;

template <bool EXT>
struct WT {
  static constexpr int H = EXT ? 48 : 64, W = H, HW = H * W, F = EXT ? 9 : 1;
  // threads per (world, floor) CTA: the classic tier has one floor per world
  // and few worlds per step, so its single floor gets more threads (classic
  // 65,536 envs: 128 / 256 / 512 / 1024 threads -> 0.090 / 0.083 / 0.087 /
  // 0.102 ms of worldgen per step)
  static constexpr int THREADS = EXT ? GR_WG_EXT_THREADS : 256, WARPS = THREADS / 32;
  static constexpr int MINB = 1024 / THREADS;   // resident CTAs the registers are fitted to (64 registers)
};

template <bool EXT>
struct WSmem {
  alignas(16) uint8_t blk[WT<EXT>::HW];
  alignas(16) uint8_t itm[WT<EXT>::HW];
  uint16_t list[EXT ? WT<EXT>::HW : 1];   // row-major PATH tiles (chests)
  float gx[252], gy[252];                 // overworld / realm gradients
  double dgx[EXT ? 106 : 1], dgy[EXT ? 106 : 1];  // cave gradients
  float prof[2][8][32];                   // [coarse/fine][a1..a4,b0..b3][i]
  double dprof[EXT ? 2 : 1][8][12];
  float ang[252];
  static constexpr int NWARP = WT<EXT>::WARPS;
  float rf[NWARP];
  double rd[NWARP];
  int ri[32];
  unsigned long long ru[NWARP];
  int res_i;
  unsigned long long res_u;
  int spawn;
  int cr[8], cc[8];
  int room[8][4];
  uint64_t rowmask[WT<EXT>::H];            // dungeon: room columns per row
};

// ------------------------------------------------------- block reductions
// The reductions, the per-floor generators and the other multi-call-site
// helpers are __noinline__: fully inlined, k_worldgen<true> was 361 KB of
// SASS and 42% of its warp stalls were no_instructions (icache misses).
template <class SM>
__device__ __noinline__ int block_argmax_f(SM& sm, float v, int idx) {   // idx = INT_MAX: no candidate
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_down_sync(0xffffffffu, v, o);
    int oi = __shfl_down_sync(0xffffffffu, idx, o);
    if (oi != INT_MAX && (idx == INT_MAX || ov > v || (ov == v && oi < idx))) { v = ov; idx = oi; }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sm.rf[w] = v; sm.ri[w] = idx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float bv = sm.rf[0];
    int bi = sm.ri[0];
    for (int k = 1; k < SM::NWARP; ++k) {
      int oi = sm.ri[k];
      float ov = sm.rf[k];
      if (oi != INT_MAX && (bi == INT_MAX || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
    }
    sm.res_i = bi == INT_MAX ? -1 : bi;
  }
  __syncthreads();
  int r = sm.res_i;
  __syncthreads();
  return r;
}

template <class SM>
__device__ __noinline__ int block_argmax_d(SM& sm, double v, int idx) {
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_down_sync(0xffffffffu, v, o);
    int oi = __shfl_down_sync(0xffffffffu, idx, o);
    if (oi != INT_MAX && (idx == INT_MAX || ov > v || (ov == v && oi < idx))) { v = ov; idx = oi; }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sm.rd[w] = v; sm.ri[w] = idx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double bv = sm.rd[0];
    int bi = sm.ri[0];
    for (int k = 1; k < SM::NWARP; ++k) {
      int oi = sm.ri[k];
      double ov = sm.rd[k];
      if (oi != INT_MAX && (bi == INT_MAX || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
    }
    sm.res_i = bi == INT_MAX ? -1 : bi;
  }
  __syncthreads();
  int r = sm.res_i;
  __syncthreads();
  return r;
}

template <class SM>
__device__ __noinline__ unsigned long long block_min_u64(SM& sm, unsigned long long v) {
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long ov = __shfl_down_sync(0xffffffffu, v, o);
    v = ov < v ? ov : v;
  }
  if ((threadIdx.x & 31) == 0) sm.ru[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long b = sm.ru[0];
    for (int k = 1; k < SM::NWARP; ++k) b = sm.ru[k] < b ? sm.ru[k] : b;
    sm.res_u = b;
  }
  __syncthreads();
  unsigned long long r = sm.res_u;
  __syncthreads();
  return r;
}

template <class SM>
__device__ __noinline__ unsigned long long block_or_u64(SM& sm, unsigned long long v) {
  for (int o = 16; o > 0; o >>= 1) v |= __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sm.ru[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long b = 0;
    for (int k = 0; k < SM::NWARP; ++k) b |= sm.ru[k];
    sm.res_u = b;
  }
  __syncthreads();
  unsigned long long r = sm.res_u;
  __syncthreads();
  return r;
}

// exclusive prefix sum over the threads of the CTA (thread order)
template <class SM>
__device__ __noinline__ int block_excl_scan(SM& sm, int v, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm.ri[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < SM::NWARP ? sm.ri[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    sm.ri[lane] = w;
  }
  __syncthreads();
  const int r = (warp ? sm.ri[warp - 1] : 0) + x - v;
  *total = sm.ri[SM::NWARP - 1];
  __syncthreads();
  return r;
}

template <bool EXT>
__device__ __noinline__ unsigned long long census(WSmem<EXT>& sm) {
  unsigned long long m = 0;
  // 16 tiles per shared-memory load (block ids < 64)
  const uint4* b4 = reinterpret_cast<const uint4*>(sm.blk);
  for (int q = threadIdx.x; q < WT<EXT>::HW / 16; q += WT<EXT>::THREADS) {
    const uint4 x = b4[q];
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int j = 0; j < 4; ++j) m |= 1ull << ((w[k] >> (8 * j)) & 63u);
  }
  return block_or_u64(sm, m);
}

__device__ __forceinline__ int cheb(int r0, int c0, int r1, int c1) { return max(abs(r0 - r1), abs(c0 - c1)); }

// worldgen._pick_tile: argmax of score(t) over tiles with pred(t)
template <bool EXT, class P, class S>
__device__ int pick(WSmem<EXT>& sm, P pred, S score) {
  float bv = 0.0f;
  int bi = INT_MAX;
  for (int t = threadIdx.x; t < WT<EXT>::HW; t += WT<EXT>::THREADS)
    if (pred(t)) {
      const float s = score(t);
      if (bi == INT_MAX || s > bv) { bv = s; bi = t; }
    }
  return block_argmax_f(sm, bv, bi);
}

// the per-tile hashed uniform field (worldgen._tile_uniform) on demand
struct UField {
  uint32_t k32;
  __device__ UField(uint64_t key, uint64_t salt) : k32((uint32_t)(hash2(key, salt) & 0xFFFFFFFFull)) {}
  __device__ __forceinline__ float operator()(int t) const { return u32f(k32, (uint32_t)t); }
};

// ------------------------------------------------------------ noise
// perlin._profiles (perlin.py:36-51) for both octave sizes, float32
template <bool EXT>
__device__ void build_profiles_f32(WSmem<EXT>& sm) {
  const int H = WT<EXT>::H;
  const int dims[2] = {H / 2, H / 8};
  for (int k = threadIdx.x; k < 2 * 32; k += WT<EXT>::THREADS) {
    const int o = k / 32, i = k % 32, d = dims[o];
    if (i >= d) continue;
    float f = __fdiv_rn((float)i, (float)d);
    float u = __fmul_rn(__fmul_rn(__fmul_rn(f, f), f),
                        __fadd_rn(__fmul_rn(f, __fsub_rn(__fmul_rn(f, 6.0f), 15.0f)), 10.0f));
    const float one = 1.0f, root2 = 1.41421353816986083984375f;
    sm.prof[o][0][i] = __fsub_rn(one, u);
    sm.prof[o][1][i] = __fmul_rn(__fsub_rn(one, u), f);
    sm.prof[o][2][i] = u;
    sm.prof[o][3][i] = __fmul_rn(u, __fsub_rn(f, one));
    sm.prof[o][4][i] = __fmul_rn(__fmul_rn(__fsub_rn(one, u), f), root2);
    sm.prof[o][5][i] = __fmul_rn(__fsub_rn(one, u), root2);
    sm.prof[o][6][i] = __fmul_rn(__fmul_rn(u, __fsub_rn(f, one)), root2);
    sm.prof[o][7][i] = __fmul_rn(u, root2);
  }
}

// one octave value at tile (r, c): perlin_octave, float32, einsum order
template <bool EXT>
__device__ __forceinline__ float octave_at(const WSmem<EXT>& sm, int o, const float* gx, const float* gy, int res,
                                           int r, int c) {
  const int d = WT<EXT>::H / res;
  const int R = r / d, i = r % d, C = c / d, j = c % d, n = res + 1;
  const float* P = &sm.prof[o][0][0];
  const float a1 = P[0 * 32 + i], a2 = P[1 * 32 + i], a3 = P[2 * 32 + i], a4 = P[3 * 32 + i];
  const float b0 = P[4 * 32 + j], b1 = P[5 * 32 + j], b2 = P[6 * 32 + j], b3 = P[7 * 32 + j];
  const int k00 = R * n + C, k10 = (R + 1) * n + C;
  float t0 = __fadd_rn(__fmul_rn(gx[k00], a1), __fmul_rn(gx[k10], a3));
  float t1 = __fadd_rn(__fmul_rn(gy[k00], a2), __fmul_rn(gy[k10], a4));
  float t2 = __fadd_rn(__fmul_rn(gx[k00 + 1], a1), __fmul_rn(gx[k10 + 1], a3));
  float t3 = __fadd_rn(__fmul_rn(gy[k00 + 1], a2), __fmul_rn(gy[k10 + 1], a4));
  return __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(t0, b0), __fmul_rn(t1, b1)), __fmul_rn(t2, b2)), __fmul_rn(t3, b3));
}

// worldgen.overworld_fields height at one tile (recomputed on demand)
template <bool EXT>
__device__ __forceinline__ float height_at(const WSmem<EXT>& sm, int t) {
  const int r = t / WT<EXT>::W, c = t % WT<EXT>::W;
  const float coarse = octave_at<EXT>(sm, 0, sm.gx, sm.gy, 2, r, c);
  const float f1 = octave_at<EXT>(sm, 1, sm.gx + 9, sm.gy + 9, 8, r, c);
  return __fdiv_rn(__fadd_rn(coarse, __fmul_rn(0.35f, f1)), 1.35f);
}

// worldgen._overworld_blocks for one tile
__device__ __forceinline__ uint8_t overworld_tile(float h, float forest, float special, float u) {
  uint8_t b = B_GRASS;
  if (h < -0.28f) b = B_WATER;
  if (h >= -0.28f && h < -0.22f) b = B_SAND;
  const bool mountain = h > 0.28f;
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

// worldgen._ensure_block with a float32 score (overworld / realm);
// score(t) is the *height* argument, negated here when low
template <bool EXT, class S>
__device__ bool ensure_f32(WSmem<EXT>& sm, uint8_t block, S hfun, bool low, int spawn) {
  using T = WT<EXT>;
  const unsigned long long present = census(sm);
  if ((present >> block) & 1ull) return true;
  auto score = [&](int t) { const float h = hfun(t); return low ? -h : h; };
  if (!low) {
    const int pos = pick(sm, [&](int t) { return sm.blk[t] == B_STONE; }, score);
    if (pos >= 0) {
      if (threadIdx.x == 0) sm.blk[pos] = block;
      __syncthreads();
      return true;
    }
  }
  const int sr = spawn >= 0 ? spawn / T::W : 0, sc = spawn >= 0 ? spawn % T::W : 0;
  auto near = [&](int t) { return spawn >= 0 && t != spawn && cheb(t / T::W, t % T::W, sr, sc) <= 8; };
  int any_near = 0, any_grass = 0;
  for (int t = threadIdx.x; t < T::HW; t += WT<EXT>::THREADS) {
    any_grass |= sm.blk[t] == B_GRASS;
    any_near |= sm.blk[t] == B_GRASS && near(t);
  }
  any_near = __syncthreads_or(any_near);
  any_grass = __syncthreads_or(any_grass);
  const int pos = pick(sm, [&](int t) {
    const uint8_t b = sm.blk[t];
    return any_near ? (b == B_GRASS && near(t)) : any_grass ? b == B_GRASS : (b == B_GRASS || b == B_TREE);
  }, score);
  if (pos < 0) return false;
  if (threadIdx.x == 0) sm.blk[pos] = block;
  __syncthreads();
  return true;
}

// first walkable tile of minimal Chebyshev distance to the centre
// (worldgen.py:267-269, and _nearest_walkable :134-143)
template <bool EXT>
__device__ __noinline__ int nearest_walkable(WSmem<EXT>& sm) {
  using T = WT<EXT>;
  unsigned long long best = ~0ull;
  for (int t = threadIdx.x; t < T::HW; t += WT<EXT>::THREADS)
    if (in_set(WALK_SET, sm.blk[t])) {
      unsigned long long k = ((unsigned long long)cheb(t / T::W, t % T::W, T::H / 2, T::W / 2) << 32) | (unsigned)t;
      best = k < best ? k : best;
    }
  best = block_min_u64(sm, best);
  return best == ~0ull ? -1 : (int)(best & 0xFFFFFFFFull);
}

// worldgen._gen_overworld (:247-327) on gradients already in sm.gx/gy.
// Returns false for _Degenerate.  Spawn -> sm.spawn, ladder -> *ld.
template <bool EXT>
__device__ __noinline__ bool gen_overworld(WSmem<EXT>& sm, uint64_t seed0, bool extended, int attempt, int* ld) {
  using T = WT<EXT>;
  const UField u(hash2(seed0, (uint64_t)attempt), 1);
  for (int t = threadIdx.x; t < T::HW; t += WT<EXT>::THREADS) {
    const int r = t / T::W, c = t % T::W;
    const float forest = octave_at<EXT>(sm, 1, sm.gx + 90, sm.gy + 90, 8, r, c);
    const float special = octave_at<EXT>(sm, 1, sm.gx + 171, sm.gy + 171, 8, r, c);
    sm.blk[t] = overworld_tile(height_at<EXT>(sm, t), forest, special, u(t));
    sm.itm[t] = 0;
  }
  __syncthreads();
  const int spawn = nearest_walkable(sm);
  if (spawn < 0) return false;
  if (threadIdx.x == 0) { sm.blk[spawn] = B_GRASS; sm.spawn = spawn; }
  __syncthreads();
  const unsigned long long cen = census(sm);
  auto height = [&](int t) { return height_at<EXT>(sm, t); };
  bool fixed_any = false;
  const uint8_t order[6] = {B_COAL, B_IRON, B_DIAMOND, B_LAVA, B_WATER, B_SAND};
#pragma unroll 1
  for (int k = 0; k < 6; ++k) {
    if (!((cen >> order[k]) & 1ull)) {
      if (!ensure_f32<EXT>(sm, order[k], height, k >= 4, spawn)) return false;
      fixed_any = true;
    }
  }
  if (!((cen >> B_STONE) & 1ull) || (fixed_any && !((census(sm) >> B_STONE) & 1ull)))
    if (!ensure_f32<EXT>(sm, B_STONE, height, false, spawn)) return false;
  const int sr = spawn / T::W, sc = spawn % T::W;
  if (!((cen >> B_TREE) & 1ull)) {
    int pos = pick(sm, [&](int t) {
      return sm.blk[t] == B_GRASS && t != spawn && cheb(t / T::W, t % T::W, sr, sc) <= 8;
    }, u);
    if (pos < 0) pos = pick(sm, [&](int t) { return sm.blk[t] == B_GRASS; }, u);
    if (pos < 0) return false;
    if (threadIdx.x == 0) sm.blk[pos] = B_TREE;
    __syncthreads();
  }
  *ld = -1;
  if (extended) {
    int pos = pick(sm, [&](int t) {
      return in_set(WALK_SET, sm.blk[t]) && cheb(t / T::W, t % T::W, sr, sc) >= 10;
    }, u);
    if (pos < 0) pos = pick(sm, [&](int t) { return in_set(WALK_SET, sm.blk[t]); }, u);
    if (pos < 0 || pos == spawn) return false;
    if (threadIdx.x == 0) sm.itm[pos] = I_LADDER_DOWN;
    __syncthreads();
    *ld = pos;
  }
  return true;
}

// gradients of the 252 angles in sm.ang (numpy float32 sin/cos)
template <bool EXT>
__device__ void overworld_gradients(WSmem<EXT>& sm) {
  for (int k = threadIdx.x; k < 252; k += WT<EXT>::THREADS) {
    sm.gx[k] = np_sincosf(sm.ang[k], true);
    sm.gy[k] = np_sincosf(sm.ang[k], false);
  }
  __syncthreads();
}

// f32(u * 2 * pi) exactly as (flat * 2.0 * np.pi).astype(np.float32)
__device__ __forceinline__ float angle_of(double u) { return __double2float_rn(__dmul_rn(__dmul_rn(u, 2.0), PI_D)); }

struct FloorOut { int spawn, ld, lu; };

// worldgen._gen_realm (:479-520)
template <bool EXT>
__device__ __noinline__ bool gen_realm(WSmem<EXT>& sm, uint64_t seed, int floor, int attempt, FloorOut* fo) {
  using T = WT<EXT>;
  const Stream s = Stream::raw(seed).split(3000 + (uint64_t)attempt);
  for (int k = threadIdx.x; k < 252; k += WT<EXT>::THREADS) sm.ang[k] = angle_of(s.at((uint64_t)k));
  __syncthreads();
  overworld_gradients<EXT>(sm);
  int ld_unused;
  if (!gen_overworld<EXT>(sm, hash2(seed, 4000 + (uint64_t)attempt), false, attempt, &ld_unused)) return false;
  const UField u(hash2(seed, 13 + (uint64_t)attempt), 6);
  const uint8_t gem = floor == 6 ? B_RUBY : B_SAPPHIRE;
  for (int t = threadIdx.x; t < T::HW; t += WT<EXT>::THREADS) {
    uint8_t b = sm.blk[t], d = b;
    if (floor == 6) {
      if (b == B_GRASS) d = B_FIRE_GRASS; else if (b == B_TREE) d = B_FIRE_TREE;
      else if (b == B_WATER) d = B_LAVA; else if (b == B_SAND) d = B_GRAVEL;
    } else {
      if (b == B_GRASS) d = B_ICE_GRASS; else if (b == B_TREE) d = B_ICE_SHRUB;
      else if (b == B_SAND) d = B_GRAVEL; else if (b == B_LAVA) d = B_WATER;
    }
    if (d == B_STONE && u(t) > 0.975f) d = gem;
    sm.blk[t] = d;
  }
  __syncthreads();
  if (!ensure_f32<EXT>(sm, gem, u, false, -1)) return false;
  const int spawn = nearest_walkable(sm);
  if (spawn < 0) return false;
  const int sr = spawn / T::W, sc = spawn % T::W;
  const int tpos = pick(sm, [&](int t) {
    return in_set(WALK_SET, sm.blk[t]) && cheb(t / T::W, t % T::W, sr, sc) <= 8;
  }, u);
  if (tpos < 0 || tpos == spawn) return false;
  if (threadIdx.x == 0) sm.blk[tpos] = floor == 6 ? B_ENCHANT_FIRE : B_ENCHANT_ICE;
  __syncthreads();
  int down = pick(sm, [&](int t) {
    return in_set(WALK_SET, sm.blk[t]) && cheb(t / T::W, t % T::W, sr, sc) >= 10;
  }, u);
  if (down < 0)   // _pick_tile(out, walk, 1.0 - u)
    down = pick(sm, [&](int t) { return in_set(WALK_SET, sm.blk[t]); },
                [&](int t) { return __fsub_rn(1.0f, u(t)); });
  if (down < 0 || down == spawn) return false;
  for (int t = threadIdx.x; t < T::HW; t += WT<EXT>::THREADS) sm.itm[t] = 0;
  __syncthreads();
  if (threadIdx.x == 0) { sm.itm[spawn] = I_LADDER_UP; sm.itm[down] = I_LADDER_DOWN; }
  __syncthreads();
  fo->spawn = spawn; fo->lu = spawn; fo->ld = down;
  return true;
}

// worldgen._carve_line
template <bool EXT>
__device__ void carve(WSmem<EXT>& sm, int r, int c, int tr, int tc) {
  using T = WT<EXT>;
  while (c != tc) { c += tc > c ? 1 : -1; sm.blk[r * T::W + c] = B_PATH; }
  while (r != tr) { r += tr > r ? 1 : -1; sm.blk[r * T::W + c] = B_PATH; }
}

// worldgen._gen_dungeon (:367-406)
template <bool EXT>
__device__ __noinline__ bool gen_dungeon(WSmem<EXT>& sm, uint64_t seed, int floor, int attempt, FloorOut* fo) {
  using T = WT<EXT>;
  // The randint chain draws hash2(key, counter) with counter 0 for the room
  // count and 1 + 4k .. 4 + 4k for room k, so the rooms are independent:
  // thread k rolls room k.
  const Stream s0 = Stream::raw(seed).split(1000 + (uint64_t)attempt);
  const int n = 4 + (int)(hash2(s0.key, 0) % 4ull);
  if (threadIdx.x < n) {
    const int k = threadIdx.x;
    const uint64_t c = 1 + 4 * (uint64_t)k;
    const int rh = 5 + (int)(hash2(s0.key, c) % 5ull), rw = 5 + (int)(hash2(s0.key, c + 1) % 5ull);
    const int r0 = 2 + (int)(hash2(s0.key, c + 2) % (uint64_t)(T::H - rh - 4));
    const int c0 = 2 + (int)(hash2(s0.key, c + 3) % (uint64_t)(T::W - rw - 4));
    sm.cr[k] = r0 + rh / 2;
    sm.cc[k] = c0 + rw / 2;
    sm.room[k][0] = r0; sm.room[k][1] = r0 + rh; sm.room[k][2] = c0; sm.room[k][3] = c0 + rw;
  }
  __syncthreads();
  // The attempt fails at the end unless both ladder tiles (the first and last
  // room centres, always PATH after carving) stay PATH: the sewer water /
  // vault gravel pass below turns a PATH tile with u > 0.82 / 0.85 into
  // water / gravel, and the two must differ.  Those outcomes are known now,
  // so a doomed attempt (a third of floor-3 / floor-4 attempts) returns
  // here instead of after the tile passes -- same result, same next attempt.
  const UField u(hash2(seed, 7 + (uint64_t)attempt), 4);
  bool doomed;
  {
    const int up = sm.cr[0] * T::W + sm.cc[0], down = sm.cr[n - 1] * T::W + sm.cc[n - 1];
    const float thr = floor == 3 ? 0.82f : floor == 4 ? 0.85f : 2.0f;
    doomed = up == down || u(up) > thr || u(down) > thr;
  }
  __syncthreads();   // every thread has read the centres before a returning one rewrites them
  if (doomed) return false;
  // the rooms as one column bitmask per row, then one lookup per tile
  for (int r = threadIdx.x; r < T::H; r += WT<EXT>::THREADS) {
    uint64_t m = 0;
    for (int k = 0; k < n; ++k)
      if (r >= sm.room[k][0] && r < sm.room[k][1])
        m |= ((1ull << (sm.room[k][3] - sm.room[k][2])) - 1ull) << sm.room[k][2];
    sm.rowmask[r] = m;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < T::HW; t += WT<EXT>::THREADS) {
    const int r = t / T::W, c = t % T::W;
    const bool in = (sm.rowmask[r] >> c) & 1ull;
    sm.blk[t] = in ? B_PATH : B_WALL;
    sm.itm[t] = 0;
  }
  __syncthreads();
  // L-corridors between consecutive rooms: every write is PATH, so the
  // corridors can be carved concurrently, one thread each
  if (threadIdx.x + 1 < n) {
    const int k = threadIdx.x;
    carve<EXT>(sm, sm.cr[k], sm.cc[k], sm.cr[k + 1], sm.cc[k + 1]);
  }
  __syncthreads();
  // moss / sewer water / vault gravel read the pre-pass PATH mask: compute
  // into registers first, write after the barrier
  constexpr int PER = (T::HW + WT<EXT>::THREADS - 1) / WT<EXT>::THREADS;
  uint8_t nb[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int t = threadIdx.x + q * WT<EXT>::THREADS;
    if (t >= T::HW) break;
    const int r = t / T::W, c = t % T::W;
    const float uu = u(t);
    const uint8_t b = sm.blk[t];
    const bool path = b == B_PATH;
    const bool near_path = path || (r > 0 && sm.blk[t - T::W] == B_PATH) || (r < T::H - 1 && sm.blk[t + T::W] == B_PATH) ||
                           (c > 0 && sm.blk[t - 1] == B_PATH) || (c < T::W - 1 && sm.blk[t + 1] == B_PATH);
    uint8_t d = b;
    if (b == B_WALL && near_path && uu < 0.25f) d = B_WALL_MOSS;
    if (floor == 3 && path && uu > 0.82f) d = B_WATER;
    if (floor == 4 && path && uu > 0.85f) d = B_GRAVEL;
    nb[q] = d;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int t = threadIdx.x + q * WT<EXT>::THREADS;
    if (t < T::HW) sm.blk[t] = nb[q];
  }
  __syncthreads();
  const int fountain = pick(sm, [&](int t) { return sm.blk[t] == B_PATH; }, u);
  if (fountain >= 0 && threadIdx.x == 0) sm.blk[fountain] = B_FOUNTAIN;
  __syncthreads();
  const int up = sm.cr[0] * T::W + sm.cc[0], down = sm.cr[n - 1] * T::W + sm.cc[n - 1];
  const bool ok = sm.blk[up] == B_PATH && sm.blk[down] == B_PATH && up != down;
  __syncthreads();
  if (!ok) return false;
  if (threadIdx.x == 0) { sm.itm[up] = I_LADDER_UP; sm.itm[down] = I_LADDER_DOWN; }
  __syncthreads();
  fo->spawn = up; fo->lu = up; fo->ld = down;
  return true;
}

// perlin._profiles in float64 for the cave octaves (res 4 and 8)
template <bool EXT>
__device__ void build_profiles_f64(WSmem<EXT>& sm) {
  const int H = WT<EXT>::H;
  const int dims[2] = {H / 4, H / 8};
  for (int k = threadIdx.x; k < 2 * 12; k += WT<EXT>::THREADS) {
    const int o = k / 12, i = k % 12, d = dims[o];
    if (i >= d) continue;
    double f = __ddiv_rn((double)i, (double)d);
    double u = __dmul_rn(__dmul_rn(__dmul_rn(f, f), f),
                         __dadd_rn(__dmul_rn(f, __dsub_rn(__dmul_rn(f, 6.0), 15.0)), 10.0));
    const double one = 1.0, root2 = 1.4142135623730951;
    sm.dprof[o][0][i] = __dsub_rn(one, u);
    sm.dprof[o][1][i] = __dmul_rn(__dsub_rn(one, u), f);
    sm.dprof[o][2][i] = u;
    sm.dprof[o][3][i] = __dmul_rn(u, __dsub_rn(f, one));
    sm.dprof[o][4][i] = __dmul_rn(__dmul_rn(__dsub_rn(one, u), f), root2);
    sm.dprof[o][5][i] = __dmul_rn(__dsub_rn(one, u), root2);
    sm.dprof[o][6][i] = __dmul_rn(__dmul_rn(u, __dsub_rn(f, one)), root2);
    sm.dprof[o][7][i] = __dmul_rn(u, root2);
  }
}

template <bool EXT>
__device__ __forceinline__ double octave_at_d(const WSmem<EXT>& sm, int o, const double* gx, const double* gy,
                                              int res, int r, int c) {
  const int d = WT<EXT>::H / res;
  const int R = r / d, i = r % d, C = c / d, j = c % d, n = res + 1;
  const double* P = &sm.dprof[o][0][0];
  const double a1 = P[0 * 12 + i], a2 = P[1 * 12 + i], a3 = P[2 * 12 + i], a4 = P[3 * 12 + i];
  const double b0 = P[4 * 12 + j], b1 = P[5 * 12 + j], b2 = P[6 * 12 + j], b3 = P[7 * 12 + j];
  const int k00 = R * n + C, k10 = (R + 1) * n + C;
  double t0 = __dadd_rn(__dmul_rn(gx[k00], a1), __dmul_rn(gx[k10], a3));
  double t1 = __dadd_rn(__dmul_rn(gy[k00], a2), __dmul_rn(gy[k10], a4));
  double t2 = __dadd_rn(__dmul_rn(gx[k00 + 1], a1), __dmul_rn(gx[k10 + 1], a3));
  double t3 = __dadd_rn(__dmul_rn(gy[k00 + 1], a2), __dmul_rn(gy[k10 + 1], a4));
  return __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(t0, b0), __dmul_rn(t1, b1)), __dmul_rn(t2, b2)), __dmul_rn(t3, b3));
}

// perlin.perlin with CAVE_OCTAVES in float64 at one tile
template <bool EXT>
__device__ __forceinline__ double cave_field_at(const WSmem<EXT>& sm, int t) {
  const int r = t / WT<EXT>::W, c = t % WT<EXT>::W;
  const double o1 = octave_at_d<EXT>(sm, 0, sm.dgx, sm.dgy, 4, r, c);
  const double o2 = octave_at_d<EXT>(sm, 1, sm.dgx + 25, sm.dgy + 25, 8, r, c);
  return __ddiv_rn(__dadd_rn(__dmul_rn(1.0, o1), __dmul_rn(0.5, o2)), 1.5);
}

// worldgen._gen_cave (:418-468)
template <bool EXT>
__device__ __noinline__ bool gen_cave(WSmem<EXT>& sm, uint64_t seed, int floor, int attempt, FloorOut* fo) {
  using T = WT<EXT>;
  const Stream s = Stream::raw(seed).split(2000 + (uint64_t)attempt);
  for (int k = threadIdx.x; k < 106; k += WT<EXT>::THREADS) {
    const float a = angle_of(s.at((uint64_t)k));
    sm.dgx[k] = gl_cos((double)a);   // np.cos / np.sin in float64 = glibc
    sm.dgy[k] = gl_sin((double)a);
  }
  __syncthreads();
  const UField u(hash2(seed, 11 + (uint64_t)attempt), 5);
  for (int t = threadIdx.x; t < T::HW; t += WT<EXT>::THREADS) {
    const double field = cave_field_at<EXT>(sm, t);
    const float uu = u(t);
    const bool open = field > -0.02;
    uint8_t b = open ? B_PATH : B_STONE;
    if (open && uu < 0.04f) b = B_STALAGMITE;
    if (b == B_STONE) {
      if (floor == 2) {
        if (uu < 0.06f) b = B_COAL;
        if (uu >= 0.90f && uu < 0.93f) b = B_IRON;
        if (uu >= 0.975f) b = B_SAPPHIRE;
      } else {
        if (uu < 0.05f) b = B_COAL;
        if (uu >= 0.90f && uu < 0.93f) b = B_IRON;
        if (uu >= 0.96f && uu < 0.975f) b = B_DIAMOND;
        if (uu >= 0.985f) b = B_RUBY;
      }
    }
    if (floor != 2 && field < -0.62) b = B_LAVA;
    sm.blk[t] = b;
    sm.itm[t] = 0;
  }
  __syncthreads();
  const uint8_t must2[3] = {B_COAL, B_IRON, B_SAPPHIRE};
  const uint8_t must5[4] = {B_COAL, B_IRON, B_DIAMOND, B_RUBY};
  const int nm = floor == 2 ? 3 : 4;
  // each _ensure_block only ever adds its own ore, so one census serves all
  const unsigned long long cen0 = census(sm);
  for (int k = 0; k < nm; ++k) {
    const uint8_t b = floor == 2 ? must2[k] : must5[k];
    if ((cen0 >> b) & 1ull) continue;
    double bv = 0.0;
    int bi = INT_MAX;
    for (int t = threadIdx.x; t < T::HW; t += WT<EXT>::THREADS)
      if (sm.blk[t] == B_STONE) {
        const double sc = -cave_field_at<EXT>(sm, t);
        if (bi == INT_MAX || sc > bv) { bv = sc; bi = t; }
      }
    const int pos = block_argmax_d(sm, bv, bi);
    if (pos < 0) return false;   // no stone and caves hold no grass / trees
    if (threadIdx.x == 0) sm.blk[pos] = b;
    __syncthreads();
  }
  int cnt = 0;
  for (int t = threadIdx.x; t < T::HW; t += WT<EXT>::THREADS) cnt += sm.blk[t] == B_PATH;
  int total;
  block_excl_scan(sm, cnt, &total);
  if (total < 40) return false;
  const int up = pick(sm, [&](int t) { return sm.blk[t] == B_PATH; }, u);
  if (up < 0) return false;
  const int ur = up / T::W, uc = up % T::W;
  // argmax of chebyshev(up)/max over open tiles == argmax of the distance
  unsigned long long best = ~0ull;
  for (int t = threadIdx.x; t < T::HW; t += WT<EXT>::THREADS)
    if (sm.blk[t] == B_PATH) {
      unsigned long long k = ((unsigned long long)(1000 - cheb(t / T::W, t % T::W, ur, uc)) << 32) | (unsigned)t;
      best = k < best ? k : best;
    }
  best = block_min_u64(sm, best);
  const int down = (int)(best & 0xFFFFFFFFull);
  if (best == ~0ull || down == up) return false;
  if (threadIdx.x == 0) {
    carve<EXT>(sm, ur, uc, down / T::W, down % T::W);
    sm.blk[up] = B_PATH;
    sm.blk[down] = B_PATH;
    sm.itm[up] = I_LADDER_UP;
    sm.itm[down] = I_LADDER_DOWN;
  }
  __syncthreads();
  fo->spawn = up; fo->lu = up; fo->ld = down;
  return true;
}

// worldgen._gen_graveyard (:523-546)
template <bool EXT>
__device__ __noinline__ void gen_graveyard(WSmem<EXT>& sm, FloorOut* fo) {
  using T = WT<EXT>;
  const int cr = T::H / 2, cc = T::W / 2;
  for (int t = threadIdx.x; t < T::HW; t += WT<EXT>::THREADS) {
    const int r = t / T::W, c = t % T::W;
    uint8_t b = B_DARKNESS;
    if (r >= cr - 10 && r <= cr + 10 && c >= cc - 10 && c <= cc + 10) b = B_WALL;
    if (r > cr - 10 && r < cr + 10 && c > cc - 10 && c < cc + 10) b = B_PATH;
    sm.blk[t] = b;
    sm.itm[t] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int go[12][2] = {{-3, -5}, {-3, 5}, {0, -7}, {0, 7}, {3, -4}, {3, 4},
                           {5, 0}, {-5, -2}, {-5, 2}, {6, -6}, {6, 6}, {2, 0}};
    for (int k = 0; k < 12; ++k) sm.blk[(cr + go[k][0]) * T::W + cc + go[k][1]] = B_GRAVE + k % 3;
    for (int r = cr + 4; r < cr + 7; ++r)
      for (int c = cc - 5; c < cc - 2; ++c) sm.blk[r * T::W + c] = B_WATER;
    sm.blk[(cr - 6) * T::W + cc] = B_NECROMANCER;
    const int up = (cr + 10 - 2) * T::W + cc;
    sm.blk[up] = B_PATH;
    sm.itm[up] = I_LADDER_UP;
  }
  __syncthreads();
  const int up = (cr + 8) * T::W + cc;
  fo->spawn = up; fo->lu = up; fo->ld = -1;
}

// worldgen._template_floor (:549-575)
template <bool EXT>
__device__ __noinline__ void gen_template(WSmem<EXT>& sm, int floor, FloorOut* fo) {
  using T = WT<EXT>;
  const int H = T::H, W = T::W, cr = H / 2, cc = W / 2;
  for (int t = threadIdx.x; t < T::HW; t += WT<EXT>::THREADS) {
    const int r = t / W, c = t % W;
    uint8_t b = floor == 0 ? B_GRASS : B_PATH;
    if (floor != 0 && (r == 0 || r == H - 1 || c == 0 || c == W - 1)) b = B_WALL;
    if (floor == 0) {
      if (r >= 2 && r < 5 && c >= 2 && c < 5) b = B_WATER;
      if (r >= 6 && r < 8 && c >= 2 && c < 6) b = B_SAND;
      if (r == cr - 4 && c == cc) b = B_TREE;
      if (r >= H - 6 && r < H - 2 && c >= W - 6 && c < W - 2) b = B_STONE;
      if (r == H - 5 && c == W - 5) b = B_COAL;
      if (r == H - 4 && c == W - 4) b = B_IRON;
      if (r == H - 3 && c == W - 3) b = B_DIAMOND;
      if (r == H - 6 && c == W - 3) b = B_LAVA;
    }
    sm.blk[t] = b;
    sm.itm[t] = 0;
  }
  __syncthreads();
  fo->spawn = cr * W + cc;
  fo->lu = floor != 0 ? cr * W + cc - 5 : -1;
  fo->ld = floor != 8 ? cr * W + cc + 5 : -1;
  if (threadIdx.x == 0) {
    if (fo->lu >= 0) sm.itm[fo->lu] = I_LADDER_UP;
    if (fo->ld >= 0) sm.itm[fo->ld] = I_LADDER_DOWN;
  }
  __syncthreads();
}

// worldgen._assign_chests for one floor (:598-623)
template <bool EXT>
__device__ __noinline__ void assign_chests(WSmem<EXT>& sm, uint64_t world_seed, int f, WMeta* meta) {
  using T = WT<EXT>;
  const int per_floor[9] = {0, 4, 2, 3, 3, 2, 2, 2, 0};
  const int nc = per_floor[f];
  if (nc == 0) {
    if (threadIdx.x == 0) meta->nch[f] = 0;
    return;
  }
  // the row-major list of PATH tiles (np.nonzero) via a block scan
  constexpr int PER = (T::HW + WT<EXT>::THREADS - 1) / WT<EXT>::THREADS;
  const int t0 = threadIdx.x * PER, t1 = min(t0 + PER, T::HW);
  int cnt = 0;
  for (int t = t0; t < t1; ++t) cnt += sm.blk[t] == B_PATH;
  int len;
  int off = block_excl_scan(sm, cnt, &len);
  for (int t = t0; t < t1; ++t)
    if (sm.blk[t] == B_PATH) sm.list[off++] = (uint16_t)t;
  __syncthreads();
  if (threadIdx.x == 0) {
    int nl = 0;
    if (len) {
      Stream s = Stream::raw(world_seed).split(5000 + (uint64_t)f);
      const int lim = min(min(nc, 6), len);
      for (int k = 0; k < lim; ++k) {
        const int t = sm.list[s.randint(0, len)];
        if (sm.blk[t] != B_PATH || sm.itm[t] != I_EMPTY) continue;
        sm.blk[t] = B_CHEST;
        int loot, qty;
        if (f == 1 && nl == 0) { loot = LOOT_BOW; qty = 1; }
        else if (f == 1 && nl == 1) { loot = LOOT_BOOK; qty = 1; }
        else {
          const double u = s.uniform01();
          // _weighted_loot: cumulative weights accumulated in float64
          double acc = 0.0;
          const int kinds[4] = {LOOT_POTION, LOOT_ARROWS, LOOT_TORCHES, LOOT_BOOK};
          const int qtys[4] = {1, 3, 4, 1};
          const double wts[4] = {0.40, 0.25, 0.20, 0.15};
          loot = kinds[3]; qty = qtys[3];
          for (int q = 0; q < 4; ++q) {
            acc = __dadd_rn(acc, wts[q]);
            if (u < acc) { loot = kinds[q]; qty = qtys[q]; break; }
          }
        }
        meta->chest[f][nl][0] = (int16_t)(t / T::W);
        meta->chest[f][nl][1] = (int16_t)(t % T::W);
        meta->chest[f][nl][2] = (int16_t)loot;
        meta->chest[f][nl][3] = (int16_t)qty;
        ++nl;
      }
    }
    meta->nch[f] = (uint8_t)nl;
  }
  __syncthreads();
}

template <bool EXT>
__global__ void __launch_bounds__(WT<EXT>::THREADS, WT<EXT>::MINB) k_worldgen(WorldJob job) {
  using T = WT<EXT>;
  __shared__ WSmem<EXT> sm;
  // mode 1: pool worlds [w0, n_pool) (w0 > 0: the speculative pass made the
  // rest); mode 3: the speculative pass, worlds [0, spec_k)
  int64_t w0 = 0, nworlds = job.count;
  uint64_t spec_key = 0;
  if (job.mode == 1) {
    const int64_t np = (int64_t)job.info->n_pool;
    w0 = job.spec_k ? (int64_t)min(*job.spec_k, (int32_t)np) : 0;
    nworlds = np - w0;
  } else if (job.mode == 3) {
    nworlds = *job.spec_k;
    spec_key = hash2(job.pool_key, (uint64_t)(*job.dstep + 1));   // = this step's StepInfo.step_key
  }
  const int64_t items = nworlds * T::F;
  // a CTA without an item leaves before building its noise tables: the
  // pool's remainder pass is usually empty when the speculative pass ran
  // (1,024 extended envs: 5.8 us of table building on the step's critical path)
  if ((int64_t)blockIdx.x >= items) return;
  build_profiles_f32<EXT>(sm);
  if (EXT) build_profiles_f64<EXT>(sm);
  __syncthreads();
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    // floor-major order: CTAs resident at the same time run the same floor
    // generator, which keeps the instruction cache warm (no_instructions
    // stalls dominated a world-major order)
    const int f = (int)(it / nworlds);
    const int64_t w = (it % nworlds) + (job.mode == 2 ? job.first : w0);   // output slot
    uint64_t seed, key;
    if (job.mode == 0) {
      seed = hash2(job.env_key, hash2((uint64_t)(job.env_offset + w), 0));
      key = hash2(seed, hash2(1, 0));
    } else if (job.mode == 1) {
      const int64_t slot = ((int64_t)job.info->offset + w) % job.M;
      seed = hash2(job.info->step_key, (uint64_t)slot);
      key = hash2(job.info->step_key, (1ull << 32) + (uint64_t)slot);
    } else if (job.mode == 3) {   // one shard: offset 0, w < cap <= M
      seed = hash2(spec_key, (uint64_t)w);
      key = hash2(spec_key, (1ull << 32) + (uint64_t)w);
    } else {
      seed = job.params.seed[w];
      key = 0;   // levels get their install key when installed
    }
    WMeta* meta = job.out.meta + w;
    // make_level_params (worldgen.py:75-87), or the explicit params
    const uint64_t base = mix64(seed);
    const uint64_t fseed = job.mode == 2 ? job.params.floor_seed[w * 9 + f] : hash2(base, hash2(100 + (uint64_t)f, 0));
    FloorOut fo{-1, -1, -1};
    int attempt = 0;
    bool ok = false;
    if (f == 0) {
      const uint64_t k1 = hash2(base, hash2(1, 0));
      for (int k = threadIdx.x; k < 252; k += WT<EXT>::THREADS)
        sm.ang[k] = job.mode == 2 ? job.params.angles[w * 252 + k] : angle_of(u64d(k1, (uint64_t)k));
      __syncthreads();
      overworld_gradients<EXT>(sm);
      for (attempt = 0; attempt < job.max_attempts && !ok; ++attempt) {
        int ld;
        ok = gen_overworld<EXT>(sm, fseed, EXT, attempt, &ld);
        if (ok) { fo.spawn = sm.spawn; fo.ld = ld; fo.lu = -1; }
      }
    } else if (f == 1 || f == 3 || f == 4) {
      for (attempt = 0; attempt < job.max_attempts && !ok; ++attempt) ok = gen_dungeon<EXT>(sm, fseed, f, attempt, &fo);
    } else if (f == 2 || f == 5) {
      for (attempt = 0; attempt < job.max_attempts && !ok; ++attempt) ok = gen_cave<EXT>(sm, fseed, f, attempt, &fo);
    } else if (f == 6 || f == 7) {
      for (attempt = 0; attempt < job.max_attempts && !ok; ++attempt) ok = gen_realm<EXT>(sm, fseed, f, attempt, &fo);
    } else if (job.max_attempts > 0) {
      gen_graveyard<EXT>(sm, &fo);
      ok = true;
      attempt = 1;
    }
    uint32_t flags = 0;
    if (attempt > 1) flags |= WG_FLAG_RETRY;
    if (!ok) {
      gen_template<EXT>(sm, f, &fo);
      flags |= WG_FLAG_TEMPLATE | (WG_FLAG_TEMPLATE_F0 << f);
    }
    if (EXT && f >= 1 && f <= 7) assign_chests<EXT>(sm, seed, f, meta);
    // write the floor out (16-byte vectors)
    uint8_t* ob = job.out.blocks + ((size_t)w * T::F + f) * T::HW;
    uint8_t* oi = job.out.items + ((size_t)w * T::F + f) * T::HW;
    for (int q = threadIdx.x; q < T::HW / 16; q += WT<EXT>::THREADS) {
      reinterpret_cast<uint4*>(ob)[q] = reinterpret_cast<const uint4*>(sm.blk)[q];
      reinterpret_cast<uint4*>(oi)[q] = reinterpret_cast<const uint4*>(sm.itm)[q];
    }
    if (threadIdx.x == 0) {
      meta->ld[f][0] = (int16_t)(fo.ld >= 0 ? fo.ld / T::W : -1);
      meta->ld[f][1] = (int16_t)(fo.ld >= 0 ? fo.ld % T::W : -1);
      meta->lu[f][0] = (int16_t)(fo.lu >= 0 ? fo.lu / T::W : -1);
      meta->lu[f][1] = (int16_t)(fo.lu >= 0 ? fo.lu % T::W : -1);
      if (f == 0) {
        meta->spawn[0] = (int16_t)(fo.spawn / T::W);
        meta->spawn[1] = (int16_t)(fo.spawn % T::W);
        meta->seed = seed;
        meta->key = key;
        // potion permutation: argsort of six hashed float32 draws
        const uint32_t pk = (uint32_t)(hash2(seed, 42) & 0xFFFFFFFFull);
        float v[6];
        uint8_t idx[6];
        bool tie = false;
        for (int q = 0; q < 6; ++q) v[q] = u32f(pk, (uint32_t)q);
        for (int a = 0; a < 6; ++a)
          for (int b = a + 1; b < 6; ++b) tie |= v[a] == v[b];
        np_argsort6(v, idx);   // numpy's tie order, not a stable sort (gr_device.cuh)
        for (int a = 0; a < 6; ++a) meta->potion[a] = idx[a];
        if (tie) flags |= WG_FLAG_POTION_TIE;   // counted only: ties are reproduced
        if (!EXT) meta->nch[0] = 0;
      }
      if (flags) {
        atomicOr(&meta->flags, flags);
        if (job.counters) {
          if (flags & WG_FLAG_RETRY) atomicAdd(&job.counters[1], 1ull);
          if (flags & WG_FLAG_TEMPLATE) atomicAdd(&job.counters[2], 1ull);
          if (flags & WG_FLAG_POTION_TIE) atomicAdd(&job.counters[3], 1ull);
        }
      }
      if (f == 0 && job.counters) atomicAdd(&job.counters[0], 1ull);
    }
    __syncthreads();
  }
}

// make_level_params (worldgen.py:75-87): 252 angles f32(u * 2 pi) from
// split(make_stream(seed), 1) and the floor seeds split(base, 100 + f).key
__global__ void k_level_params(LevelParamsBuf p, int64_t first, int64_t count) {
  const int64_t l = first + blockIdx.x;
  if (blockIdx.x >= count) return;
  const uint64_t base = mix64(p.seed[l]);
  const uint64_t k1 = hash2(base, hash2(1, 0));
  for (int k = threadIdx.x; k < 252; k += blockDim.x) p.angles[l * 252 + k] = angle_of(u64d(k1, (uint64_t)k));
  for (int f = threadIdx.x; f < 9; f += blockDim.x) p.floor_seed[l * 9 + f] = hash2(base, hash2(100 + (uint64_t)f, 0));
}

void launch_level_params(const LevelParamsBuf& p, int64_t first, int64_t count, cudaStream_t st) {
  if (count > 0) k_level_params<<<(unsigned)count, 128, 0, st>>>(p, first, count);
}

void launch_worldgen(bool ext, const WorldJob& j, cudaStream_t st) {
#if !GR_WG_WIDE
  if (ext && j.wide) {
    wide::launch_worldgen(ext, j, st);
    return;
  }
#endif
  // persistent grid: CTAs walk the (world, floor) items
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t max_items = (j.mode == 1 || j.mode == 3 ? j.out.cap : j.count) * (ext ? 9 : 1);
  int grid = (int)std::min<int64_t>(max_items, (int64_t)sms * (j.ctas_per_sm > 0 ? j.ctas_per_sm
                                                                : ext ? WT<true>::MINB : WT<false>::MINB));
  if (grid <= 0) return;
  if (j.pdl) {   // starts once every CTA of the preceding kernel (k_step) is resident
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(ext ? WT<true>::THREADS : WT<false>::THREADS);
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (ext) cudaLaunchKernelEx(&cfg, k_worldgen<true>, j);
    else cudaLaunchKernelEx(&cfg, k_worldgen<false>, j);
    return;
  }
  if (ext) k_worldgen<true><<<grid, WT<true>::THREADS, 0, st>>>(j);
  else k_worldgen<false><<<grid, WT<false>::THREADS, 0, st>>>(j);
}

#if GR_WG_WIDE
}  // namespace wide
#endif
}  // namespace gr
