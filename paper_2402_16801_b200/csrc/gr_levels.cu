// gr_levels.cu -- level buffers for curriculum methods (UED): the mutation
// operators of mutate.py on device, and installing a level into chosen envs.
//
//   mutate_noise  (mutate.py:36-44)   every overworld angle + U(-s, s), mod 2 pi
//   mutate_swap   (mutate.py:58-72)   swap two overworld tiles, the first in
//                                     the centred 16x16 window
//   mutate_rswap  (mutate.py:75-103)  the class-restricted swap (ores with
//                                     ores, grass with trees)
//   install       (state.install_world, state.py:169-249) level -> env slot
//
// A mutation is one (level, stream) pair; each stream is the reference's
// RngStream (key, counter), so the draws (hash2(key, counter + j)) are the
// reference's.  Worlds are regenerated from mutated params by k_worldgen's
// explicit-params mode (gr_world.cu).
#include <cstdint>
#include <algorithm>
#include "gr_device.cuh"
#include "gr_state.cuh"
#include "gr_kernels.cuh"
#include "gr_levels.cuh"

namespace gr {

template <bool EXT>
struct LT {
  static constexpr int H = EXT ? 48 : 64, W = H, HW = H * W, F = EXT ? 9 : 1;
  // _central_window (mutate.py:47-51), SWAP_WINDOW = 16
  static constexpr int R0 = H / 2 - 8 > 0 ? H / 2 - 8 : 0, C0 = W / 2 - 8 > 0 ? W / 2 - 8 : 0;
  static constexpr int R1 = R0 + 16 < H ? R0 + 16 : H, C1 = C0 + 16 < W ? C0 + 16 : W;
};

// rng.randint (rng.py:126-131): lo + hash2(key, counter) % (hi - lo)
__device__ __forceinline__ int64_t randint(uint64_t key, uint64_t& ctr, int64_t lo, int64_t hi) {
  const uint64_t raw = hash2(key, ctr);
  ctr += 1;
  return lo + (int64_t)(raw % (uint64_t)(hi - lo));
}

// RSWAP_CLASSES (mutate.py:29-32): 0 ores / stone, 1 grass / tree, -1 other
__device__ __forceinline__ int rswap_class(uint8_t b) {
  if (b == B_STONE || b == B_COAL || b == B_IRON || b == B_DIAMOND || b == B_SAPPHIRE || b == B_RUBY) return 0;
  if (b == B_GRASS || b == B_TREE) return 1;
  return -1;
}

// mutate_noise on the params of level idx[m]: one thread per angle
__global__ void k_mutate_noise(LevelParamsBuf p, const int64_t* idx, const uint64_t* key, const uint64_t* ctr,
                               int64_t count, double scale) {
  const int64_t m = blockIdx.x;
  if (m >= count) return;
  const double two_pi = 2.0 * 3.141592653589793;
  const int64_t l = idx[m];
  for (int j = threadIdx.x; j < 252; j += blockDim.x) {
    // uniform_array consumes one counter per value, grid after grid
    const double delta = u64d(key[m], ctr[m] + (uint64_t)j);
    const double x = __dadd_rn((double)p.angles[l * 252 + j], __dmul_rn(__dsub_rn(__dmul_rn(delta, 2.0), 1.0), scale));
    // np.mod (npy_divmod): fmod, then the sign of the divisor
    double r = fmod(x, two_pi);
    if (r != 0.0) {
      if (r < 0.0) r = __dadd_rn(r, two_pi);
    } else {
      r = 0.0;
    }
    p.angles[l * 252 + j] = __double2float_rn(r);
  }
}

// mutate_swap: one thread per mutation (sequential draws)
template <bool EXT>
__global__ void k_mutate_swap(WBuf w, const int64_t* idx, const uint64_t* key, const uint64_t* ctr0, int64_t count) {
  using T = LT<EXT>;
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= count) return;
  uint8_t* blk = w.blocks + (size_t)idx[m] * T::F * T::HW;   // floor 0
  const uint64_t k = key[m];
  uint64_t c = ctr0[m];
  const int ar = (int)randint(k, c, T::R0, T::R1), ac = (int)randint(k, c, T::C0, T::C1);
  int br, bc;
  do {
    br = (int)randint(k, c, 0, T::H);
    bc = (int)randint(k, c, 0, T::W);
  } while (br == ar && bc == ac);
  const uint8_t t = blk[ar * T::W + ac];
  blk[ar * T::W + ac] = blk[br * T::W + bc];
  blk[br * T::W + bc] = t;
}

// index of the n-th (0-based) set lane over a warp-strided scan: helper for
// "the n-th tile of a row-major np.nonzero" (returns -1 past the end)
template <class Pred>
__device__ __forceinline__ int nth_match(int begin_count, int n, int total, Pred pred) {
  const int lane = threadIdx.x & 31;
  int seen = 0;
  for (int base = 0; base < total; base += 32) {
    const int t = base + lane;
    const bool hit = t < total && pred(t);
    const unsigned b = __ballot_sync(0xffffffffu, hit);
    const int c = __popc(b);
    if (n < seen + c) {
      // the (n - seen)-th set bit of b
      unsigned x = b;
      for (int k = 0; k < n - seen; ++k) x &= x - 1;
      return base + __ffs(x) - 1;
    }
    seen += c;
  }
  (void)begin_count;
  return -1;
}

template <class Pred>
__device__ __forceinline__ int count_matches(int total, Pred pred) {
  const int lane = threadIdx.x & 31;
  int cnt = 0;
  for (int base = 0; base < total; base += 32) {
    const int t = base + lane;
    cnt += __popc(__ballot_sync(0xffffffffu, t < total && pred(t)));
  }
  return cnt;
}

// mutate_rswap: one warp per mutation
template <bool EXT>
__global__ void k_mutate_rswap(WBuf w, const int64_t* idx, const uint64_t* key, const uint64_t* ctr0, int64_t count) {
  using T = LT<EXT>;
  const int64_t m = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (m >= count) return;   // warp-uniform
  uint8_t* blk = w.blocks + (size_t)idx[m] * T::F * T::HW;
  const uint64_t k = key[m];
  uint64_t c = ctr0[m];
  constexpr int WW = T::C1 - T::C0, WN = (T::R1 - T::R0) * WW;
  auto in_win = [&](int t) { return rswap_class(blk[(T::R0 + t / WW) * T::W + T::C0 + t % WW]) >= 0; };
  const int nwin = count_matches(WN, in_win);
  if (nwin == 0) return;
  const int i = (int)randint(k, c, 0, nwin);
  const int tw = nth_match(0, i, WN, in_win);
  const int ar = T::R0 + tw / WW, ac = T::C0 + tw % WW;
  const int cls = rswap_class(blk[ar * T::W + ac]);
  auto same = [&](int t) { return t != ar * T::W + ac && rswap_class(blk[t]) == cls; };
  const int nsame = count_matches(T::HW, same);
  if (nsame == 0) return;
  const int j = (int)randint(k, c, 0, nsame);
  const int tb = nth_match(0, j, T::HW, same);
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    const uint8_t t = blk[ar * T::W + ac];
    blk[ar * T::W + ac] = blk[tb];
    blk[tb] = t;
  }
}

void launch_mutate(bool ext, int op, const LevelParamsBuf& p, const WBuf& w, const int64_t* idx, const uint64_t* key,
                   const uint64_t* ctr, int64_t count, double scale, cudaStream_t st) {
  if (count <= 0) return;
  if (op == MUT_NOISE) {
    k_mutate_noise<<<(unsigned)count, 128, 0, st>>>(p, idx, key, ctr, count, scale);
  } else if (op == MUT_SWAP) {
    const unsigned g = (unsigned)((count + 127) / 128);
    if (ext) k_mutate_swap<true><<<g, 128, 0, st>>>(w, idx, key, ctr, count);
    else k_mutate_swap<false><<<g, 128, 0, st>>>(w, idx, key, ctr, count);
  } else {
    const unsigned g = (unsigned)((count * 32 + 127) / 128);
    if (ext) k_mutate_rswap<true><<<g, 128, 0, st>>>(w, idx, key, ctr, count);
    else k_mutate_rswap<false><<<g, 128, 0, st>>>(w, idx, key, ctr, count);
  }
}

}  // namespace gr
