// PPO minibatch objective, forward and gradient in one kernel (the learner
// of SURVEY.md 8(f) f1; not part of the env step).
//
// The eager objective in ppo.py is ~35 small kernels forward and as many
// backward per minibatch (log-softmax, gather, ratio, clipped surrogate,
// advantage normalisation, clipped value loss, entropy).  Here one launch
// computes, for a minibatch of B rows:
//   A_n   = (A - mean A) / (std A + 1e-8)           (std with Bessel's correction)
//   r     = exp(logp(a) - logp_old)
//   pg    = -mean(min(r A_n, clip(r, 1-e, 1+e) A_n))
//   vl    = 0.5 mean(max((v - R)^2, (V + clip(v - V, -e, e) - R)^2))
//   H     = mean(-sum_j p_j log p_j)
//   loss  = pg + c_v vl - c_e H
// and writes d loss / d logits [B, NA] and d loss / d v [B] (closed forms of
// the same branches the eager autograd takes), plus [loss, pg, vl, H].
// Every CTA recomputes the advantage mean / std over the whole minibatch
// (B floats, a few microseconds of L2 reads) so no second launch is needed;
// the four sums are accumulated with atomics into `out` (zeroed by the caller).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/gridrogue_ppo.h"

namespace {

constexpr int THREADS = 256;   // 8 rows (one warp each) per CTA pass

__device__ __forceinline__ float warp_sum(float x) {
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ float warp_max(float x) {
  for (int o = 16; o; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16(x); }

// logits / values of type TI with row strides ldl / ldv; gradients of type TO
// (bf16: what the head's GEMMs consume) with row stride ldd, the columns
// [NA, npad) of each gradient row written as zeros (a padded head)
template <int NA, typename TI, typename TO>
__global__ void __launch_bounds__(THREADS) k_ppo_loss(const TI* __restrict__ logits, int64_t ldl,
                                                      const TI* __restrict__ v, int64_t ldv,
                                                      const int64_t* __restrict__ act,
                                                      const float* __restrict__ logp_old,
                                                      const float* __restrict__ adv,
                                                      const float* __restrict__ v_old,
                                                      const float* __restrict__ ret, int B, float clip_eps,
                                                      float vf_coef, float ent_coef, TO* __restrict__ dlogits,
                                                      int64_t ldd, int npad, TO* __restrict__ dv, int64_t lddv,
                                                      float* __restrict__ out, const int64_t* __restrict__ index) {
  // index != null: the per-sample inputs (act, logp_old, adv, v_old, ret)
  // of minibatch row i are entry index[i] of the rollout-wide arrays
  auto src = [&](int i) -> int64_t { return index ? index[i] : (int64_t)i; };
  constexpr int PER = (NA + 31) / 32;
  __shared__ float red[2][THREADS / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // advantage mean and unbiased std over the minibatch
  float s = 0.f, s2 = 0.f;
  for (int i = threadIdx.x; i < B; i += THREADS) {
    const float a = adv[src(i)];
    s += a;
    s2 += a * a;
  }
  s = warp_sum(s);
  s2 = warp_sum(s2);
  if (lane == 0) {
    red[0][warp] = s;
    red[1][warp] = s2;
  }
  __syncthreads();
  float tot = 0.f, tot2 = 0.f;
#pragma unroll
  for (int w = 0; w < THREADS / 32; ++w) {
    tot += red[0][w];
    tot2 += red[1][w];
  }
  const float mean = tot / (float)B;
  const float var = fmaxf((tot2 - (float)B * mean * mean) / (float)(B > 1 ? B - 1 : 1), 0.f);
  const float inv_std = 1.f / (sqrtf(var) + 1e-8f);
  const float invB = 1.f / (float)B;

  float acc_pg = 0.f, acc_vl = 0.f, acc_h = 0.f;
  const int nw = gridDim.x * (THREADS / 32);
  for (int row = blockIdx.x * (THREADS / 32) + warp; row < B; row += nw) {
    const TI* z = logits + (size_t)row * ldl;
    float zl[PER];
    float m = -INFINITY;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int j = lane + 32 * k;
      zl[k] = j < NA ? to_f(z[j]) : -INFINITY;
      m = fmaxf(m, zl[k]);
    }
    m = warp_max(m);
    float se = 0.f;
#pragma unroll
    for (int k = 0; k < PER; ++k) se += lane + 32 * k < NA ? expf(zl[k] - m) : 0.f;
    se = warp_sum(se);
    const float lse = m + logf(se);
    // entropy H = -sum p log p
    float h = 0.f;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int j = lane + 32 * k;
      if (j < NA) {
        const float lp = zl[k] - lse;
        h -= expf(lp) * lp;
      }
    }
    h = warp_sum(h);
    const int64_t sr = src(row);
    const int a = (int)act[sr];
    float zsel = 0.f;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const float zk = __shfl_sync(0xffffffffu, zl[k], a & 31);
      if (k == a / 32) zsel = zk;
    }
    const float logp = zsel - lse;
    const float r = expf(logp - logp_old[sr]);
    const float an = (adv[sr] - mean) * inv_std;
    const float s1 = r * an;
    const float rc = fminf(fmaxf(r, 1.f - clip_eps), 1.f + clip_eps);
    const float s2c = rc * an;
    const float pg = -fminf(s1, s2c);
    // d pg_row / d logp (then / B): the branch min() took
    float g_logp;
    if (s1 <= s2c) g_logp = -an * r;
    else g_logp = (r > 1.f - clip_eps && r < 1.f + clip_eps) ? -an * r : 0.f;
    g_logp *= invB;
    // value loss
    const float vv = to_f(v[(size_t)row * ldv]), vo = v_old[sr], R = ret[sr];
    const float dvu = vv - vo;
    const float vc = vo + fminf(fmaxf(dvu, -clip_eps), clip_eps);
    const float e1 = (vv - R) * (vv - R), e2 = (vc - R) * (vc - R);
    const float vl = 0.5f * fmaxf(e1, e2);
    float g_v = e1 >= e2 ? (vv - R) : ((dvu > -clip_eps && dvu < clip_eps) ? (vc - R) : 0.f);
    g_v *= vf_coef * invB;
    // d loss / d z_j = g_logp (1[j==a] - p_j) + c_e/B p_j (log p_j + H)
    TO* dz = dlogits + (size_t)row * ldd;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int j = lane + 32 * k;
      if (j < NA) {
        const float lp = zl[k] - lse, p = expf(lp);
        dz[j] = from_f<TO>(g_logp * ((j == a ? 1.f : 0.f) - p) + ent_coef * invB * p * (lp + h));
      }
    }
    for (int j = NA + lane; j < npad; j += 32) dz[j] = from_f<TO>(0.f);
    if (lane == 0) {
      dv[(size_t)row * lddv] = from_f<TO>(g_v);
      acc_pg += pg;
      acc_vl += vl;
      acc_h += h;
    }
  }
  // CTA sums -> out (lane 0 of each warp holds its rows' sums)
  __syncthreads();
  if (lane == 0) {
    red[0][warp] = acc_pg;
    red[1][warp] = acc_vl;
  }
  __syncthreads();
  float cpg = 0.f, cvl = 0.f;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < THREADS / 32; ++w) {
      cpg += red[0][w];
      cvl += red[1][w];
    }
  }
  __syncthreads();
  if (lane == 0) red[0][warp] = acc_h;
  __syncthreads();
  if (threadIdx.x == 0) {
    float ch = 0.f;
#pragma unroll
    for (int w = 0; w < THREADS / 32; ++w) ch += red[0][w];
    cpg *= invB;
    cvl *= invB;
    ch *= invB;
    atomicAdd(&out[0], cpg + vf_coef * cvl - ent_coef * ch);
    atomicAdd(&out[1], cpg);
    atomicAdd(&out[2], cvl);
    atomicAdd(&out[3], ch);
  }
}


// ---------------------------------------------------------------- sampling
// One rollout step's action sampling: a ~ Categorical(softmax(logits)) by
// Gumbel-max with counter-based uniforms (splitmix64 / lowbias32 of (seed,
// *counter, t, env, action) -- no generator state, so the step replays as a
// CUDA graph), log p(a), the value, and the previous step's reward / done
// into the rollout buffers.  One warp per env.
__device__ __forceinline__ uint64_t smix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
  x ^= x >> 16; x *= 0x7FEB352Du; x ^= x >> 15; x *= 0x846CA68Bu; x ^= x >> 16;
  return x;
}

template <int NA, typename TI>
__global__ void __launch_bounds__(THREADS) k_sample(const TI* __restrict__ logits, const TI* __restrict__ values,
                                                    int n, int64_t ldl, int64_t ldv, uint64_t seed,
                                                    const unsigned long long* __restrict__ counter, uint32_t t,
                                                    int64_t* __restrict__ act_a, int64_t* __restrict__ act_b,
                                                    float* __restrict__ logp_out, float* __restrict__ v_out,
                                                    const float* __restrict__ prev_rew, const uint8_t* __restrict__ prev_done,
                                                    float* __restrict__ rew_out, float* __restrict__ done_out) {
  constexpr int PER = (NA + 31) / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int env = blockIdx.x * (THREADS / 32) + warp;
  if (env >= n) return;
  const uint64_t key = smix64(seed ^ smix64((uint64_t)*counter * 0x100000001B3ull + t));
  const uint32_t k32 = (uint32_t)key ^ (uint32_t)(key >> 32);
  float zl[PER];
  float m = -INFINITY, best = -INFINITY;
  int arg = 0x7fffffff;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int j = lane + 32 * k;
    zl[k] = j < NA ? (float)logits[(size_t)env * ldl + j] : -INFINITY;
    m = fmaxf(m, zl[k]);
    if (j < NA) {
      const uint32_t h = lowbias32(k32 ^ ((uint32_t)(env * NA + j) * 0x9E3779B9u + 0x9E3779B9u));
      const float u = fmaxf(((float)(h >> 8) + 0.5f) * 5.9604644775390625e-08f, 1e-20f);   // (0, 1)
      const float g = zl[k] - logf(-logf(u));
      if (g > best) { best = g; arg = j; }
    }
  }
  // argmax over lanes (first index on ties)
  for (int o = 16; o; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
    if (ob > best || (ob == best && oa < arg)) { best = ob; arg = oa; }
  }
  m = warp_max(m);
  float se = 0.f;
#pragma unroll
  for (int k = 0; k < PER; ++k) se += lane + 32 * k < NA ? expf(zl[k] - m) : 0.f;
  se = warp_sum(se);
  float za = 0.f;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const float zk = __shfl_sync(0xffffffffu, zl[k], arg & 31);
    if (k == arg / 32) za = zk;
  }
  if (lane == 0) {
    act_a[env] = arg;
    if (act_b) act_b[env] = arg;
    logp_out[env] = za - (m + logf(se));
    v_out[env] = (float)values[(size_t)env * ldv];
    if (rew_out) {
      rew_out[env] = prev_rew[env];
      done_out[env] = (float)prev_done[env];
    }
  }
}


// ------------------------------------------------------ hand-written backward
// One layer's bias gradient, and for a tanh layer the activation's backward,
// in one pass over the layer's [rows, cols] output gradient:
//   dy[i, j] = j < split ? dy_a[i * ld_a + j] : dy_b[i * ld_b + j - split]
//   dz[i, j] = bf16(dy[i, j] * (1 - y[i, j]^2))        (y: the tanh output; y == null: dz = dy)
//   db[j]    = sum_i dz[i, j]                            (fp32, a fixed summation order)
// The two dy halves are the actor's and the critic's gradients of the shared
// first layer.  CTA (x, r) sums rows [r * rows / RCH, (r + 1) * rows / RCH)
// of a 64-column tile into work[r * cols + j]; the tile's last CTA (counter)
// adds the RCH partials in order, so the result is deterministic.
constexpr int BG_COLS = 64, BG_THREADS = 256, BG_TR = BG_THREADS / 8;   // 8 columns per thread, 32 row lanes

template <bool VEC>
__global__ void __launch_bounds__(BG_THREADS) k_bias_grad(const __nv_bfloat16* __restrict__ y, int64_t ldy,
                                                          const __nv_bfloat16* __restrict__ dya, int64_t lda,
                                                          const __nv_bfloat16* __restrict__ dyb, int64_t ldb,
                                                          int split, int rows, int cols,
                                                          __nv_bfloat16* __restrict__ dz, float* __restrict__ db,
                                                          float* __restrict__ work, unsigned* __restrict__ counters,
                                                          int64_t bsy, int64_t bsa, int64_t bsz) {
  __shared__ float red[BG_TR][BG_COLS + 1];
  __shared__ bool last;
  {   // batch entry blockIdx.z: its own operands, bias gradient, partials and counters
    const int z = blockIdx.z;
    if (y) y += z * bsy;
    dya += z * bsa;
    if (dz) dz += z * bsz;
    db += (size_t)z * cols;
    work += (size_t)z * gridDim.y * cols;
    counters += (size_t)z * gridDim.x;
  }
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  const int c0 = blockIdx.x * BG_COLS + tx * 8;
  const int RCH = gridDim.y;
  const int r0 = (int)((int64_t)rows * blockIdx.y / RCH), r1 = (int)((int64_t)rows * (blockIdx.y + 1) / RCH);
  float acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.f;
  for (int i = r0 + ty; i < r1; i += BG_TR) {
    if (VEC) {   // cols, split, leading dimensions and pointers 16-byte aligned
      if (c0 >= cols) break;
      const __nv_bfloat16* src = c0 < split ? dya + (size_t)i * lda + c0 : dyb + (size_t)i * ldb + (c0 - split);
      uint4 g = *reinterpret_cast<const uint4*>(src);
      __nv_bfloat16* gv = reinterpret_cast<__nv_bfloat16*>(&g);
      if (y) {
        uint4 yy = *reinterpret_cast<const uint4*>(y + (size_t)i * ldy + c0);
        const __nv_bfloat16* yv = reinterpret_cast<const __nv_bfloat16*>(&yy);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float t = __bfloat162float(yv[q]);
          gv[q] = __float2bfloat16(__bfloat162float(gv[q]) * (1.f - t * t));
        }
        *reinterpret_cast<uint4*>(dz + (size_t)i * cols + c0) = g;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] += __bfloat162float(gv[q]);
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int c = c0 + q;
        if (c >= cols) break;
        float g = __bfloat162float(c < split ? dya[(size_t)i * lda + c] : dyb[(size_t)i * ldb + (c - split)]);
        if (y) {
          const float t = __bfloat162float(y[(size_t)i * ldy + c]);
          const __nv_bfloat16 gz = __float2bfloat16(g * (1.f - t * t));
          dz[(size_t)i * cols + c] = gz;
          g = __bfloat162float(gz);
        }
        acc[q] += g;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) red[ty][tx * 8 + q] = acc[q];
  __syncthreads();
  if (threadIdx.x < BG_COLS) {
    float s = 0.f;
    for (int r = 0; r < BG_TR; ++r) s += red[r][threadIdx.x];
    const int c = blockIdx.x * BG_COLS + threadIdx.x;
    if (c < cols) work[(size_t)blockIdx.y * cols + c] = s;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&counters[blockIdx.x], 1u) == (unsigned)RCH - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < BG_COLS) {
    const int c = blockIdx.x * BG_COLS + threadIdx.x;
    if (c < cols) {
      float s = 0.f;
      for (int r = 0; r < RCH; ++r) s += __ldcg(work + (size_t)r * cols + c);
      db[c] = s;
    }
  }
  if (threadIdx.x == 0) counters[blockIdx.x] = 0;   // ready for the next launch (graph replays)
}

// z[b, i, j] = bf16(tanh(z[b, i, j] + bias[b, j])) in place over a contiguous
// [batch, rows, cols] bf16 tensor (the actor's and critic's hidden layers as
// one batched GEMM without a bias epilogue, then this); 8 elements per thread.
__global__ void __launch_bounds__(256) k_bias_tanh(__nv_bfloat16* __restrict__ z,
                                                   const __nv_bfloat16* __restrict__ bias, int64_t n8, int cols,
                                                   int64_t per_batch) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n8; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = k * 8;
    const int b = (int)(e / per_batch), j = (int)(e % cols);
    uint4 v = reinterpret_cast<uint4*>(z)[k];
    const uint4 bb = *reinterpret_cast<const uint4*>(bias + (size_t)b * cols + j);
    __nv_bfloat16* vv = reinterpret_cast<__nv_bfloat16*>(&v);
    const __nv_bfloat16* bv = reinterpret_cast<const __nv_bfloat16*>(&bb);
#pragma unroll
    for (int q = 0; q < 8; ++q) vv[q] = __float2bfloat16(tanhf(__bfloat162float(vv[q]) + __bfloat162float(bv[q])));
    reinterpret_cast<uint4*>(z)[k] = v;
  }
}

// dst[i * ld_dst + j] = bf16(src[i * w + j]) for j < w (float4 loads, 8-byte
// stores; the rollout buffer's copy of a step's observation, which the
// writer has just left in L2)
__global__ void __launch_bounds__(256) k_f32_to_bf16_rows(const float* __restrict__ src, int64_t rows, int w4,
                                                          __nv_bfloat16* __restrict__ dst, int64_t ld_dst) {
  const int64_t total = rows * w4;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / w4;
    const int j4 = (int)(k - i * w4);
    const float4 v = __ldcs(reinterpret_cast<const float4*>(src) + k);
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 packed;
    packed.x = *reinterpret_cast<uint32_t*>(&lo);
    packed.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(dst + i * ld_dst + (int64_t)j4 * 4) = packed;
  }
}

__global__ void __launch_bounds__(256) k_f32_to_bf16_any(const float* __restrict__ src, int64_t rows, int w,
                                                         __nv_bfloat16* __restrict__ dst, int64_t ld_dst) {
  const int64_t total = rows * w;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / w;
    dst[i * ld_dst + (k - i * w)] = __float2bfloat16(__ldcs(src + k));
  }
}

// ------------------------------------------------ global-norm clip + Adam
// torch.nn.utils.clip_grad_norm_ followed by torch.optim.Adam (capturable,
// no weight decay, no amsgrad) over one flat fp32 parameter buffer, in two
// launches: k_sumsq (a fixed grid of partial sums of g^2; its last CTA forms
// the clip factor, increments the step and the bias corrections into
// `coef`), then k_adam (m, v, p, and the bf16 copy of p the next forward
// reads).  The gradients themselves are not modified.
constexpr int AD_THREADS = 256, SQ_CTAS = 296;

__global__ void __launch_bounds__(AD_THREADS) k_sumsq(const float* __restrict__ g, int64_t n, float grad_scale,
                                                      float max_norm, const float* __restrict__ lr, float* step,
                                                      float beta1, float beta2, float* __restrict__ partial,
                                                      unsigned* __restrict__ counter, float* __restrict__ coef) {
  __shared__ float red[AD_THREADS / 32];
  __shared__ bool last;
  float s = 0.f;
  const int64_t n4 = n / 4;
  for (int64_t k = (int64_t)blockIdx.x * AD_THREADS + threadIdx.x; k < n4; k += (int64_t)gridDim.x * AD_THREADS) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(g) + k);
    s += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  if (blockIdx.x == 0)
    for (int64_t k = n4 * 4 + threadIdx.x; k < n; k += AD_THREADS) s += g[k] * g[k];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < AD_THREADS / 32; ++w) t += red[w];
    partial[blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  double tot = 0.0;
  for (unsigned b = 0; b < gridDim.x; ++b) tot += (double)__ldcg(partial + b);
  const float norm = grad_scale * sqrtf((float)tot);
  const float clip = fminf(max_norm / (norm + 1e-6f), 1.f);
  const float st = *step + 1.f;
  *step = st;
  const float bc1 = 1.f - powf(beta1, st), bc2 = 1.f - powf(beta2, st);
  coef[0] = grad_scale * clip;    // gradient multiplier
  coef[1] = *lr / bc1;            // step size
  coef[2] = sqrtf(bc2);
  coef[3] = norm;                 // the pre-clip global norm (stats)
  *counter = 0;
}

__global__ void __launch_bounds__(AD_THREADS) k_adam(float* __restrict__ p, const float* __restrict__ g,
                                                     float* __restrict__ m, float* __restrict__ v,
                                                     __nv_bfloat16* __restrict__ pb, int64_t n,
                                                     const float* __restrict__ coef, float beta1, float beta2,
                                                     float eps) {
  const float gs = coef[0], step_size = coef[1], bc2s = coef[2];
  auto one = [&](float& pp, float gg, float& mm, float& vv) {
    gg *= gs;
    mm = beta1 * mm + (1.f - beta1) * gg;
    vv = beta2 * vv + (1.f - beta2) * gg * gg;
    const float denom = sqrtf(vv) / bc2s + eps;
    pp -= step_size * (mm / denom);
  };
  const int64_t n4 = n / 4;
  for (int64_t k = (int64_t)blockIdx.x * AD_THREADS + threadIdx.x; k < n4; k += (int64_t)gridDim.x * AD_THREADS) {
    float4 pp = reinterpret_cast<float4*>(p)[k], mm = reinterpret_cast<float4*>(m)[k],
           vv = reinterpret_cast<float4*>(v)[k];
    const float4 gg = __ldg(reinterpret_cast<const float4*>(g) + k);
    one(pp.x, gg.x, mm.x, vv.x);
    one(pp.y, gg.y, mm.y, vv.y);
    one(pp.z, gg.z, mm.z, vv.z);
    one(pp.w, gg.w, mm.w, vv.w);
    reinterpret_cast<float4*>(p)[k] = pp;
    reinterpret_cast<float4*>(m)[k] = mm;
    reinterpret_cast<float4*>(v)[k] = vv;
    __nv_bfloat162 lo = __floats2bfloat162_rn(pp.x, pp.y), hi = __floats2bfloat162_rn(pp.z, pp.w);
    uint2 packed;
    packed.x = *reinterpret_cast<uint32_t*>(&lo);
    packed.y = *reinterpret_cast<uint32_t*>(&hi);
    reinterpret_cast<uint2*>(pb)[k] = packed;
  }
  if (blockIdx.x == 0)
    for (int64_t k = n4 * 4 + threadIdx.x; k < n; k += AD_THREADS) {
      one(p[k], g[k], m[k], v[k]);
      pb[k] = __float2bfloat16(p[k]);
    }
}

}  // namespace

extern "C" int grp_ppo_loss(const float* logits, const float* v, const int64_t* actions, const float* logp_old,
                            const float* adv, const float* v_old, const float* ret, int32_t batch,
                            int32_t n_actions, float clip_eps, float vf_coef, float ent_coef, float* dlogits,
                            float* dv, float* out, void* stream) {
  if (batch <= 0) return -1;
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // >= 8 rows per warp: every CTA first re-reads the whole advantage column
  // (mean / std), so fewer, fuller CTAs (8,192 rows: 128 CTAs)
  const int rows_per_cta = 8 * (THREADS / 32);
  const int grid = (int)std::min<int64_t>((batch + rows_per_cta - 1) / rows_per_cta, (int64_t)sms);
#define GRP_CASE(N)                                                                                          \
  case N:                                                                                                    \
    k_ppo_loss<N, float, float><<<grid, THREADS, 0, st>>>(logits, N, v, 1, actions, logp_old, adv, v_old, ret, \
                                                         batch, clip_eps, vf_coef, ent_coef, dlogits, N, N, dv, 1,  \
                                                         out, nullptr);                                           \
    break;
  switch (n_actions) {
    GRP_CASE(17)
    GRP_CASE(43)
    default:
      return -1;
  }
#undef GRP_CASE
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int grp_sample_actions(const void* logits, const void* values, int32_t bf16, int32_t n, int32_t n_actions,
                                  int64_t ld_logits, int64_t ld_values, uint64_t seed,
                                  const unsigned long long* counter, uint32_t t, int64_t* actions_a,
                                  int64_t* actions_b, float* logp, float* value, const float* prev_reward,
                                  const uint8_t* prev_done, float* reward_out, float* done_out, void* stream) {
  if (n <= 0) return -1;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = (n + THREADS / 32 - 1) / (THREADS / 32);
#define GRS_CASE(N)                                                                                             \
  case N:                                                                                                       \
    if (bf16)                                                                                                   \
      k_sample<N, __nv_bfloat16><<<grid, THREADS, 0, st>>>(                                                     \
          (const __nv_bfloat16*)logits, (const __nv_bfloat16*)values, n, ld_logits, ld_values, seed, counter, t, \
          actions_a, actions_b, logp, value, prev_reward, prev_done, reward_out, done_out);                     \
    else                                                                                                        \
      k_sample<N, float><<<grid, THREADS, 0, st>>>((const float*)logits, (const float*)values, n, ld_logits,   \
                                                   ld_values, seed, counter, t, actions_a, actions_b, logp,    \
                                                   value, prev_reward, prev_done, reward_out, done_out);       \
    break;
  switch (n_actions) {
    GRS_CASE(17)
    GRS_CASE(43)
    default:
      return -1;
  }
#undef GRS_CASE
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int grp_ppo_loss_bf16(const void* logits, int64_t ld_logits, const void* values, int64_t ld_values,
                                 const int64_t* actions, const float* logp_old, const float* adv,
                                 const float* v_old, const float* ret, int32_t batch, int32_t n_actions,
                                 float clip_eps, float vf_coef, float ent_coef, void* dlogits, int64_t ld_dlogits,
                                 int32_t n_pad, void* dvalues, int64_t ld_dvalues, float* out, const int64_t* index,
                                 void* stream) {
  if (batch <= 0 || n_pad < n_actions || ld_dlogits < n_pad) return -1;
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // >= 8 rows per warp: every CTA first re-reads the whole advantage column
  // (mean / std), so fewer, fuller CTAs (8,192 rows: 128 CTAs)
  const int rows_per_cta = 8 * (THREADS / 32);
  const int grid = (int)std::min<int64_t>((batch + rows_per_cta - 1) / rows_per_cta, (int64_t)sms);
  using B16 = __nv_bfloat16;
#define GRB_CASE(N)                                                                                       \
  case N:                                                                                                 \
    k_ppo_loss<N, B16, B16><<<grid, THREADS, 0, st>>>(                                                    \
        (const B16*)logits, ld_logits, (const B16*)values, ld_values, actions, logp_old, adv, v_old, ret, \
        batch, clip_eps, vf_coef, ent_coef, (B16*)dlogits, ld_dlogits, n_pad, (B16*)dvalues, ld_dvalues,  \
        out, index);                                                                                      \
    break;
  switch (n_actions) {
    GRB_CASE(17)
    GRB_CASE(43)
    default:
      return -1;
  }
#undef GRB_CASE
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int grp_bias_grad(const void* y, int64_t ld_y, const void* dy_a, int64_t ld_a, const void* dy_b,
                             int64_t ld_b, int32_t split, int32_t rows, int32_t cols, void* dz, float* db,
                             float* work, int32_t row_chunks, unsigned* counters, int32_t batch, int64_t bs_y,
                             int64_t bs_a, int64_t bs_dz, void* stream) {
  if (rows <= 0 || cols <= 0 || row_chunks <= 0 || split < 0 || split > cols || (y && !dz)) return -1;
  if (split < cols && !dy_b) return -1;
  if (split > 0 && !dy_a) return -1;
  if (batch < 1 || (batch > 1 && split != cols)) return -1;   // batched: one source per entry
  auto al16 = [](const void* q) { return ((uintptr_t)q & 15) == 0; };
  const bool vec = cols % 8 == 0 && split % 8 == 0 && ld_a % 8 == 0 && ld_b % 8 == 0 && ld_y % 8 == 0 &&
                   bs_y % 8 == 0 && bs_a % 8 == 0 && bs_dz % 8 == 0 &&
                   (!dy_a || al16(dy_a)) && (!dy_b || al16(dy_b)) && (!y || al16(y)) && (!dz || al16(dz));
  const dim3 grid((cols + BG_COLS - 1) / BG_COLS, row_chunks, batch);
  using B16 = __nv_bfloat16;
  cudaStream_t st = (cudaStream_t)stream;
  if (vec)
    k_bias_grad<true><<<grid, BG_THREADS, 0, st>>>((const B16*)y, ld_y, (const B16*)dy_a, ld_a, (const B16*)dy_b,
                                                   ld_b, split, rows, cols, (B16*)dz, db, work, counters, bs_y, bs_a,
                                                   bs_dz);
  else
    k_bias_grad<false><<<grid, BG_THREADS, 0, st>>>((const B16*)y, ld_y, (const B16*)dy_a, ld_a, (const B16*)dy_b,
                                                    ld_b, split, rows, cols, (B16*)dz, db, work, counters, bs_y, bs_a,
                                                    bs_dz);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int grp_clip_adam(float* params, const float* grads, float* exp_avg, float* exp_avg_sq,
                             void* params_bf16, int64_t n, const float* lr, float* step, float beta1, float beta2,
                             float eps, float grad_scale, float max_norm, float* work, unsigned* counter,
                             void* stream) {
  if (n <= 0) return -1;
  if (((uintptr_t)params | (uintptr_t)grads | (uintptr_t)exp_avg | (uintptr_t)exp_avg_sq) & 15) return -1;
  if ((uintptr_t)params_bf16 & 7) return -1;
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k_sumsq<<<SQ_CTAS, AD_THREADS, 0, st>>>(grads, n, grad_scale, max_norm, lr, step, beta1, beta2, work + 4, counter,
                                          work);
  k_adam<<<sms * 4, AD_THREADS, 0, st>>>(params, grads, exp_avg, exp_avg_sq, (__nv_bfloat16*)params_bf16, n, work,
                                         beta1, beta2, eps);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int grp_bias_tanh(void* z, const void* bias, int32_t batch, int32_t rows, int32_t cols, void* stream) {
  if (batch < 1 || rows <= 0 || cols <= 0 || cols % 8 || ((uintptr_t)z & 15) || ((uintptr_t)bias & 15)) return -1;
  const int64_t n8 = (int64_t)batch * rows * cols / 8;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>((n8 + 255) / 256, (int64_t)sms * 8);
  k_bias_tanh<<<grid, 256, 0, (cudaStream_t)stream>>>((__nv_bfloat16*)z, (const __nv_bfloat16*)bias, n8, cols,
                                                      (int64_t)rows * cols);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int grp_rows_to_bf16(const float* src, int64_t rows, int32_t width, void* dst, int64_t ld_dst,
                                void* stream) {
  if (rows <= 0 || width <= 0 || ld_dst < width) return -1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaStream_t st = (cudaStream_t)stream;
  if (width % 4 == 0 && ld_dst % 4 == 0 && !((uintptr_t)src & 15) && !((uintptr_t)dst & 7)) {
    const int64_t total = rows * (width / 4);
    const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sms * 8);
    k_f32_to_bf16_rows<<<grid, 256, 0, st>>>(src, rows, width / 4, (__nv_bfloat16*)dst, ld_dst);
  } else {   // any width (Craftax-Classic: 1,345 floats per row)
    const int64_t total = rows * width;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sms * 8);
    k_f32_to_bf16_any<<<grid, 256, 0, st>>>(src, rows, width, (__nv_bfloat16*)dst, ld_dst);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
