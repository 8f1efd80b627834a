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

template <int NA>
__global__ void __launch_bounds__(THREADS) k_ppo_loss(const float* __restrict__ logits, const float* __restrict__ v,
                                                      const int64_t* __restrict__ act,
                                                      const float* __restrict__ logp_old,
                                                      const float* __restrict__ adv,
                                                      const float* __restrict__ v_old,
                                                      const float* __restrict__ ret, int B, float clip_eps,
                                                      float vf_coef, float ent_coef, float* __restrict__ dlogits,
                                                      float* __restrict__ dv, float* __restrict__ out) {
  constexpr int PER = (NA + 31) / 32;
  __shared__ float red[2][THREADS / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // advantage mean and unbiased std over the minibatch
  float s = 0.f, s2 = 0.f;
  for (int i = threadIdx.x; i < B; i += THREADS) {
    const float a = adv[i];
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
    const float* z = logits + (size_t)row * NA;
    float zl[PER];
    float m = -INFINITY;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int j = lane + 32 * k;
      zl[k] = j < NA ? z[j] : -INFINITY;
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
    const int a = (int)act[row];
    float zsel = 0.f;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const float zk = __shfl_sync(0xffffffffu, zl[k], a & 31);
      if (k == a / 32) zsel = zk;
    }
    const float logp = zsel - lse;
    const float r = expf(logp - logp_old[row]);
    const float an = (adv[row] - mean) * inv_std;
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
    const float vv = v[row], vo = v_old[row], R = ret[row];
    const float dvu = vv - vo;
    const float vc = vo + fminf(fmaxf(dvu, -clip_eps), clip_eps);
    const float e1 = (vv - R) * (vv - R), e2 = (vc - R) * (vc - R);
    const float vl = 0.5f * fmaxf(e1, e2);
    float g_v = e1 >= e2 ? (vv - R) : ((dvu > -clip_eps && dvu < clip_eps) ? (vc - R) : 0.f);
    g_v *= vf_coef * invB;
    // d loss / d z_j = g_logp (1[j==a] - p_j) + c_e/B p_j (log p_j + H)
    float* dz = dlogits + (size_t)row * NA;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int j = lane + 32 * k;
      if (j < NA) {
        const float lp = zl[k] - lse, p = expf(lp);
        dz[j] = g_logp * ((j == a ? 1.f : 0.f) - p) + ent_coef * invB * p * (lp + h);
      }
    }
    if (lane == 0) {
      dv[row] = g_v;
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
  const int rows_per_cta = THREADS / 32;
  const int grid = (int)std::min<int64_t>((batch + rows_per_cta - 1) / rows_per_cta, (int64_t)sms * 4);
#define GRP_CASE(N)                                                                                          \
  case N:                                                                                                    \
    k_ppo_loss<N><<<grid, THREADS, 0, st>>>(logits, v, actions, logp_old, adv, v_old, ret, batch, clip_eps, \
                                           vf_coef, ent_coef, dlogits, dv, out);                            \
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
