// gr_reset.cu -- optimistic auto-reset: done-rank scan, pool bookkeeping and
// world install.
//
// batch.batch_step (batch.py:216-231): the pool serving step s is
// WorldPool(pool_key, s + 1, M); done envs, in ascending global env order,
// take slot rank % M; install_worlds (state.py:198-249) resets each one.
// Worlds are generated only for the slots this shard consumes
// (gr_world.cu); pool entry p holds slot (offset + p) % M, so the env of
// local done rank r installs entry r % M.
#include <cstdint>
#include <algorithm>
#include "gr_device.cuh"
#include "gr_state.cuh"
#include "gr_kernels.cuh"
#include "gr_desc.cuh"
#include "gr_tail.cuh"
#include "gr_levels.cuh"

namespace gr {

// combine the all-gathered exchange records of every rank
__global__ void k_finish_info(const int32_t* ex_all, int rank, int world, int64_t M, uint64_t pool_key,
                              unsigned long long* dstep, StepInfo* info, uint32_t* flags_out) {
  combine_info(ex_all, rank, world, M, pool_key, dstep, info, flags_out);
}

// the block / item maps of one env, 16-byte vectors [part, nparts) of them:
// all threads of the CTA
template <bool EXT>
__device__ void install_maps(const DS& S, int64_t i, const uint8_t* src_blk, const uint8_t* src_itm, int part,
                             int nparts) {
  constexpr int F = EXT ? 9 : 1, H = EXT ? 48 : 64, W = H, HW = H * W;
  {
    uint4* db = reinterpret_cast<uint4*>((uint8_t*)S.f[GR_F_BLOCKS] + (size_t)i * F * HW);
    uint4* di = reinterpret_cast<uint4*>((uint8_t*)S.f[GR_F_ITEMS] + (size_t)i * F * HW);
    const uint4* sb = reinterpret_cast<const uint4*>(src_blk);
    const uint4* si = reinterpret_cast<const uint4*>(src_itm);
    // 2 x U vector loads in flight per thread before their stores: the copy
    // is a chain of round trips otherwise (small batches wait on it)
    constexpr int NVA = F * HW / 16, U = 4;
    const int v0 = (int)((int64_t)NVA * part / nparts), NV = (int)((int64_t)NVA * (part + 1) / nparts);
    for (int q0 = v0 + threadIdx.x; q0 < NV; q0 += U * blockDim.x) {
      uint4 vb[U], vi[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + u * blockDim.x;
        if (q < NV) {
          vb[u] = sb[q];
          vi[u] = si[q];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + u * blockDim.x;
        if (q < NV) {
          db[q] = vb[u];
          di[q] = vi[u];
        }
      }
    }
  }
}

// install_worlds for one env (state.py:198-249) without the maps; all threads of the CTA
template <bool EXT>
__device__ void install_fields(const DS& S, int64_t i, const WMeta& m) {
  constexpr int F = EXT ? 9 : 1, H = EXT ? 48 : 64, W = H;
  // per-floor lanes and chests: spread over threads
#define Z(fid, T_, c) GR_AT(S, fid, T_, c, i) = (T_)0
  for (int c = threadIdx.x; c < F * 6; c += blockDim.x) {
    const int f = c / 6, j = c % 6;
    const bool has = EXT && j < m.nch[f];
    GR_AT(S, GR_F_CHEST_POS, int16_t, 2 * c, i) = has ? m.chest[f][j][0] : (int16_t)-1;
    GR_AT(S, GR_F_CHEST_POS, int16_t, 2 * c + 1, i) = has ? m.chest[f][j][1] : (int16_t)-1;
    GR_AT(S, GR_F_CHEST_LOOT, uint8_t, c, i) = has ? (uint8_t)m.chest[f][j][2] : (uint8_t)0;
    GR_AT(S, GR_F_CHEST_QTY, uint8_t, c, i) = has ? (uint8_t)m.chest[f][j][3] : (uint8_t)0;
    GR_AT(S, GR_F_CHEST_AUX, uint8_t, c, i) = has ? (uint8_t)(hash2(m.key, 800 + (uint64_t)c) % 6) : (uint8_t)0;
  }
  for (int c = threadIdx.x; c < F * 3; c += blockDim.x) {
    Z(GR_F_MEL_POS, int16_t, 2 * c); Z(GR_F_MEL_POS, int16_t, 2 * c + 1);
    Z(GR_F_MEL_HP, float, c); Z(GR_F_MEL_CD, uint8_t, c); Z(GR_F_MEL_ALIVE, uint8_t, c); Z(GR_F_MEL_TYPE, uint8_t, c);
    Z(GR_F_PAS_POS, int16_t, 2 * c); Z(GR_F_PAS_POS, int16_t, 2 * c + 1);
    Z(GR_F_PAS_HP, float, c); Z(GR_F_PAS_ALIVE, uint8_t, c); Z(GR_F_PAS_TYPE, uint8_t, c);
  }
  for (int c = threadIdx.x; c < F * 2; c += blockDim.x) {
    Z(GR_F_RAN_POS, int16_t, 2 * c); Z(GR_F_RAN_POS, int16_t, 2 * c + 1);
    Z(GR_F_RAN_HP, float, c); Z(GR_F_RAN_CD, uint8_t, c); Z(GR_F_RAN_ALIVE, uint8_t, c); Z(GR_F_RAN_TYPE, uint8_t, c);
  }
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    GR_AT(S, GR_F_LADDER_DOWN, int16_t, 2 * f, i) = m.ld[f][0];
    GR_AT(S, GR_F_LADDER_DOWN, int16_t, 2 * f + 1, i) = m.ld[f][1];
    GR_AT(S, GR_F_LADDER_UP, int16_t, 2 * f, i) = m.lu[f][0];
    GR_AT(S, GR_F_LADDER_UP, int16_t, 2 * f + 1, i) = m.lu[f][1];
    GR_AT(S, GR_F_FLOORS_VISITED, uint8_t, f, i) = f == 0;
    GR_AT(S, GR_F_FLOOR_CLEARED, uint8_t, f, i) = 0;
  }
  for (int l = threadIdx.x; l < 10; l += blockDim.x) {
    Z(GR_F_PLANT_POS, int16_t, 2 * l); Z(GR_F_PLANT_POS, int16_t, 2 * l + 1);
    Z(GR_F_PLANT_AGE, uint16_t, l); Z(GR_F_PLANT_ALIVE, uint8_t, l);
  }
  for (int l = threadIdx.x; l < 3; l += blockDim.x) {
    Z(GR_F_PPROJ_POS, int16_t, 2 * l); Z(GR_F_PPROJ_POS, int16_t, 2 * l + 1);
    Z(GR_F_PPROJ_DIR, uint8_t, l); Z(GR_F_PPROJ_TYPE, uint8_t, l); Z(GR_F_PPROJ_TTL, uint8_t, l);
    Z(GR_F_PPROJ_ALIVE, uint8_t, l);
    Z(GR_F_EPROJ_POS, int16_t, 2 * l); Z(GR_F_EPROJ_POS, int16_t, 2 * l + 1);
    Z(GR_F_EPROJ_DIR, uint8_t, l); Z(GR_F_EPROJ_TYPE, uint8_t, l); Z(GR_F_EPROJ_TTL, uint8_t, l);
    Z(GR_F_EPROJ_ALIVE, uint8_t, l);
    for (int k = 0; k < 3; ++k) { Z(GR_F_PPROJ_DMG, float, 3 * l + k); Z(GR_F_EPROJ_DMG, float, 3 * l + k); }
  }
  for (int k = threadIdx.x; k < 6; k += blockDim.x) {
    GR_AT(S, GR_F_POTION_MAP, uint8_t, k, i) = m.potion[k];
    Z(GR_F_INV_POTION, uint8_t, k);
    Z(GR_F_CLOCKS, uint16_t, k);
  }
  if (threadIdx.x == 0) {
    GR_AT(S, GR_F_SPAWN0, int16_t, 0, i) = m.spawn[0];
    GR_AT(S, GR_F_SPAWN0, int16_t, 1, i) = m.spawn[1];
    GR_AT(S, GR_F_PARAMS_SEED, uint64_t, 0, i) = m.seed;
    GR_AT(S, GR_F_PROW, int16_t, 0, i) = m.spawn[0];
    GR_AT(S, GR_F_PCOL, int16_t, 0, i) = m.spawn[1];
    if (EXT) {
      GR_AT(S, GR_F_NECRO_POS, int16_t, 0, i) = (int16_t)(H / 2 - 6);
      GR_AT(S, GR_F_NECRO_POS, int16_t, 1, i) = (int16_t)(W / 2);
    }
    GR_AT(S, GR_F_FACING, uint8_t, 0, i) = 3;
    GR_AT(S, GR_F_DEX, uint8_t, 0, i) = 1;
    GR_AT(S, GR_F_STR, uint8_t, 0, i) = 1;
    GR_AT(S, GR_F_INTEL, uint8_t, 0, i) = 1;
    Z(GR_F_XP, uint8_t, 0); Z(GR_F_SWORD_TIER, uint8_t, 0); Z(GR_F_PICK_TIER, uint8_t, 0);
    Z(GR_F_HAS_BOW, uint8_t, 0); Z(GR_F_SWORD_ENCH, uint8_t, 0); Z(GR_F_BOW_ENCH, uint8_t, 0);
    Z(GR_F_LEARNED_FIRE, uint8_t, 0); Z(GR_F_LEARNED_ICE, uint8_t, 0);
    Z(GR_F_SLEEPING, uint8_t, 0); Z(GR_F_RESTING, uint8_t, 0);
    for (int fid = GR_F_INV_WOOD; fid <= GR_F_INV_BOOK; ++fid) GR_AT(S, fid, uint8_t, 0, i) = 0;
    for (int k = 0; k < 4; ++k) { Z(GR_F_ARMOUR, uint8_t, k); Z(GR_F_ARMOUR_ENCH, uint8_t, k); }
    for (int k = 0; k < 3; ++k) Z(GR_F_ACH, uint32_t, k);
    Z(GR_F_TIME, uint32_t, 0);
    Z(GR_F_BOSS_WAVE, uint8_t, 0); Z(GR_F_BOSS_VULN, uint8_t, 0); Z(GR_F_BOSS_TIMER, uint8_t, 0);
    Z(GR_F_DONE, uint8_t, 0);
    Z(GR_F_PFLOOR, uint8_t, 0);
    GR_AT(S, GR_F_HEALTH, float, 0, i) = 10.0f;
    GR_AT(S, GR_F_FOOD, float, 0, i) = 13.0f;
    GR_AT(S, GR_F_DRINK, float, 0, i) = 13.0f;
    GR_AT(S, GR_F_ENERGY, float, 0, i) = 13.0f;
    GR_AT(S, GR_F_MANA, float, 0, i) = 17.0f;
    GR_AT(S, GR_F_RNG_KEY, uint64_t, 0, i) = m.key;
    GR_AT(S, GR_F_BOSS_HP, float, 0, i) = EXT ? 60.0f : 0.0f;
    S.cd_pending[i] = 0;
    S.torch_bits[i] = 0;
    S.ep_return[i] = 0.0;
    S.ep_length[i] = 0;
  }
  // observation descriptor of the fresh episode (gr_desc.cuh)
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    constexpr int NINV = EXT ? 50 : 18;
    uint32_t* d = S.desc + (size_t)i * DESC_WORDS;
    __shared__ float inv_s[50];
    if (lane == 0) {
      InvSrc s{};
      s.dex = s.str_ = s.intel = 1;
      s.facing = 3;
      s.health = 10.0f; s.food = 13.0f; s.drink = 13.0f; s.energy = 13.0f; s.mana = 17.0f;
      inv_section<EXT>(s, inv_s, S.lut);
    }
    __syncwarp();
    for (int k = lane; k < DESC_WORDS; k += 32) {
      uint32_t w = 0;
      if (k < NINV) w = __float_as_uint(inv_s[k]);
      else if (k == D_BASE) w = __float_as_uint(lut_daylight(S.lut, 0));
      else if (k == D_POS) w = (uint32_t)(uint16_t)m.spawn[0] | ((uint32_t)(uint16_t)m.spawn[1] << 16);
      else if (k >= D_CRE && k < D_CRE + 7) w = 0xFFFFFFFFu;
      d[k] = w;
    }
  }
#undef Z
}

// install_worlds for one env (state.py:198-249); all threads of the CTA
template <bool EXT>
__device__ void install_one(const DS& S, int64_t i, const WMeta& m, const uint8_t* src_blk, const uint8_t* src_itm) {
  if (src_blk) install_maps<EXT>(S, i, src_blk, src_itm, 0, 1);
  install_fields<EXT>(S, i, m);
}

// level buffer -> chosen envs (UED): level_idx[k] installed into env_idx[k]
// with install key keys[k] (state.install_world, state.py:169-171)
template <bool EXT>
__global__ void __launch_bounds__(128) k_install_levels(DS S, WBuf w, const int64_t* env_idx, const int64_t* level_idx,
                                                        const uint64_t* keys, int64_t count) {
  constexpr int F = EXT ? 9 : 1, HW = EXT ? 48 * 48 : 64 * 64;
  __shared__ WMeta m;
  for (int64_t k = blockIdx.x; k < count; k += gridDim.x) {
    const int64_t l = level_idx[k];
    if (threadIdx.x == 0) {
      m = w.meta[l];
      m.key = keys[k];
    }
    __syncthreads();
    install_one<EXT>(S, env_idx[k], m, w.blocks + (size_t)l * F * HW, w.items + (size_t)l * F * HW);
    __syncthreads();
  }
}

void launch_install_levels(bool ext, const DS& S, const WBuf& w, const int64_t* env_idx, const int64_t* level_idx,
                           const uint64_t* keys, int64_t count, cudaStream_t st) {
  if (count <= 0) return;
  const int grid = (int)std::min<int64_t>(count, 148 * 8);
  if (ext) k_install_levels<true><<<grid, 128, 0, st>>>(S, w, env_idx, level_idx, keys, count);
  else k_install_levels<false><<<grid, 128, 0, st>>>(S, w, env_idx, level_idx, keys, count);
}

// initial reset: world w was generated straight into env w's maps
template <bool EXT>
__global__ void __launch_bounds__(128) k_install_initial(DS S, WBuf wb, int64_t n) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) install_one<EXT>(S, i, wb.meta[i], nullptr, nullptr);
}

// done envs in ascending order: local rank = block offset (k_step's tail scan) + rank
// inside the 128-env block (ballots)
__global__ void __launch_bounds__(128) k_compact(const uint8_t* done, int64_t n, const int32_t* block_off,
                                                 int32_t* list) {
  __shared__ int wcnt[4];
  const int64_t i = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const bool d = i < n && done[i];
  const unsigned bal = __ballot_sync(0xffffffffu, d);
  if ((threadIdx.x & 31) == 0) wcnt[threadIdx.x >> 5] = __popc(bal);
  __syncthreads();
  int pre = 0;
  for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) pre += wcnt[w];
  if (d) list[block_off[blockIdx.x] + pre + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u))] = (int32_t)i;
}

// auto-reset: a.parts CTAs per done env (persistent grid over the done list
// x parts): part 0 the EpisodeStats and the state fields, every part a slice
// of the maps.  The copy of one env's 41 KB of extended maps is a chain of
// round trips on one CTA, on the critical path of small batches (1,024
// envs: 0.0549 -> 0.0538 ms per step with 4 parts); large batches have
// enough envs per step to fill the machine and keep one part (65,536 envs:
// 4 parts measured 0.5 % slower beside the observation writer)
template <bool EXT>
__global__ void __launch_bounds__(128) k_install_pool(DS S, InstallArgs a) {
  constexpr int F = EXT ? 9 : 1, HW = EXT ? 48 * 48 : 64 * 64, A = EXT ? 67 : 22;
  const int NP = a.parts;
  const int k = a.info->k_local;
  if (a.dstep_advance && blockIdx.x == 0 && threadIdx.x == 0) {
    *a.dstep_advance += 1;
    // next step's speculation: this step's pool size + 25 % + 8 (the done
    // count moves slowly; a shortfall is generated after the step as before)
    const int np = a.info->n_pool;
    *a.spec_k = (int32_t)min((int64_t)(np + (np >> 2) + 8), a.spec_cap);
  }
  for (int w = blockIdx.x; w < k * NP; w += gridDim.x) {
    const int r = w / NP, part = w - r * NP;   // CTA-uniform
    const int64_t env = a.done_list[r];
    const int64_t p = r % a.M;                   // pool entry
    if (part == 0) {
      if (threadIdx.x == 0) {
        atomicAdd(a.st_episodes, 1ull);
        atomicAdd(a.st_steps, (unsigned long long)S.ep_length[env]);
        atomicAdd(a.st_return, S.ep_return[env]);
      }
      for (int q = threadIdx.x; q < A; q += blockDim.x)
        if ((GR_AT(S, GR_F_ACH, uint32_t, q >> 5, env) >> (q & 31)) & 1u) atomicAdd(&a.st_ach[q], 1ull);
      __syncthreads();
      install_fields<EXT>(S, env, a.pool.meta[p]);
    }
    install_maps<EXT>(S, env, a.pool.blocks + (size_t)p * F * HW, a.pool.items + (size_t)p * F * HW, part, NP);
    __syncthreads();
  }
}

void launch_finish_info(const int32_t* ex_all, int rank, int world, int64_t M, uint64_t pool_key,
                        unsigned long long* dstep, StepInfo* info, uint32_t* flags_out, cudaStream_t st) {
  k_finish_info<<<1, 1, 0, st>>>(ex_all, rank, world, M, pool_key, dstep, info, flags_out);
}

void launch_install_initial(bool ext, const DS& S, const WBuf& wb, int64_t n, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>(n, 148 * 16);
  if (grid <= 0) return;
  if (ext) k_install_initial<true><<<grid, 128, 0, st>>>(S, wb, n);
  else k_install_initial<false><<<grid, 128, 0, st>>>(S, wb, n);
}

void launch_compact(const uint8_t* done, int64_t n, const int32_t* block_off, int32_t* list, cudaStream_t st) {
  const int grid = (int)((n + 127) / 128);
  if (grid > 0) k_compact<<<grid, 128, 0, st>>>(done, n, block_off, list);
}

void launch_install_pool(bool ext, const DS& S, const InstallArgs& a, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(a.n * a.parts, (int64_t)sms * 4);
  if (grid <= 0) return;
  if (ext) k_install_pool<true><<<grid, 128, 0, st>>>(S, a);
  else k_install_pool<false><<<grid, 128, 0, st>>>(S, a);
}

}  // namespace gr
