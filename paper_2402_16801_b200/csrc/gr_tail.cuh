// gr_tail.cuh -- the per-step bookkeeping after the env update: exclusive
// scan of the per-block done counts, the exchange record, and the combine
// of the all-gathered records into StepInfo (batch.py:206-231).  The last
// CTA of k_step runs the scan and writes the exchange record; the combine
// runs there too for one-shard steps (no extra launches), or in
// k_finish_info after the all-gather of a multi-shard step.
#pragma once
#include <cstdint>
#include "gr_device.cuh"
#include "gr_kernels.cuh"

namespace gr {

// exclusive scan of block_done[0, nb) into block_off by the whole CTA
// (blockDim.x a multiple of 32, <= 1024); returns the total to every thread
__device__ __forceinline__ int32_t cta_scan_blocks(const int32_t* block_done, int32_t* block_off, int nb) {
  __shared__ int32_t warp_tot[32];
  __shared__ int32_t carry;
  const int nw = blockDim.x >> 5, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int v = i < nb ? *((volatile const int32_t*)block_done + i) : 0;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = lane < nw ? warp_tot[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_tot[lane] = w;
    }
    __syncthreads();
    const int wpre = warp ? warp_tot[warp - 1] : 0;
    if (i < nb) block_off[i] = carry + wpre + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_tot[31];
    __syncthreads();
  }
  return carry;
}

// combine the exchange records of every rank (one thread).  The step
// counter lives on the device (so a captured step graph replays as is):
// the pool serving this step is WorldPool(pool_key, step + 1, M)
// (batch.py:217), and the counter advances here, once per step.
__device__ __forceinline__ void combine_info(const int32_t* ex_all, int rank, int world, int64_t M, uint64_t pool_key,
                                             unsigned long long* dstep, StepInfo* info, uint32_t* flags_out,
                                             bool advance = true) {
  const unsigned long long step = *dstep;
  const uint64_t step_key = hash2(pool_key, (uint64_t)(step + 1));
  if (advance) *dstep = step + 1;   // else k_install_pool advances it (speculative pool)
  int off = 0;
  uint32_t fl = 0;
  for (int r = 0; r < world; ++r) {
    if (r < rank) off += ex_all[4 * r];
    fl |= (uint32_t)ex_all[4 * r + 1];
  }
  const int k = ex_all[4 * rank];
  info->k_local = k;
  info->offset = off;
  info->n_pool = (int32_t)(k < M ? k : M);
  info->flags = fl;
  info->step_key = step_key;
  *flags_out = fl;
}

}  // namespace gr
