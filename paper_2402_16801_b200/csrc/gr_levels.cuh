// gr_levels.cuh -- level buffers (UED): mutation operators and install.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "gr_state.cuh"
#include "gr_kernels.cuh"

namespace gr {

enum { MUT_NOISE = 0, MUT_SWAP = 1, MUT_RSWAP = 2 };   // == GR_MUT_* of the C ABI

void launch_mutate(bool ext, int op, const LevelParamsBuf& p, const WBuf& w, const int64_t* idx, const uint64_t* key,
                   const uint64_t* ctr, int64_t count, double scale, cudaStream_t st);
// level_idx[k] -> env_idx[k] with install key keys[k] (install_world)
void launch_install_levels(bool ext, const DS& S, const WBuf& w, const int64_t* env_idx, const int64_t* level_idx,
                           const uint64_t* keys, int64_t count, cudaStream_t st);

}  // namespace gr
