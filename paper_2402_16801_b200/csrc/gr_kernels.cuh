// gr_kernels.cuh -- kernel argument blocks and host-side launchers.
#pragma once
#include <atomic>
#include <mutex>
#include <cstdint>
#include <cuda_runtime.h>
#include "gr_state.cuh"

namespace gr {

// Launch attributes (cudaFuncSetAttribute) belong to each device's context:
// `init` runs once per device per process, before any caller on that device
// proceeds (handles may live on different devices and threads).
struct PerDeviceOnce {
  std::atomic<uint64_t> done{0};
  std::mutex m;
  template <class F>
  void operator()(F&& init) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    std::lock_guard<std::mutex> g(m);
    if (done.load(std::memory_order_relaxed) & bit) return;
    init(dev & 63);
    done.fetch_or(bit, std::memory_order_release);
  }
};


struct StepInfo;
struct StepArgs {
  const int64_t* actions;   // int64[n]
  float* reward;            // float32[n]
  double* reward64;         // optional float64[n]
  uint8_t* done;            // uint8[n]
  uint8_t* newly;           // optional uint8[n, A]
  uint32_t* itime;          // optional
  uint8_t* ifloor;          // optional
  int64_t n;
  int64_t max_len;
  const uint32_t* prev_flags;  // batch-wide flags of the previous step
  uint32_t* cur_flags;         // this step: bit0 melee alive, bit1 ranged alive, bit2 dark floor
  int32_t* block_done;         // done count per 128-env block
  const int64_t* bad;          // >=0: validation failed, do nothing
  // step tail run by the last CTA to finish (arrive != null): done-count
  // scan -> block_off, exchange record; with info != null (one shard) also
  // the StepInfo combine of k_finish_info
  unsigned int* arrive;        // CTA arrival counter, 0 between steps
  int32_t* block_off;
  int nb;
  int32_t* exchange;
  StepInfo* info;
  uint64_t pool_key;
  unsigned long long* dstep;   // device step counter (combine_info)
  int64_t M;
  uint32_t* flags_out;
  int defer_advance;           // 1: the counter advances in k_install_pool (speculative pool)
};

// step bookkeeping shared by the post-step kernels (device memory)
struct StepInfo {
  int32_t k_local;      // done envs of this shard
  int32_t offset;       // global rank of this shard's first done env
  int32_t n_pool;       // worlds to generate = min(k_local, M)
  int32_t pad;
  uint32_t flags;       // OR over ranks of cur_flags
  uint32_t pad2;
  uint64_t step_key;    // WorldPool._step_key of the pool serving this step
};

// explicit LevelParams (worldgen.LevelParams) of a level buffer
struct LevelParamsBuf {
  uint64_t* seed;         // [cap]
  float* angles;          // [cap][252]: the overworld octave grids, flattened in order
  uint64_t* floor_seed;   // [cap][9]
};

struct WorldJob {
  int mode;               // 0: initial reset (env-indexed seeds), 1: pool, 2: explicit params
  int64_t count;          // worlds (mode 0: n envs; mode 1: read from info->n_pool)
  const StepInfo* info;   // mode 1
  uint64_t env_key;       // mode 0: split(make_stream(seed), 0).key
  int64_t env_offset;     // mode 0: global index of env 0
  int64_t M;              // pool size (mode 1)
  WBuf out;
  unsigned long long* counters;  // [5] diagnostics
  int ctas_per_sm;               // resident CTAs per SM (0 = default)
  LevelParamsBuf params;         // mode 2: world w of the job <- params / out slot first + w
  int64_t first;
  // speculative pool (one shard): mode 3 generates slots [0, *spec_k) of the
  // pool of the step about to run, WorldPool(pool_key, *dstep + 1), before
  // its done count is known; mode 1 with spec_k set then generates only
  // slots [min(*spec_k, n_pool), n_pool)
  const int32_t* spec_k;
  uint64_t pool_key;
  const unsigned long long* dstep;
  int wide;                      // extended tier: 512-thread CTAs (gr_world_wide.cu)
  int pdl = 0;                   // launch as a programmatic dependent of the preceding kernel in the stream
  int max_attempts = 16;         // worldgen.MAX_GEN_RETRIES (worldgen.py:36)
};

struct InstallArgs {
  int mode;                   // 0: initial (world w -> env w, maps already in place), 1: pool
  // speculative pool: CTA 0 advances the step counter (deferred from the
  // step tail, so the speculative worldgen read a stable value) and sizes
  // the next step's speculation from this step's n_pool
  unsigned long long* dstep_advance;
  int32_t* spec_k;
  int64_t spec_cap;
  int64_t n;                  // mode 0 env count
  int parts;                  // mode 1: CTAs per installed env (>= 1)
  const int32_t* done_list;   // mode 1: env index per local done rank (k_compact)
  const StepInfo* info;
  WBuf pool;
  int64_t M;
  // EpisodeStats accumulators (batch.py:109-124)
  unsigned long long* st_episodes;
  unsigned long long* st_steps;
  double* st_return;
  unsigned long long* st_ach;    // [A]
};

struct ObsArgs {
  void* out;                // float32[n, L] or uint8[n, H, W, 3]
  int64_t n;
  const uint32_t* flags;    // bit2: some env stands on a dark floor (glow on)
  int tile_px;
  const uint8_t* done;      // this step's done flags (for sel 1/2)
  int sel;                  // 0: every env, 1: envs not reset this step, 2: envs reset this step
  int tma;                  // extended rows leave shared memory through TMA bulk stores
  int ctas_per_sm;          // resident CTAs per SM of the writer (0 = default)
  const int32_t* list;      // sel 2: the done list (k_compact) ...
  const StepInfo* info;     // ... of info->k_local entries
  uint32_t* pix;            // pixels: per-env scratch of k_pixprep (pix_words per env)
};

// words per env of the pixel scratch (k_pixprep -> k_pixels): tile colours,
// inset colours, bar fills, padded to a 16-byte multiple
__host__ __device__ constexpr int pix_scratch_words(bool ext) { return ext ? 212 : 140; }

void launch_step(bool ext, const DS& S, const StepArgs& a, cudaStream_t st);
void launch_init_lut(float* lut, cudaStream_t st);
void launch_make_desc(bool ext, const DS& S, int64_t n, cudaStream_t st);
void launch_worldgen(bool ext, const WorldJob& j, cudaStream_t st);
// make_level_params(seed) for params slots [first, first + count) (seeds already set)
void launch_level_params(const LevelParamsBuf& p, int64_t first, int64_t count, cudaStream_t st);
void launch_install(bool ext, const DS& S, const InstallArgs& a, int64_t grid_envs, cudaStream_t st);
void launch_pixprep(bool ext, const DS& S, const ObsArgs& a, cudaStream_t st);
void launch_symbolic(bool ext, const DS& S, const ObsArgs& a, cudaStream_t st);
void launch_pixels(bool ext, const DS& S, const ObsArgs& a, cudaStream_t st);
// the row-class structure of a pixel frame (gr_obs.cu): row y of a frame is
// the class row in slot slot_of_row[y]; rep[k] is a row of slot k's class
struct PixRowMap {
  int FH, RB, FB, nused;
  int16_t slot_of_row[176];
  int16_t rep[64];
};
int pixel_row_map(bool ext, int px, PixRowMap* m);
void launch_pix_gather(const uint8_t* frames, int64_t r0, int64_t r1, const PixRowMap& m, uint8_t* out,
                       cudaStream_t st);

}  // namespace gr
