// gr_api.cu -- the C ABI (include/gridrogue_b200.h): device state
// ownership, the per-step launch sequence, and the reference-layout state
// channel.
//
// One step (BatchEnv.step, bindings/.../__init__.py:63-84) on the handle's
// stream:
//   k_step        game logic for every env, rewards/done/info, per-block
//                 done counts, batch-wide flags; its last CTA scans the
//                 done counts -> local done ranks + exchange record, and
//                 for one shard combines StepInfo       (gr_step.cu)
//   [all-gather of the 4 x int32 exchange record + k_finish_info -- multi-GPU only]
//   k_compact     done list (side stream from here on, beside the obs)
//   k_worldgen    fresh worlds for the pool slots this shard consumes
//   k_install_pool  EpisodeStats + install_worlds for done envs
//   k_symbolic_stage / k_pixels  post-reset observation
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdarg>
#include <cstdlib>
#include <climits>
#include <string>
#include <vector>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <cuda_runtime.h>
#include <immintrin.h>

#include "gr_device.cuh"
#include "gr_state.cuh"
#include "gr_kernels.cuh"
#include "gr_desc.cuh"
#include "gr_levels.cuh"

namespace gr {
void launch_finish_info(const int32_t* ex_all, int rank, int world, int64_t M, uint64_t pool_key,
                        unsigned long long* dstep, StepInfo* info, uint32_t* flags_out, cudaStream_t st);
void launch_install_initial(bool ext, const DS& S, const WBuf& wb, int64_t n, cudaStream_t st);
void launch_install_pool(bool ext, const DS& S, const InstallArgs& a, cudaStream_t st);
void launch_compact(const uint8_t* done, int64_t n, const int32_t* block_off, int32_t* list, cudaStream_t st);

// policies.RandomPolicy.actions (policies.py:31-37)
__global__ void k_random_actions(int64_t* out, int64_t n, int64_t env0, uint32_t key, int na) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float u = u32f(key, (uint32_t)(env0 + i));
  out[i] = (int64_t)__fmul_rn(u, (float)na) % na;
}

// numerics self-test (gr_selftest_*): the device routines worldgen uses
__global__ void k_selftest_sincos64(const float* x, double* s, double* c, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = (double)x[i];
  s[i] = gl_sin(v);
  c[i] = gl_cos(v);
}
__global__ void k_selftest_argsort6(const float* keys, uint8_t* idx, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float v[6];
  uint8_t o[6];
  for (int k = 0; k < 6; ++k) v[k] = keys[i * 6 + k];
  np_argsort6(v, o);
  for (int k = 0; k < 6; ++k) idx[i * 6 + k] = o[k];
}

// first invalid action (engine.py:715-717)
__global__ void k_validate(const int64_t* a, int64_t n, int na, unsigned long long* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && (a[i] < 0 || a[i] >= na)) atomicMin(bad, (unsigned long long)i);
}

// bit2 of flags: does some env stand on a dark floor (obs.py:236)
__global__ void k_dark(DS S, int64_t n, uint32_t* flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool d = i < n && C_FLOOR_AMB[GR_AT(S, GR_F_PFLOOR, uint8_t, 0, i)] < 1.0f;
  if (__syncthreads_or(d) && threadIdx.x == 0) atomicOr(flags, 4u);
}

// apply the deferred dead-lane cooldown decrements (see gr_step.cu)
__global__ void k_materialize(DS S, int64_t n, int F, const uint32_t* flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t p = S.cd_pending[i];
  if (!p) return;
  const int pf = F > 1 ? GR_AT(S, GR_F_PFLOOR, uint8_t, 0, i) : 0;
  const uint32_t fl = flags[0];
  for (int l = 0; l < 3; ++l)
    if ((fl & 1u) && ((p >> l) & 1)) {
      uint8_t& c = GR_AT(S, GR_F_MEL_CD, uint8_t, pf * 3 + l, i);
      if (c > 0) c -= 1;
    }
  for (int l = 0; l < 2; ++l)
    if ((fl & 2u) && ((p >> (3 + l)) & 1)) {
      uint8_t& c = GR_AT(S, GR_F_RAN_CD, uint8_t, pf * 2 + l, i);
      if (c > 0) c -= 1;
    }
  S.cd_pending[i] = 0;
}

}  // namespace gr

using namespace gr;

static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) return fail(GR_E_CUDA, "%s: %s", #x, cudaGetErrorString(e_));   \
  } while (0)

// per-kernel CUDA-event timing (gr_set_profiling / gr_kernel_times)
enum { PK_STEP, PK_SCAN, PK_INFO, PK_WORLDGEN, PK_INSTALL, PK_OBS, PK_POLICY, PK_OTHER, PK_OBS_RESET, PK_OBS_PREP,
       PK_N };

struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[PK_N];
  cudaEvent_t get() {
    if (pool.empty()) {
      cudaEvent_t x;
      cudaEventCreate(&x);
      return x;
    }
    cudaEvent_t x = pool.back();
    pool.pop_back();
    return x;
  }
};

struct StepGraph {
  const void* key[7];   // actions, obs, reward, done, newly, time, floor
  cudaGraphExec_t exec;
  int64_t launches;     // kernels per replay
};

// A host observation buffer whose contents the handle owns
// (gr_host_obs_attach): `shadow` is a device copy of what the host buffer
// holds, so a delivery moves only the words that changed since the last
// observation written into this buffer.
struct HostObs {
  uint32_t* ptr = nullptr;      // host
  uint32_t* shadow = nullptr;   // device, same contents
  bool dirty = false;           // host and shadow may differ (an interrupted delivery): re-zero both
};

// A small persistent pool of host threads for the delta scatter (no OpenMP
// runtime in the library: the process already carries torch's).
class HostPool {
 public:
  explicit HostPool(int n) : n_(std::max(1, n)) {
    for (int k = 1; k < n_; ++k) th_.emplace_back([this, k] { loop(k); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return n_; }
  // fn(lo, hi) over n_ contiguous parts of [0, count); the caller runs part 0;
  // below min_parallel items the caller does it all (waking the pool costs more)
  void run(int64_t count, const std::function<void(int64_t, int64_t)>& fn, int64_t min_parallel = 4096) {
    if (count <= 0) return;
    if (n_ == 1 || count < min_parallel) { fn(0, count); return; }
    {
      std::lock_guard<std::mutex> g(m_);
      fn_ = &fn;
      count_ = count;
      left_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0, part(0));
    std::unique_lock<std::mutex> g(m_);
    done_cv_.wait(g, [this] { return left_ == 0; });
  }

 private:
  int64_t part(int k) const { return count_ * (k + 1) / n_; }
  void loop(int k) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int64_t, int64_t)>* fn;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        fn = fn_;
      }
      (*fn)(count_ * k / n_, part(k));
      std::lock_guard<std::mutex> g(m_);
      if (--left_ == 0) done_cv_.notify_one();
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  uint64_t gen_ = 0;
  bool stop_ = false;
  const std::function<void(int64_t, int64_t)>* fn_ = nullptr;
  int64_t count_ = 0;
  int left_ = 0;
};

#ifndef GR_DL_CHUNKS
#define GR_DL_CHUNKS 16   // 8 / 16 / 32 measured: 16 best on average (pixels 2.3 -> 2.5 M, symbolic within noise)
#endif
constexpr int DL_CHUNKS = GR_DL_CHUNKS;   // row chunks of one delivery: chunk c's scatter overlaps chunk c+1's kernel

struct gr_env {
  Prof prof;
  gr_config cfg;
  bool ext;
  TierDims d;
  int64_t n, M, nb;
  DS S;
  WBuf pool;
  WMeta* init_meta = nullptr;
  int32_t *block_done = nullptr, *block_off = nullptr, *exchange = nullptr;
  int32_t* done_list = nullptr;     // this step's done envs, local rank order
  unsigned int* arrive = nullptr;   // k_step CTA arrival counter
  uint32_t* pix = nullptr;          // pixels: k_pixprep -> k_pixels scratch
  unsigned long long* dstep = nullptr;   // device step counter (pool of step s = WorldPool(s + 1))
  uint32_t *cur_flags = nullptr, *prev_flags = nullptr;
  StepInfo* info = nullptr;
  unsigned long long* bad = nullptr;
  unsigned long long* counters = nullptr;       // worldgen [5]
  unsigned long long *st_episodes = nullptr, *st_steps = nullptr, *st_ach = nullptr;
  double* st_return = nullptr;
  uint64_t pool_key = 0, env_key = 0;
  int64_t step_index = 0;
  bool have_reset = false;
  bool validate = true;
  int wg_attempts = 16;       // worldgen.MAX_GEN_RETRIES (gr_set_worldgen_attempts)
  int64_t launches = 0;
  int64_t last_bad_env = -1, last_bad_action = 0;
  // e2e scratch
  void* h_obs_dev = nullptr;
  int64_t* h_act_dev = nullptr;
  float* h_rew_dev = nullptr;
  uint8_t *h_done_dev = nullptr, *h_newly_dev = nullptr, *h_floor_dev = nullptr;
  uint32_t* h_time_dev = nullptr;
  cudaStream_t h_stream = nullptr;
  // delta observation transfer into attached host buffers
  std::vector<HostObs> host_obs;
  // the changed-word list: device copy written by k_obs_delta, pinned host
  // stage it is copied into chunk by chunk on dl_copy
  uint2* dl_host = nullptr;
  uint2* dl_dev = nullptr;
  int64_t dl_cap = 0;                          // entries, split evenly over DL_CHUNKS
  unsigned long long* dl_cnt_host = nullptr;   // [DL_CHUNKS] pinned copies of the chunk counters
  unsigned long long* dl_cnt_dev = nullptr;
  cudaStream_t dl_copy = nullptr;
  cudaEvent_t dl_ev[DL_CHUNKS] = {};           // chunk listed + its count on the host
  cudaEvent_t dl_evd[DL_CHUNKS] = {};          // chunk's list on the host
  std::unique_ptr<HostPool> hpool;            // host threads of the delta scatter
  int scatter_prefetch = 16;                   // GR_SCATTER_PF: prefetch distance of the scatter (0: off)
  // compact transfer of symbolic observations into plain host arrays: per
  // row a non-zero bitmap + the row's offset into a packed value list
  uint32_t* cp_bm_dev = nullptr;               // [n][NB] bitmaps
  uint32_t* cp_val_dev = nullptr;              // [n][W] worst case: chunk c packs into rows [r0, r1)'s region
  int64_t* cp_off_dev = nullptr;               // [n] offset of each row's values in its chunk's list
  uint32_t* cp_bm_host = nullptr;              // pinned twins
  uint32_t* cp_val_host = nullptr;             // capacity cp_val_cap words, split over the chunks
  int64_t* cp_off_host = nullptr;
  int64_t cp_val_cap = 0;
  bool compact = true;                         // GR_HOST_COMPACT=0: plain 2 GB copy into the host array
  // pixel frames to plain host arrays: one row per row class
  PixRowMap prmap{};
  uint8_t* pr_dev = nullptr;                   // [n][nused][RB] class rows
  uint8_t* pr_stage[2] = {nullptr, nullptr};   // pinned, one chunk each
  double host_ms[4] = {0, 0, 0, 0};            // enqueue, wait, scatter / decode, tail (gr_host_phase_times)
  int64_t host_calls = 0;
  int64_t host_words = 0;                      // changed words delivered
  // reset work (worldgen + install + obs of reset envs) overlaps the obs of
  // the other envs on a second stream
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  const uint8_t* last_done = nullptr;
  bool overlap = true;    // GR_OVERLAP=0: reset work serialised after the step on one stream
  bool tma = true;        // GR_TMA=0: plain 16-byte stores for the observation rows
  int obs_ctas_overlap = 2;   // writer CTAs/SM while the reset work runs beside it
  int obs_ctas_solo = 0;      // writer CTAs/SM otherwise (0: launcher default)
  int wg_ctas = 0;            // worldgen CTAs/SM (0: launcher default)
  bool obs_first = true;      // enqueue the big obs launch before the reset work (GR_OBS_FIRST=0: after);
                              // inside a step graph the other order starves the writer (0.55 vs 0.49 ms)
  int side_prio = 0;          // side stream priority (0 default, >0 lowest, <0 highest)
  bool graph_prio = true;     // GR_GRAPH_PRIO=0: step graphs instantiated without per-node priorities
  int install_parts = 1;      // CTAs per env in the pool install (GR_INSTALL_PARTS; 4 up to 16,384 extended envs)
  bool spec_pdl = true;       // GR_SPEC_PDL=0: the speculative pass as a second graph root on the side stream
  bool spec_main = false;     // this step's speculative pass runs behind k_step on the caller's stream
  cudaEvent_t ev_k = nullptr; // k_step complete (spec_pdl)
  bool graphs = true;         // GR_GRAPH=0: launch the step kernel by kernel
  // speculative pool (one-shard steps): the side stream generates the first
  // spec_k worlds of this step's pool beside k_step, before the done count
  // is known; on by default while k_step's grid leaves SMs free (GR_SPEC=0/1)
  bool spec_on = false;
  bool wg_wide = false;       // pool worldgen with 512-thread extended CTAs (small batches; GR_WG_WIDE=0/1)
  bool spec_pending = false;
  int32_t* spec_k = nullptr;
  cudaEvent_t ev_spec = nullptr;
  cudaStream_t cap_stream = nullptr;
  std::vector<StepGraph> step_graphs;
  std::vector<void*> allocs;
};

// records a (start, stop) event pair around one launch when profiling
struct PTimer {
  gr_env* e;
  int cls;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  PTimer(gr_env* e_, int cls_, cudaStream_t st_) : e(e_), cls(cls_), st(st_) {
    if (e->prof.on) {
      a = e->prof.get();
      b = e->prof.get();
      cudaEventRecord(a, st);
    }
    e->launches++;
  }
  ~PTimer() {
    if (a) {
      cudaEventRecord(b, st);
      e->prof.ev[cls].push_back({a, b});
    }
  }
};

static int64_t obs_elems_of(const gr_env* e) {
  if (e->cfg.obs_mode == GR_OBS_SYMBOLIC) return e->ext ? 8268 : 1345;
  if (e->cfg.obs_mode == GR_OBS_PIXELS) {
    const int px = e->cfg.tile_px;
    return (int64_t)(e->d.VR + 2) * px * (e->d.VC + (e->ext ? 2 : 0)) * px * 3;
  }
  return 0;
}

static int dev_alloc(gr_env* e, void** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t err = cudaMalloc(p, bytes);
  if (err != cudaSuccess) return fail(GR_E_OOM, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(err));
  e->allocs.push_back(*p);
  err = cudaMemset(*p, 0, bytes);
  if (err != cudaSuccess) return fail(GR_E_CUDA, "cudaMemset: %s", cudaGetErrorString(err));
  return GR_OK;
}

// ---------------------------------------------------------- level buffers
struct gr_levels {
  gr_env* e;
  int64_t cap;
  WBuf w;
  LevelParamsBuf p;
  std::vector<void*> allocs;
};

// host index / key arrays -> device scratch (freed on return)
struct DevArrays {
  std::vector<void*> p;
  ~DevArrays() {
    for (void* q : p) cudaFree(q);
  }
  template <class T>
  T* put(const T* host, int64_t n) {
    void* d = nullptr;
    if (cudaMalloc(&d, std::max<int64_t>(n, 1) * sizeof(T)) != cudaSuccess) return nullptr;
    p.push_back(d);
    if (n && cudaMemcpy(d, host, n * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    return (T*)d;
  }
};

extern "C" {

const char* gr_last_error(void) { return g_err.c_str(); }
int gr_version(void) { return GR_ABI_VERSION; }

int gr_field_info(int32_t tier, int32_t field, int64_t* elems_per_env, int32_t* elem_size) {
  if (field < 0 || field >= GR_NFIELDS) return fail(GR_E_INVALID, "unknown field id %d", field);
  if (tier != GR_TIER_CLASSIC && tier != GR_TIER_EXTENDED) return fail(GR_E_INVALID, "unknown tier %d", tier);
  const TierDims& d = tier == GR_TIER_EXTENDED ? EXT_DIMS : CLASSIC_DIMS;
  if (elems_per_env) *elems_per_env = ref_elems(field, d);
  if (elem_size) *elem_size = ref_esz(field);
  return GR_OK;
}

void gr_destroy(gr_env* e) {
  if (!e) return;
  cudaSetDevice(e->cfg.device);
  cudaDeviceSynchronize();
  for (void* p : e->allocs) cudaFree(p);
  if (e->h_stream) cudaStreamDestroy(e->h_stream);
  for (auto& h : e->host_obs)
    if (h.shadow) cudaFree(h.shadow);
  if (e->dl_host) cudaFreeHost(e->dl_host);
  if (e->dl_dev) cudaFree(e->dl_dev);
  if (e->cp_bm_dev) cudaFree(e->cp_bm_dev);
  if (e->cp_val_dev) cudaFree(e->cp_val_dev);
  if (e->cp_off_dev) cudaFree(e->cp_off_dev);
  if (e->cp_bm_host) cudaFreeHost(e->cp_bm_host);
  if (e->cp_val_host) cudaFreeHost(e->cp_val_host);
  if (e->cp_off_host) cudaFreeHost(e->cp_off_host);
  if (e->pr_dev) cudaFree(e->pr_dev);
  for (auto& p : e->pr_stage)
    if (p) cudaFreeHost(p);
  if (e->dl_cnt_host) cudaFreeHost(e->dl_cnt_host);
  if (e->dl_cnt_dev) cudaFree(e->dl_cnt_dev);
  if (e->dl_copy) cudaStreamDestroy(e->dl_copy);
  for (auto& ev : e->dl_ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : e->dl_evd)
    if (ev) cudaEventDestroy(ev);
  e->hpool.reset();
  if (e->side) cudaStreamDestroy(e->side);
  for (auto& g : e->step_graphs) cudaGraphExecDestroy(g.exec);
  if (e->cap_stream) cudaStreamDestroy(e->cap_stream);
  if (e->ev_fork) cudaEventDestroy(e->ev_fork);
  if (e->ev_join) cudaEventDestroy(e->ev_join);
  if (e->ev_spec) cudaEventDestroy(e->ev_spec);
  if (e->ev_k) cudaEventDestroy(e->ev_k);
  for (auto x : e->prof.pool) cudaEventDestroy(x);
  delete e;
}

int gr_create(const gr_config* cfg, gr_env** out) {
  if (!cfg || !out) return fail(GR_E_INVALID, "null argument");
  *out = nullptr;
  if (cfg->tier != GR_TIER_CLASSIC && cfg->tier != GR_TIER_EXTENDED)
    return fail(GR_E_INVALID, "unknown tier %d", cfg->tier);
  if (cfg->obs_mode < GR_OBS_NONE || cfg->obs_mode > GR_OBS_PIXELS)
    return fail(GR_E_INVALID, "unknown obs_mode %d", cfg->obs_mode);
  if (cfg->obs_mode == GR_OBS_PIXELS && cfg->tile_px != 7 && cfg->tile_px != 10 && cfg->tile_px != 16)
    return fail(GR_E_INVALID, "tile_px must be one of (7, 10, 16)");
  if (cfg->n_envs < 1) return fail(GR_E_INVALID, "n_envs must be >= 1");
  if (cfg->reset_ratio < 1) return fail(GR_E_INVALID, "reset_ratio must be >= 1");
  const int64_t ng = cfg->n_envs_global > 0 ? cfg->n_envs_global : cfg->n_envs;
  if (cfg->env_offset < 0 || cfg->env_offset + cfg->n_envs > ng)
    return fail(GR_E_INVALID, "shard [%lld, %lld) outside the %lld-env batch", (long long)cfg->env_offset,
                (long long)(cfg->env_offset + cfg->n_envs), (long long)ng);
  cudaError_t ce = cudaSetDevice(cfg->device);
  if (ce != cudaSuccess) return fail(GR_E_CUDA, "cudaSetDevice(%d): %s", cfg->device, cudaGetErrorString(ce));
  gr_env* e = new gr_env();
  e->cfg = *cfg;
  e->cfg.n_envs_global = ng;
  if (e->cfg.max_episode_length <= 0) e->cfg.max_episode_length = 100000;
  if (const char* ov = getenv("GR_OVERLAP")) e->overlap = atoi(ov) != 0;
  if (const char* tm = getenv("GR_TMA")) e->tma = atoi(tm) != 0;
  if (const char* oc = getenv("GR_OBS_CTAS")) e->obs_ctas_overlap = atoi(oc);
  if (const char* oc = getenv("GR_OBS_CTAS0")) e->obs_ctas_solo = atoi(oc);
  // extended symbolic: the pool worldgen beside the writer at 3 CTAs/SM (not
  // 8) ends about when the writer does and leaves it more issue slots (writer
  // 0.407 -> 0.395 ms, step 0.470 -> 0.468; pixels and obs-off measured slower)
  // pool worldgen CTAs per SM beside the extended symbolic writer: 2 leave the
  // writer 0.396 ms instead of 0.406 at 65,536 envs while worldgen (0.31 ms)
  // still ends first (round 2, after the glibc sin/cos and dungeon early exit)
  if (cfg->tier == GR_TIER_EXTENDED && cfg->obs_mode == GR_OBS_SYMBOLIC) e->wg_ctas = cfg->n_envs >= 32768 ? 2 : 3;
  if (const char* wc = getenv("GR_WG_CTAS")) e->wg_ctas = atoi(wc);
  if (const char* of = getenv("GR_OBS_FIRST")) e->obs_first = atoi(of) != 0;
  if (const char* sp = getenv("GR_SIDE_PRIO")) e->side_prio = atoi(sp);
  if (const char* gp = getenv("GR_GRAPH_PRIO")) e->graph_prio = atoi(gp) != 0;
  e->install_parts = e->ext && cfg->n_envs <= 16384 ? 4 : 1;
  if (const char* ip = getenv("GR_INSTALL_PARTS")) e->install_parts = std::max(1, atoi(ip));
  // without observations the worldgen, not k_step, is the step's critical
  // path: there the speculative pass keeps its own root (worldgen first
  // pays: extended / classic obs-off 65,536 envs 335 / 774-833 M as a second
  // root vs 287 / 773-781 M behind k_step)
  e->spec_pdl = cfg->obs_mode != GR_OBS_NONE;
  if (const char* sp = getenv("GR_SPEC_PDL")) e->spec_pdl = atoi(sp) != 0;
  if (const char* gg = getenv("GR_GRAPH")) e->graphs = atoi(gg) != 0;
  if (const char* pf = getenv("GR_SCATTER_PF")) e->scatter_prefetch = atoi(pf);
  if (const char* hc = getenv("GR_HOST_COMPACT")) e->compact = atoi(hc) != 0;
  e->ext = cfg->tier == GR_TIER_EXTENDED;
  e->d = e->ext ? EXT_DIMS : CLASSIC_DIMS;
  e->n = cfg->n_envs;
  e->M = std::max<int64_t>(1, (ng + cfg->reset_ratio - 1) / cfg->reset_ratio);
  e->nb = (e->n + 127) / 128;
  {
    // below ~40 MB of observations per step the plain copy to a host array is
    // as quick as packing + waking the host threads (extended symbolic 1,024
    // envs, 34 MB: 1.14 vs 1.33 M env-steps/s packed vs copied; classic 8,192
    // envs, 44 MB: 10.3 vs 8.7 M; extended 4,096 / 16,384 / 65,536: 1.95 /
    // 3.34 / 3.89 vs 1.56 / 1.66 / 1.67 M)
    double min_mb = 40.0;
    if (const char* mm = getenv("GR_HOST_COMPACT_MIN_MB")) min_mb = atof(mm);
    const double mb = (double)obs_elems_of(e) * (e->cfg.obs_mode == GR_OBS_PIXELS ? 1 : 4) * e->n / 1048576.0;
    if (mb < min_mb) e->compact = false;
  }
  {
    // measured (tools/dev/spec_ab.sh): classic 1,024 envs 19.4 -> 24.3 M
    // env-steps/s, extended 4,096 28.7 -> 31.8 M; extended 16,384 88 ->
    // 81 M and 65,536 139 -> 110 M (the speculative CTAs crowd k_step and
    // the writer, and the extra worlds cost more than the hidden latency)
    // classic (one 64x64 floor per world, 256-thread worldgen CTAs) without
    // pixels gains at every size: symbolic 65,536 envs 414 -> 423 M, 16,384
    // 178 -> 204 M; obs off 65,536 749 -> 829 M, 4,096 74 -> 92 M.  Classic
    // pixels lose beyond 1,024 envs (4,096: 59.7 -> 57.1 M, 65,536: 171 -> 166 M)
    // Extended without observations (the reset chain follows k_step with no
    // writer to hide behind) gains too: 65,536 envs 288 -> 299 M.
    // End of round 2 the pass became k_step's programmatic dependent (it
    // starts once k_step's CTAs are resident, in every graph instantiation),
    // which removed the slow schedules the figures above were partly taken
    // from; re-measured: on for every classic and every pixel configuration
    // (classic pixels 4,096 / 65,536: 61.6 -> 66.7 / 180 -> 187 M; extended
    // pixels 4,096 / 16,384 / 65,536: 32.1 -> 34.7 / 55.7 -> 61.3 / 72.5 ->
    // 73.2 M) and for extended symbolic up to 16,384 envs (8,192: 61.1 ->
    // 71.8 M, 16,384: 95.7 -> 97.4 M; 24,576: 119 -> 110 M, 65,536: 143 -> 122 M)
    // Short episode caps (reset stress: thousands of worlds a step) leave it
    // off when there are observations: a quarter more worlds than needed
    // then costs more than it hides (extended pixels, 16-step episodes:
    // 69.7 M off, 63-64 M on either way)
    const bool short_eps = cfg->max_episode_length > 0 && cfg->max_episode_length < 64;
    const bool any_size = !e->ext || cfg->obs_mode == GR_OBS_PIXELS;
    e->spec_on = ng == cfg->n_envs &&
                 (cfg->obs_mode == GR_OBS_NONE || (!short_eps && (any_size || e->n <= 16384)));
    if (const char* sp = getenv("GR_SPEC")) e->spec_on = atoi(sp) != 0 && ng == cfg->n_envs;
    e->wg_wide = e->nb <= 64;   // 512-thread worldgen up to 8,192 envs (8,192: 0.1136 -> 0.1108 ms; 16,384: 0.169 -> 0.187)
    if (const char* ww = getenv("GR_WG_WIDE")) e->wg_wide = atoi(ww) != 0;
  }
  int rc = GR_OK;
  e->S.ns = e->n;
  for (int f = 0; f < GR_NFIELDS && rc == GR_OK; ++f) {
    const size_t bytes = (size_t)device_comps(f, e->d) * e->n * FIELD_TABLE[f].esz;
    rc = dev_alloc(e, &e->S.f[f], bytes);
  }
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->S.cd_pending, e->n);
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->S.ep_return, e->n * sizeof(double));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->S.ep_length, e->n * sizeof(int32_t));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->S.desc, e->n * 256);
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->S.torch_bits, e->n * sizeof(uint16_t));
  if (rc == GR_OK) {
    float* lut = nullptr;
    rc = dev_alloc(e, (void**)&lut, LUT_N * sizeof(float));
    if (rc == GR_OK) {
      launch_init_lut(lut, 0);
      if (cudaDeviceSynchronize() != cudaSuccess) rc = fail(GR_E_CUDA, "lut init failed");
    }
    e->S.lut = lut;
  }
  const int64_t cap = std::min(e->n, e->M);
  const size_t wbytes = (size_t)cap * e->d.F * e->d.H * e->d.W;
  e->pool.cap = cap;
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->pool.blocks, wbytes);
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->pool.items, wbytes);
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->pool.meta, cap * sizeof(WMeta));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->block_done, e->nb * sizeof(int32_t));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->block_off, e->nb * sizeof(int32_t));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->done_list, e->n * sizeof(int32_t));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->exchange, 4 * sizeof(int32_t));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->arrive, sizeof(unsigned int));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->dstep, sizeof(unsigned long long));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->spec_k, sizeof(int32_t));
  if (rc == GR_OK && cudaMemset(e->spec_k, 0, sizeof(int32_t)) != cudaSuccess) rc = fail(GR_E_CUDA, "memset");
  if (rc == GR_OK && cfg->obs_mode == GR_OBS_PIXELS)
    rc = dev_alloc(e, (void**)&e->pix, (size_t)e->n * pix_scratch_words(e->ext) * sizeof(uint32_t));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->cur_flags, sizeof(uint32_t));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->prev_flags, sizeof(uint32_t));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->info, sizeof(StepInfo));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->bad, sizeof(unsigned long long));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->counters, 5 * sizeof(unsigned long long));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->st_episodes, sizeof(unsigned long long));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->st_steps, sizeof(unsigned long long));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->st_ach, 67 * sizeof(unsigned long long));
  if (rc == GR_OK) rc = dev_alloc(e, (void**)&e->st_return, sizeof(double));
  if (rc == GR_OK) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);   // lo: least urgent
    // GR_SIDE_PRIO: > 0 least urgent, < 0 most urgent, 0 default
    if (cudaStreamCreateWithPriority(&e->side, cudaStreamNonBlocking,
                                     e->side_prio > 0 ? lo : e->side_prio < 0 ? hi : 0) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_spec, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_k, cudaEventDisableTiming) != cudaSuccess)
      rc = fail(GR_E_CUDA, "stream/event creation failed");
  }
  if (rc != GR_OK) {
    gr_destroy(e);
    return rc;
  }
  // batch.BatchState keys (batch.py:144-155)
  const uint64_t base = mix64(cfg->seed);
  e->pool_key = hash2(base, hash2(1, 0));
  e->env_key = hash2(base, hash2(0, 0));
  *out = e;
  return GR_OK;
}

int64_t gr_obs_elems(const gr_env* e) { return e ? obs_elems_of(e) : 0; }
int32_t gr_n_actions(const gr_env* e) { return e ? e->d.NA : 0; }
int32_t gr_n_achievements(const gr_env* e) { return e ? e->d.A : 0; }
int64_t gr_kernel_launches(const gr_env* e) { return e ? e->launches : 0; }

int gr_set_validate(gr_env* e, int32_t on) {
  if (!e) return fail(GR_E_INVALID, "null env");
  e->validate = on != 0;
  return GR_OK;
}

int gr_bad_action(const gr_env* e, int64_t* env_index, int64_t* action) {
  if (!e) return fail(GR_E_INVALID, "null env");
  if (env_index) *env_index = e->last_bad_env;
  if (action) *action = e->last_bad_action;
  return GR_OK;
}

// sel: 0 every env, 1 envs not reset this step, 2 envs reset this step
static int observe(gr_env* e, void* obs_dev, cudaStream_t st, bool recompute_flags, int sel = 0) {
  if (!obs_dev || e->cfg.obs_mode == GR_OBS_NONE) return GR_OK;
  if (recompute_flags) {
    CK(cudaMemsetAsync(e->cur_flags, 0, sizeof(uint32_t), st));
    PTimer t(e, PK_OTHER, st);
    k_dark<<<(unsigned)e->nb, 128, 0, st>>>(e->S, e->n, e->cur_flags);
  }
  ObsArgs oa{obs_dev, e->n, recompute_flags ? e->cur_flags : e->prev_flags, e->cfg.tile_px, e->last_done, sel,
             e->tma && (reinterpret_cast<uintptr_t>(obs_dev) & 15u) == 0 ? 1 : 0, sel == 1 ? e->obs_ctas_overlap : e->obs_ctas_solo, e->done_list, e->info,
             e->pix};
  const bool pixels = e->cfg.obs_mode == GR_OBS_PIXELS;
  if (pixels) {   // k_pixprep
    PTimer t(e, sel == 2 ? PK_OBS_RESET : PK_OBS_PREP, st);
    launch_pixprep(e->ext, e->S, oa, st);
  }
  {
    PTimer t(e, sel == 2 ? PK_OBS_RESET : PK_OBS, st);
    if (pixels) launch_pixels(e->ext, e->S, oa, st);
    else launch_symbolic(e->ext, e->S, oa, st);
  }
  if (recompute_flags) CK(cudaMemsetAsync(e->cur_flags, 0, sizeof(uint32_t), st));   // k_step expects it zero
  CK(cudaGetLastError());
  return GR_OK;
}

int gr_reset(gr_env* e, void* obs_dev, void* stream) {
  if (!e) return fail(GR_E_INVALID, "null env");
  CK(cudaSetDevice(e->cfg.device));
  cudaStream_t st = (cudaStream_t)stream;
  if (!e->init_meta) {
    int rc = dev_alloc(e, (void**)&e->init_meta, e->n * sizeof(WMeta));
    if (rc) return rc;
  }
  CK(cudaMemsetAsync(e->init_meta, 0, e->n * sizeof(WMeta), st));
  // batch_reset: world i = generate_world(make_level_params(split(env_stream, i).key))
  WorldJob j{};
  j.mode = 0;
  j.count = e->n;
  j.env_key = e->env_key;
  j.env_offset = e->cfg.env_offset;
  j.M = e->M;
  j.out = WBuf{(uint8_t*)e->S.f[GR_F_BLOCKS], (uint8_t*)e->S.f[GR_F_ITEMS], e->init_meta, e->n};
  j.counters = e->counters;
  j.max_attempts = e->wg_attempts;
  {
    PTimer t(e, PK_WORLDGEN, st);
    launch_worldgen(e->ext, j, st);
  }
  {
    PTimer t(e, PK_INSTALL, st);
    launch_install_initial(e->ext, e->S, j.out, e->n, st);
  }
  CK(cudaMemsetAsync(e->prev_flags, 0, sizeof(uint32_t), st));
  CK(cudaMemsetAsync(e->dstep, 0, sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(e->st_episodes, 0, sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(e->st_steps, 0, sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(e->st_ach, 0, 67 * sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(e->st_return, 0, sizeof(double), st));
  CK(cudaGetLastError());
  e->step_index = 0;
  e->have_reset = true;
  return observe(e, obs_dev, st, true);
}

int gr_random_actions(gr_env* e, uint32_t seed, uint64_t t, int64_t* actions_dev, void* stream) {
  if (!e || !actions_dev) return fail(GR_E_INVALID, "null argument");
  const uint32_t key = (uint32_t)((uint64_t)seed + t * 2654435761ull);
  PTimer tm(e, PK_POLICY, (cudaStream_t)stream);
  k_random_actions<<<(unsigned)((e->n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      actions_dev, e->n, e->cfg.env_offset, key, e->d.NA);
  CK(cudaGetLastError());
  return GR_OK;
}

// engine.py:715-717: the first invalid action raises before any mutation
static int validate_actions(gr_env* e, const int64_t* actions_dev, cudaStream_t st) {
  CK(cudaMemsetAsync(e->bad, 0xFF, sizeof(unsigned long long), st));
  {
    PTimer t(e, PK_OTHER, st);
    k_validate<<<(unsigned)((e->n + 255) / 256), 256, 0, st>>>(actions_dev, e->n, e->d.NA, e->bad);
  }
  unsigned long long bad = 0;
  CK(cudaMemcpyAsync(&bad, e->bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (bad != ~0ull) {
    int64_t a = 0;
    CK(cudaMemcpy(&a, actions_dev + bad, sizeof(a), cudaMemcpyDeviceToHost));
    e->last_bad_env = (int64_t)bad;
    e->last_bad_action = a;
    return fail(GR_E_BAD_ACTION, "invalid action %lld for env %lld", (long long)a, (long long)bad);
  }
  return GR_OK;
}

// the env update; its last CTA also runs the done-count scan and, for a
// one-shard step (fuse_info), the StepInfo combine
static int step_local(gr_env* e, const int64_t* actions_dev, float* reward_dev, uint8_t* done_dev,
                      uint8_t* newly_dev, uint32_t* time_dev, uint8_t* floor_dev, int32_t* exchange_dev, void* stream,
                      bool fuse_info, bool validate = true) {
  if (!e) return fail(GR_E_INVALID, "null env");
  if (!e->have_reset) return fail(GR_E_STATE, "call reset() before step()");
  if (!actions_dev || !reward_dev || !done_dev) return fail(GR_E_INVALID, "actions/reward/done are required");
  cudaStream_t st = (cudaStream_t)stream;
  if (e->validate && validate) {
    const int rc = validate_actions(e, actions_dev, st);
    if (rc) return rc;
  }
  // cur_flags is zero here: k_step's last CTA clears it after use, observe()
  // after its k_dark pass (no memset node per step)
  StepArgs a{};
  a.actions = actions_dev;
  a.reward = reward_dev;
  a.done = done_dev;
  a.newly = newly_dev;
  a.itime = time_dev;
  a.ifloor = floor_dev;
  a.n = e->n;
  a.max_len = e->cfg.max_episode_length;
  a.prev_flags = e->prev_flags;
  a.cur_flags = e->cur_flags;
  a.block_done = e->block_done;
  a.bad = nullptr;
  a.arrive = e->arrive;
  a.block_off = e->block_off;
  a.nb = (int)e->nb;
  a.exchange = exchange_dev ? exchange_dev : e->exchange;
  if (fuse_info) {
    a.info = e->info;
    a.pool_key = e->pool_key;
    a.dstep = e->dstep;
    a.M = e->M;
    a.flags_out = e->prev_flags;
  }
  e->spec_pending = false;
  const bool spec = fuse_info && e->spec_on;
  WorldJob sj{};
  if (spec) {
    // the first spec_k worlds of this step's pool beside k_step; k_step
    // leaves the step counter to k_install_pool so the speculative pass
    // reads a stable value
    sj.mode = 3;
    sj.M = e->M;
    sj.out = e->pool;
    sj.counters = e->counters;
    sj.max_attempts = e->wg_attempts;
    sj.ctas_per_sm = e->wg_ctas;
    sj.spec_k = e->spec_k;
    sj.pool_key = e->pool_key;
    sj.dstep = e->dstep;
    sj.wide = e->wg_wide;
    a.defer_advance = 1;
    e->spec_pending = true;
    e->spec_main = e->spec_pdl;
    if (!e->spec_pdl) {
      // a second root on the side stream.  Captured this way, about one graph
      // instantiation in four (classic 65,536 envs: one in two) dispatched
      // the worldgen's CTAs first; they fill the SMs and k_step starts ~18
      // us late (4,096 extended envs 0.114 instead of 0.087 ms per step)
      CK(cudaEventRecord(e->ev_fork, st));
      CK(cudaStreamWaitEvent(e->side, e->ev_fork, 0));
      {
        PTimer t(e, PK_WORLDGEN, e->side);
        launch_worldgen(e->ext, sj, e->side);
      }
      CK(cudaEventRecord(e->ev_spec, e->side));
    }
  }
  e->last_done = done_dev;
  {
    PTimer t(e, PK_STEP, st);
    launch_step(e->ext, e->S, a, st);
  }
  if (spec && e->spec_pdl) {
    // behind k_step on the same stream as its programmatic dependent: the
    // worldgen starts once every k_step CTA is resident and fills the rest
    // of the machine, in that order in every graph instantiation; the
    // observation writer moves to the side stream (step_finish)
    CK(cudaEventRecord(e->ev_k, st));
    sj.pdl = 1;
    PTimer t(e, PK_WORLDGEN, st);
    launch_worldgen(e->ext, sj, st);
  }
  CK(cudaGetLastError());
  return GR_OK;
}

int gr_step_local(gr_env* e, const int64_t* actions_dev, float* reward_dev, uint8_t* done_dev, uint8_t* newly_dev,
                  uint32_t* time_dev, uint8_t* floor_dev, int32_t* exchange_dev, void* stream) {
  return step_local(e, actions_dev, reward_dev, done_dev, newly_dev, time_dev, floor_dev, exchange_dev, stream, false);
}

static int step_finish(gr_env* e, const int32_t* exchange_all_dev, int32_t rank, int32_t world, void* obs_dev,
                       void* stream, bool info_done) {
  if (!e) return fail(GR_E_INVALID, "null env");
  if (world < 1 || rank < 0 || rank >= world) return fail(GR_E_INVALID, "bad rank %d / world %d", rank, world);
  cudaStream_t st = (cudaStream_t)stream;
  if (!info_done) {
    PTimer t(e, PK_INFO, st);
    launch_finish_info(exchange_all_dev ? exchange_all_dev : e->exchange, rank, world, e->M, e->pool_key, e->dstep,
                       e->info, e->prev_flags, st);
  }
  // reset work on the side stream, overlapping the obs of the other envs --
  // or, with the speculative pool behind k_step on the caller's stream
  // (spec_main), the reset work behind it there and the obs writer forked off
  const bool split = e->overlap && obs_dev && e->cfg.obs_mode != GR_OBS_NONE && e->last_done;
  const bool spec = e->spec_pending;
  const bool spec_main = spec && e->spec_main;
  e->spec_pending = false;
  cudaStream_t rs = split && !spec_main ? e->side : st;
  if (spec_main) CK(cudaStreamWaitEvent(st, e->ev_k, 0));   // k_step complete (the worldgen only followed its start)
  if (split) {
    if (spec_main) {
      CK(cudaStreamWaitEvent(e->side, e->ev_k, 0));
      const int rc = observe(e, obs_dev, e->side, false, 1);
      if (rc) return rc;
    } else {
      CK(cudaEventRecord(e->ev_fork, st));
      CK(cudaStreamWaitEvent(e->side, e->ev_fork, 0));
      if (e->obs_first) {   // the non-reset obs reaches the block scheduler first
        const int rc = observe(e, obs_dev, st, false, 1);
        if (rc) return rc;
      }
    }
  }
  {
    PTimer t(e, PK_SCAN, rs);
    launch_compact((const uint8_t*)e->S.f[GR_F_DONE], e->n, e->block_off, e->done_list, rs);
  }
  if (spec && !spec_main && rs != e->side) CK(cudaStreamWaitEvent(rs, e->ev_spec, 0));
  WorldJob j{};
  j.mode = 1;
  j.info = e->info;
  j.M = e->M;
  j.out = e->pool;
  j.counters = e->counters;
  j.max_attempts = e->wg_attempts;
  j.ctas_per_sm = e->wg_ctas;
  j.spec_k = spec ? e->spec_k : nullptr;   // only the slots the speculative pass did not make
  j.wide = e->wg_wide;
  {
    PTimer t(e, PK_WORLDGEN, rs);
    launch_worldgen(e->ext, j, rs);
  }
  InstallArgs ia{};
  ia.mode = 1;
  ia.n = e->n;
  ia.parts = e->install_parts;
  ia.done_list = e->done_list;
  ia.info = e->info;
  ia.pool = e->pool;
  ia.M = e->M;
  ia.st_episodes = e->st_episodes;
  ia.st_steps = e->st_steps;
  ia.st_return = e->st_return;
  ia.st_ach = e->st_ach;
  if (spec) {
    ia.dstep_advance = e->dstep;
    ia.spec_k = e->spec_k;
    ia.spec_cap = e->pool.cap;
  }
  {
    PTimer t(e, PK_INSTALL, rs);
    launch_install_pool(e->ext, e->S, ia, rs);
  }
  CK(cudaGetLastError());
  e->step_index += 1;
  if (!split) return observe(e, obs_dev, st, false);
  int rc = observe(e, obs_dev, rs, false, 2);   // reset envs, after their install
  if (rc) return rc;
  if (!e->obs_first && !spec_main) {
    rc = observe(e, obs_dev, st, false, 1);     // everyone else, concurrently
    if (rc) return rc;
  }
  CK(cudaEventRecord(e->ev_join, e->side));
  CK(cudaStreamWaitEvent(st, e->ev_join, 0));
  return GR_OK;
}

int gr_step_finish(gr_env* e, const int32_t* exchange_all_dev, int32_t rank, int32_t world, void* obs_dev,
                   void* stream) {
  return step_finish(e, exchange_all_dev, rank, world, obs_dev, stream, false);
}

int gr_account_replay(gr_env* e, int64_t steps, int64_t launches_per_step) {
  if (!e || steps < 0 || launches_per_step < 0) return fail(GR_E_INVALID, "bad replay accounting");
  e->step_index += steps;
  e->launches += steps * launches_per_step;
  return GR_OK;
}

// One-shard steps replay a CUDA graph of the whole launch sequence (step,
// scan tail, compaction, worldgen, install, observation writers on two
// streams), captured once per set of output buffers on the handle's own
// capture stream and launched into the caller's stream: the per-step
// inputs that change (the step counter and pool key) live on the device.
int gr_step(gr_env* e, const int64_t* actions_dev, void* obs_dev, float* reward_dev, uint8_t* done_dev,
            uint8_t* newly_dev, uint32_t* time_dev, uint8_t* floor_dev, void* stream) {
  if (!e) return fail(GR_E_INVALID, "null env");
  if (!e->graphs || e->prof.on) {
    int rc = step_local(e, actions_dev, reward_dev, done_dev, newly_dev, time_dev, floor_dev, nullptr, stream, true);
    if (rc) return rc;
    return step_finish(e, nullptr, 0, 1, obs_dev, stream, true);
  }
  if (!e->have_reset) return fail(GR_E_STATE, "call reset() before step()");
  if (!actions_dev || !reward_dev || !done_dev) return fail(GR_E_INVALID, "actions/reward/done are required");
  cudaStream_t st = (cudaStream_t)stream;
  if (e->validate) {
    const int rc = validate_actions(e, actions_dev, st);
    if (rc) return rc;
  }
  const void* key[7] = {actions_dev, obs_dev, reward_dev, done_dev, newly_dev, time_dev, floor_dev};
  StepGraph* g = nullptr;
  for (auto& x : e->step_graphs)
    if (!memcmp(x.key, key, sizeof(key))) g = &x;
  if (!g) {
    if (e->step_graphs.size() >= 4) {   // a small cache: buffers rarely change
      cudaGraphExecDestroy(e->step_graphs.front().exec);
      e->step_graphs.erase(e->step_graphs.begin());
    }
    if (!e->cap_stream) CK(cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking));
    const int64_t l0 = e->launches, s0 = e->step_index;
    CK(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal));
    int rc = step_local(e, actions_dev, reward_dev, done_dev, newly_dev, time_dev, floor_dev, nullptr, e->cap_stream,
                        true, false);
    if (!rc) rc = step_finish(e, nullptr, 0, 1, obs_dev, e->cap_stream, true);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(e->cap_stream, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (ce != cudaSuccess) return fail(GR_E_CUDA, "step graph capture: %s", cudaGetErrorString(ce));
    if (const char* dot = getenv("GR_GRAPH_DOT")) {   // dev: dump each captured step graph
      static int ndot = 0;
      char path[512];
      snprintf(path, sizeof(path), "%s.%d.dot", dot, ndot++);
      cudaGraphDebugDotPrint(graph, path, cudaGraphDebugDotFlagsVerbose);
    }
    StepGraph ng{};
    memcpy(ng.key, key, sizeof(key));
    // per-node priorities (all equal unless GR_SIDE_PRIO is set) make the
    // launch order of the graph's independent roots -- the speculative
    // worldgen and k_step -- the capture order: without the flag one
    // instantiation in about four dispatched k_step first, 0.115 instead of
    // 0.087 ms per step at 4,096 extended envs
    const cudaError_t ie =
        cudaGraphInstantiate(&ng.exec, graph, e->graph_prio ? cudaGraphInstantiateFlagUseNodePriority : 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) return fail(GR_E_CUDA, "step graph instantiate: %s", cudaGetErrorString(ie));
    ng.launches = e->launches - l0;
    e->launches = l0;        // nothing ran during the capture
    e->step_index = s0;
    e->step_graphs.push_back(ng);
    g = &e->step_graphs.back();
  }
  CK(cudaGraphLaunch(g->exec, st));
  e->launches += g->launches;
  e->step_index += 1;
  e->last_done = done_dev;
  return GR_OK;
}

static int ensure_host_scratch(gr_env* e) {
  if (e->h_act_dev) return GR_OK;
  int rc = dev_alloc(e, (void**)&e->h_act_dev, e->n * sizeof(int64_t));
  if (!rc) rc = dev_alloc(e, (void**)&e->h_rew_dev, e->n * sizeof(float));
  if (!rc) rc = dev_alloc(e, (void**)&e->h_done_dev, e->n);
  if (!rc) rc = dev_alloc(e, (void**)&e->h_newly_dev, e->n * e->d.A);
  if (!rc) rc = dev_alloc(e, (void**)&e->h_time_dev, e->n * sizeof(uint32_t));
  if (!rc) rc = dev_alloc(e, (void**)&e->h_floor_dev, e->n);
  const int64_t ob = obs_elems_of(e) * (e->cfg.obs_mode == GR_OBS_PIXELS ? 1 : 4);
  if (!rc) rc = dev_alloc(e, &e->h_obs_dev, (size_t)ob * e->n);
  if (!rc) {
    cudaError_t ce = cudaStreamCreateWithFlags(&e->h_stream, cudaStreamNonBlocking);
    if (ce != cudaSuccess) return fail(GR_E_CUDA, "stream: %s", cudaGetErrorString(ce));
  }
  return rc;
}

// ---- delta observation transfer -------------------------------------------
// Between two observations written into the same host buffer (two steps
// apart with BatchEnv's two buffers) ~1.3 % of the words of a symbolic row
// change, in ~20 % of its 64-byte lines.  An attached buffer therefore
// receives only the changed words as (word index, value bits) pairs, and the
// host rewrites only those: the dense path moves 2.17 GB across PCIe into
// every line of the host array per step at 65,536 extended envs.
//
// One warp per row, one pass over HBM: the warp compares the row with its
// shadow 32 words at a time and keeps the ballot masks in shared memory
// (259 words per extended row), reserves the row's slice of the list with
// one atomic, then walks the masks: only the changed words are re-read (from
// L2: the row was just streamed) and written to the list and to the
// shadow.  Row order in the list varies run to run; positions are distinct,
// so the host array after the scatter does not.
constexpr int DL_WARPS = 8;
constexpr int DL_MAXCH = 272;   // >= ceil(8268 / 32)
__global__ void __launch_bounds__(DL_WARPS * 32) k_obs_delta(const uint32_t* __restrict__ obs,
                                                              uint32_t* __restrict__ shadow, int64_t r0, int64_t r1,
                                                              int W, uint2* __restrict__ out, int64_t cap,
                                                              unsigned long long* __restrict__ cursor) {
  __shared__ uint32_t masks[DL_WARPS][DL_MAXCH];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nch = (W + 31) >> 5;
  uint32_t* mk = masks[wid];
  const int64_t nwarps = (int64_t)gridDim.x * DL_WARPS;
  for (int64_t r = r0 + (int64_t)blockIdx.x * DL_WARPS + wid; r < r1; r += nwarps) {
    const uint32_t* row = obs + r * W;
    uint32_t* sh = shadow + r * W;
    int cnt = 0;
#pragma unroll 4
    for (int ch = 0; ch < nch; ++ch) {
      const int c = (ch << 5) + lane;
      const bool d = c < W && __ldcs(row + c) != __ldcs(sh + c);
      const uint32_t m = __ballot_sync(~0u, d);
      if (lane == 0) mk[ch] = m;
      cnt += __popc(m);
    }
    __syncwarp();
    if (!cnt) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(cursor, (unsigned long long)cnt);
    base = __shfl_sync(~0u, base, 0);
    for (int ch = 0; ch < nch; ++ch) {
      const uint32_t m = mk[ch];
      if (!m) continue;
      if ((m >> lane) & 1u) {
        const int c = (ch << 5) + lane;
        const unsigned long long p = base + __popc(m & ((1u << lane) - 1u));
        if (p < (unsigned long long)cap) {   // beyond: left for the next pass, shadow unchanged
          const uint32_t v = row[c];
          out[p] = make_uint2((uint32_t)(r * W + c), v);
          sh[c] = v;
        }
      }
      base += __popc(m);
    }
    __syncwarp();
  }
}

static HostObs* find_host_obs(gr_env* e, const void* p) {
  for (auto& h : e->host_obs)
    if (h.ptr == p) return &h;
  return nullptr;
}

static int64_t host_obs_words(const gr_env* e) { return obs_elems_of(e) * e->n; }

// zero the host buffer and its shadow.  Everything that may still touch the
// shadow (a delivery's k_obs_delta on h_stream) is drained first, and the
// clear is ordered on h_stream and completed before returning, so the next
// delivery never compares against a half-cleared shadow.
static int host_obs_zero(gr_env* e, HostObs& h) {
  CK(cudaStreamSynchronize(e->h_stream));
  memset(h.ptr, 0, (size_t)host_obs_words(e) * 4);
  CK(cudaMemsetAsync(h.shadow, 0, (size_t)host_obs_words(e) * 4, e->h_stream));
  CK(cudaStreamSynchronize(e->h_stream));
  h.dirty = false;
  return GR_OK;
}

int gr_host_obs_attach(gr_env* e, void* obs_host) {
  if (!e) return fail(GR_E_INVALID, "null env");
  if (!obs_host) return fail(GR_E_INVALID, "null host buffer");
  if (e->cfg.obs_mode != GR_OBS_SYMBOLIC) return fail(GR_E_INVALID, "delta transfer needs symbolic observations");
  if (host_obs_words(e) > (int64_t)UINT32_MAX) return fail(GR_E_INVALID, "n_envs x obs width exceeds 2^32 words");
  if (find_host_obs(e, obs_host)) return GR_OK;
  CK(cudaSetDevice(e->cfg.device));
  int rc = ensure_host_scratch(e);   // creates h_stream, which host_obs_zero orders on
  if (rc) return rc;
  HostObs h;
  h.ptr = (uint32_t*)obs_host;
  CK(cudaMalloc((void**)&h.shadow, (size_t)host_obs_words(e) * 4));
  e->host_obs.push_back(h);
  return host_obs_zero(e, e->host_obs.back());
}

int gr_host_obs_detach(gr_env* e, void* obs_host) {
  if (!e) return fail(GR_E_INVALID, "null env");
  for (size_t k = 0; k < e->host_obs.size(); ++k)
    if (e->host_obs[k].ptr == obs_host) {
      cudaDeviceSynchronize();
      if (e->host_obs[k].shadow) cudaFree(e->host_obs[k].shadow);
      e->host_obs.erase(e->host_obs.begin() + (ptrdiff_t)k);
      return GR_OK;
    }
  return fail(GR_E_INVALID, "buffer %p is not attached", obs_host);
}

using hclock = std::chrono::steady_clock;

// host threads of the delta scatter / compact expansion (GR_HOST_THREADS, default: every hardware thread, <= 32)
static int host_threads() {
  if (const char* t = getenv("GR_HOST_THREADS")) {
    const int v = atoi(t);
    if (v > 0) return std::min(v, 64);
  }
  const unsigned hc = std::thread::hardware_concurrency();
  return (int)std::min<unsigned>(hc ? hc : 1, 32);
}
static double ms_since(hclock::time_point t0) {
  return std::chrono::duration<double, std::milli>(hclock::now() - t0).count();
}

static int ensure_delta_list(gr_env* e, int64_t cap) {
  if (e->dl_host && e->dl_cap >= cap) return GR_OK;
  if (e->dl_host) cudaFreeHost(e->dl_host);
  if (e->dl_dev) cudaFree(e->dl_dev);
  e->dl_host = nullptr;
  e->dl_dev = nullptr;
  e->dl_cap = 0;
  CK(cudaMalloc((void**)&e->dl_dev, (size_t)cap * sizeof(uint2)));
  CK(cudaHostAlloc((void**)&e->dl_host, (size_t)cap * sizeof(uint2), cudaHostAllocDefault));
  e->dl_cap = cap;
  return GR_OK;
}

// after the observation is in e->h_obs_dev (ordered on st): list the words
// that differ from the buffer's shadow and scatter them into the host
// buffer, pipelined over DL_CHUNKS row ranges: kernel c (+ its count) on st,
// the copy of chunk c's list on dl_copy once its count is known, and the
// host scatter of chunk c-1 meanwhile.  If a chunk outgrows its share of the
// list, whole-buffer passes with a larger list follow (each pass applies
// what it listed).  Synchronous.
static int host_obs_deliver(gr_env* e, HostObs& h, cudaStream_t st, hclock::time_point t_call) {
  const int W = (int)obs_elems_of(e);
  if (!e->dl_cnt_host) {
    CK(cudaHostAlloc((void**)&e->dl_cnt_host, DL_CHUNKS * sizeof(unsigned long long), cudaHostAllocDefault));
    CK(cudaMalloc((void**)&e->dl_cnt_dev, DL_CHUNKS * sizeof(unsigned long long)));
    CK(cudaStreamCreateWithFlags(&e->dl_copy, cudaStreamNonBlocking));
    for (auto& ev : e->dl_ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    for (auto& ev : e->dl_evd) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->hpool.reset(new HostPool(host_threads()));
  }
  int rc = ensure_delta_list(e, e->n * (int64_t)std::min(W, 256));
  if (rc) return rc;
  h.dirty = true;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned long long* cnt = e->dl_cnt_host;
  const int pf = e->scatter_prefetch;
  auto scatter = [&](const uint2* list, int64_t k) {
    uint32_t* p = h.ptr;
    e->hpool->run(k, [&](int64_t lo, int64_t hi) {
      if (pf > 0) {   // software prefetch pf entries ahead: more misses in flight per thread
        const int64_t mid = std::max(lo, hi - pf);
        for (int64_t i = lo; i < mid; ++i) {
          __builtin_prefetch(p + list[i + pf].x, 1, 0);
          p[list[i].x] = list[i].y;
        }
        for (int64_t i = mid; i < hi; ++i) p[list[i].x] = list[i].y;
      } else {
        for (int64_t i = lo; i < hi; ++i) p[list[i].x] = list[i].y;
      }
    });
    e->host_words += k;
  };
  double t_wait = 0, t_scatter = 0;
  auto wait = [&](cudaEvent_t ev) -> int {
    const auto t0 = hclock::now();
    CK(cudaEventSynchronize(ev));
    t_wait += ms_since(t0);
    return GR_OK;
  };
  // pipelined pass
  const int C = (int)std::min<int64_t>(DL_CHUNKS, std::max<int64_t>(1, e->n / 256));
  const int64_t capc = e->dl_cap / C;
  CK(cudaMemsetAsync(e->dl_cnt_dev, 0, C * sizeof(unsigned long long), st));
  for (int c = 0; c < C; ++c) {
    const int64_t r0 = e->n * c / C, r1 = e->n * (c + 1) / C;
    const int grid = (int)std::min<int64_t>((r1 - r0 + DL_WARPS - 1) / DL_WARPS, (int64_t)sms * 8);
    k_obs_delta<<<grid, DL_WARPS * 32, 0, st>>>((const uint32_t*)e->h_obs_dev, h.shadow, r0, r1, W,
                                                 e->dl_dev + c * capc, capc, e->dl_cnt_dev + c);
    e->launches += 1;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(e->dl_cnt_host + c, e->dl_cnt_dev + c, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       st));
    CK(cudaEventRecord(e->dl_ev[c], st));
  }
  e->host_ms[0] += ms_since(t_call);
  bool overflow = false;
  int64_t total = 0;
  int64_t kc[DL_CHUNKS];
  for (int c = 0; c <= C; ++c) {
    if (c < C) {
      if ((rc = wait(e->dl_ev[c]))) return rc;
      total += (int64_t)cnt[c];
      overflow |= (int64_t)cnt[c] > capc;
      kc[c] = std::min((int64_t)cnt[c], capc);
      CK(cudaStreamWaitEvent(e->dl_copy, e->dl_ev[c], 0));
      if (kc[c])
        CK(cudaMemcpyAsync(e->dl_host + c * capc, e->dl_dev + c * capc, (size_t)kc[c] * sizeof(uint2),
                           cudaMemcpyDeviceToHost, e->dl_copy));
      CK(cudaEventRecord(e->dl_evd[c], e->dl_copy));
    }
    if (c > 0) {
      if ((rc = wait(e->dl_evd[c - 1]))) return rc;
      const auto t0 = hclock::now();
      scatter(e->dl_host + (c - 1) * capc, kc[c - 1]);
      t_scatter += ms_since(t0);
    }
  }
  // overflow: whole-buffer passes until every changed word is listed
  for (int pass = 0; overflow && pass < 64; ++pass) {
    rc = ensure_delta_list(e, std::min<int64_t>(total + total / 4 + 1024, host_obs_words(e)));
    if (rc) return rc;
    CK(cudaMemsetAsync(e->dl_cnt_dev, 0, sizeof(unsigned long long), st));
    k_obs_delta<<<sms * 8, DL_WARPS * 32, 0, st>>>((const uint32_t*)e->h_obs_dev, h.shadow, 0, e->n, W, e->dl_dev,
                                                    e->dl_cap, e->dl_cnt_dev);
    e->launches += 1;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(e->dl_cnt_host, e->dl_cnt_dev, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(e->dl_ev[0], st));
    if ((rc = wait(e->dl_ev[0]))) return rc;
    total = (int64_t)cnt[0];
    const int64_t k = std::min(total, e->dl_cap);
    if (k) CK(cudaMemcpyAsync(e->dl_host, e->dl_dev, (size_t)k * sizeof(uint2), cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(e->dl_ev[0], st));
    if ((rc = wait(e->dl_ev[0]))) return rc;
    const auto t0 = hclock::now();
    scatter(e->dl_host, k);
    t_scatter += ms_since(t0);
    overflow = total > e->dl_cap;
  }
  e->host_ms[1] += t_wait;
  e->host_ms[2] += t_scatter;
  if (overflow) return fail(GR_E_CUDA, "delta transfer did not converge");
  h.dirty = false;
  return GR_OK;
}

// ---- compact observation transfer ------------------------------------------
// The reference hands back a fresh, writable float32 array per step
// (__init__.py:79): 2.17 GB at 65,536 extended envs, which as a plain copy
// is PCIe-bound (~55 GB/s: 40 ms).  A symbolic row is ~95 % zeros, and the
// host writes memory 3x faster than PCIe delivers it (measured on the GPU
// box: 159-188 GB/s with non-temporal stores), so the rows travel packed --
// per row a bitmap of its non-zero words (bitwise: -0.0f counts) and its
// values, ~190 MB -- and host threads expand them into the caller's array
// (AVX-512 masked expand + streaming stores), chunk by chunk so chunk c's
// expansion overlaps chunk c+1's packing and copy.  Every word of the array
// is written each step: the result is the dense copy, bit for bit.
__global__ void __launch_bounds__(DL_WARPS * 32) k_obs_pack(const uint32_t* __restrict__ obs, int64_t r0, int64_t r1,
                                                             int W, int NB, uint32_t* __restrict__ bm,
                                                             uint32_t* __restrict__ vals, int64_t* __restrict__ off,
                                                             unsigned long long* __restrict__ cursor) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * DL_WARPS;
  for (int64_t r = r0 + (int64_t)blockIdx.x * DL_WARPS + wid; r < r1; r += nwarps) {
    const uint32_t* row = obs + r * W;
    uint32_t* b = bm + r * NB;
    int cnt = 0;
    for (int ch = 0; ch < NB; ++ch) {
      const int c = (ch << 5) + lane;
      const uint32_t m = __ballot_sync(~0u, c < W && __ldcg(row + c) != 0u);
      if (lane == 0) b[ch] = m;
      cnt += __popc(m);
    }
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(cursor, (unsigned long long)cnt);
    base = __shfl_sync(~0u, base, 0);
    if (lane == 0) off[r] = (int64_t)base;
    __syncwarp();
    for (int ch = 0; ch < NB; ++ch) {
      const uint32_t m = b[ch];   // this warp's own store, visible after __syncwarp
      if (!m) continue;
      if ((m >> lane) & 1u) vals[base + __popc(m & ((1u << lane) - 1u))] = row[(ch << 5) + lane];
      base += __popc(m);
    }
  }
}

// expand rows [r0, r1) of a chunk into the host array
__attribute__((target("avx512f,avx512bw"))) static void cp_expand_avx512(float* out, int W, int NB, const uint32_t* bm,
                                                                           const float* vals, const int64_t* off,
                                                                           int64_t r0, int64_t r1) {
  for (int64_t r = r0; r < r1; ++r) {
    float* dst = out + r * W;
    const uint32_t* b = bm + r * NB;
    const float* v = vals + off[r];
    auto bits16 = [&](int k) -> uint32_t {   // bitmap bits k .. k+15
      const int w = k >> 5, s = k & 31;
      uint64_t x = b[w];
      if (w + 1 < NB) x |= (uint64_t)b[w + 1] << 32;
      return (uint32_t)(x >> s) & 0xFFFFu;
    };
    // scalar head up to the first 64-byte aligned word, streaming stores of
    // 16 words, scalar tail
    int k = (int)(((64 - ((uintptr_t)dst & 63)) & 63) >> 2);
    if (k > W) k = W;
    for (int q = 0; q < k; ++q) dst[q] = (b[q >> 5] >> (q & 31)) & 1u ? *v++ : 0.0f;
    for (; k + 16 <= W; k += 16) {
      const uint32_t m = bits16(k);
      _mm512_stream_ps(dst + k, _mm512_maskz_expandloadu_ps((__mmask16)m, v));
      v += __builtin_popcount(m);
    }
    for (int q = k; q < W; ++q) dst[q] = (b[q >> 5] >> (q & 31)) & 1u ? *v++ : 0.0f;
  }
  _mm_sfence();
}

static void cp_expand_scalar(float* out, int W, int NB, const uint32_t* bm, const float* vals, const int64_t* off,
                             int64_t r0, int64_t r1) {
  for (int64_t r = r0; r < r1; ++r) {
    uint32_t* dst = reinterpret_cast<uint32_t*>(out + r * W);
    const uint32_t* b = bm + r * NB;
    const uint32_t* v = reinterpret_cast<const uint32_t*>(vals + off[r]);
    for (int q = 0; q < W; ++q) dst[q] = (b[q >> 5] >> (q & 31)) & 1u ? *v++ : 0u;
  }
}

static int host_obs_compact(gr_env* e, const uint32_t* src, float* out, cudaStream_t st, hclock::time_point t_call) {
  const int W = (int)obs_elems_of(e), NB = (W + 31) / 32;
  if (!e->dl_cnt_host) {
    CK(cudaHostAlloc((void**)&e->dl_cnt_host, DL_CHUNKS * sizeof(unsigned long long), cudaHostAllocDefault));
    CK(cudaMalloc((void**)&e->dl_cnt_dev, DL_CHUNKS * sizeof(unsigned long long)));
    CK(cudaStreamCreateWithFlags(&e->dl_copy, cudaStreamNonBlocking));
    for (auto& ev : e->dl_ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    for (auto& ev : e->dl_evd) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->hpool.reset(new HostPool(host_threads()));
  }
  if (!e->cp_bm_dev) {
    CK(cudaMalloc((void**)&e->cp_bm_dev, (size_t)e->n * NB * 4));
    CK(cudaMalloc((void**)&e->cp_val_dev, (size_t)e->n * W * 4));
    CK(cudaMalloc((void**)&e->cp_off_dev, (size_t)e->n * 8));
    CK(cudaHostAlloc((void**)&e->cp_bm_host, (size_t)e->n * NB * 4, cudaHostAllocDefault));
    CK(cudaHostAlloc((void**)&e->cp_off_host, (size_t)e->n * 8, cudaHostAllocDefault));
    e->cp_val_cap = e->n * (int64_t)std::min(W, 640);   // symbolic rows hold <= ~450 non-zeros
    CK(cudaHostAlloc((void**)&e->cp_val_host, (size_t)e->cp_val_cap * 4, cudaHostAllocDefault));
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static const bool avx512 = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw");
  const int C = (int)std::min<int64_t>(DL_CHUNKS, std::max<int64_t>(1, e->n / 256));
  double t_wait = 0, t_dec = 0;
  auto wait = [&](cudaEvent_t ev) -> int {
    const auto t0 = hclock::now();
    CK(cudaEventSynchronize(ev));
    t_wait += ms_since(t0);
    return GR_OK;
  };
  CK(cudaMemsetAsync(e->dl_cnt_dev, 0, C * sizeof(unsigned long long), st));
  for (int c = 0; c < C; ++c) {
    const int64_t r0 = e->n * c / C, r1 = e->n * (c + 1) / C;
    const int grid = (int)std::min<int64_t>((r1 - r0 + DL_WARPS - 1) / DL_WARPS, (int64_t)sms * 8);
    k_obs_pack<<<grid, DL_WARPS * 32, 0, st>>>(src, r0, r1, W, NB, e->cp_bm_dev,
                                                e->cp_val_dev + r0 * W, e->cp_off_dev, e->dl_cnt_dev + c);
    e->launches += 1;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(e->dl_cnt_host + c, e->dl_cnt_dev + c, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(e->dl_ev[c], st));
  }
  e->host_ms[0] += ms_since(t_call);
  int rc;
  int64_t vofs[DL_CHUNKS + 1];
  bool dense[DL_CHUNKS];
  vofs[0] = 0;
  for (int c = 0; c <= C; ++c) {
    if (c < C) {
      const int64_t r0 = e->n * c / C, r1 = e->n * (c + 1) / C;
      if ((rc = wait(e->dl_ev[c]))) return rc;
      const int64_t k = (int64_t)e->dl_cnt_host[c];
      dense[c] = vofs[c] + k > e->cp_val_cap;   // stage full: this chunk goes as a plain copy
      vofs[c + 1] = dense[c] ? vofs[c] : vofs[c] + k;
      CK(cudaStreamWaitEvent(e->dl_copy, e->dl_ev[c], 0));
      if (dense[c]) {
        CK(cudaMemcpyAsync(out + r0 * W, (const float*)src + r0 * W, (size_t)(r1 - r0) * W * 4,
                           cudaMemcpyDeviceToHost, e->dl_copy));
      } else {
        CK(cudaMemcpyAsync(e->cp_bm_host + r0 * NB, e->cp_bm_dev + r0 * NB, (size_t)(r1 - r0) * NB * 4,
                           cudaMemcpyDeviceToHost, e->dl_copy));
        CK(cudaMemcpyAsync(e->cp_off_host + r0, e->cp_off_dev + r0, (size_t)(r1 - r0) * 8, cudaMemcpyDeviceToHost,
                           e->dl_copy));
        if (k)
          CK(cudaMemcpyAsync(e->cp_val_host + vofs[c], e->cp_val_dev + r0 * W, (size_t)k * 4, cudaMemcpyDeviceToHost,
                             e->dl_copy));
      }
      CK(cudaEventRecord(e->dl_evd[c], e->dl_copy));
    }
    if (c > 0) {
      const int cc = c - 1;
      const int64_t r0 = e->n * cc / C, r1 = e->n * (cc + 1) / C;
      if ((rc = wait(e->dl_evd[cc]))) return rc;
      if (!dense[cc]) {
        const auto t0 = hclock::now();
        const float* vals = reinterpret_cast<const float*>(e->cp_val_host + vofs[cc]);
        e->hpool->run(r1 - r0, [&](int64_t lo, int64_t hi) {
          if (avx512) cp_expand_avx512(out, W, NB, e->cp_bm_host, vals, e->cp_off_host, r0 + lo, r0 + hi);
          else cp_expand_scalar(out, W, NB, e->cp_bm_host, vals, e->cp_off_host, r0 + lo, r0 + hi);
        }, 32);   // rows: a few dozen are worth the pool
        t_dec += ms_since(t0);
        e->host_words += vofs[cc + 1] - vofs[cc];
      }
    }
  }
  e->host_ms[1] += t_wait;
  e->host_ms[2] += t_dec;
  return GR_OK;
}

static int host_obs_pixrows(gr_env* e, const uint8_t* src, uint8_t* out, cudaStream_t st, hclock::time_point t_call);

int gr_reset_host(gr_env* e, void* obs_host) {
  if (!e) return fail(GR_E_INVALID, "null env");
  CK(cudaSetDevice(e->cfg.device));
  int rc = ensure_host_scratch(e);
  if (rc) return rc;
  HostObs* hz = obs_host ? find_host_obs(e, obs_host) : nullptr;
  if (hz && hz->dirty && (rc = host_obs_zero(e, *hz))) return rc;
  const auto t_call = hclock::now();
  rc = gr_reset(e, obs_host ? e->h_obs_dev : nullptr, e->h_stream);
  if (rc) return rc;
  const int64_t ob = obs_elems_of(e) * (e->cfg.obs_mode == GR_OBS_PIXELS ? 1 : 4);
  if (HostObs* ho = obs_host ? find_host_obs(e, obs_host) : nullptr)
    return host_obs_deliver(e, *ho, e->h_stream, t_call);
  if (obs_host && ob && e->compact && e->cfg.obs_mode == GR_OBS_SYMBOLIC) {
    rc = host_obs_compact(e, (const uint32_t*)e->h_obs_dev, (float*)obs_host, e->h_stream, t_call);
    if (rc) return rc;
  } else if (obs_host && ob && e->compact && e->cfg.obs_mode == GR_OBS_PIXELS) {
    rc = host_obs_pixrows(e, (const uint8_t*)e->h_obs_dev, (uint8_t*)obs_host, e->h_stream, t_call);
    if (rc) return rc;
  } else if (obs_host && ob) {
    CK(cudaMemcpyAsync(obs_host, e->h_obs_dev, (size_t)ob * e->n, cudaMemcpyDeviceToHost, e->h_stream));
  }
  CK(cudaStreamSynchronize(e->h_stream));
  return GR_OK;
}

int gr_step_host(gr_env* e, const int64_t* actions_host, void* obs_host, float* reward_host, uint8_t* done_host,
                 uint8_t* newly_host, uint32_t* time_host, uint8_t* floor_host) {
  if (!e) return fail(GR_E_INVALID, "null env");
  if (!e->have_reset) return fail(GR_E_STATE, "call reset() before step()");
  if (!actions_host) return fail(GR_E_INVALID, "actions are required");
  CK(cudaSetDevice(e->cfg.device));
  // validation on the host copy: nothing is mutated on a bad action
  for (int64_t i = 0; i < e->n; ++i)
    if (actions_host[i] < 0 || actions_host[i] >= e->d.NA) {
      e->last_bad_env = i;
      e->last_bad_action = actions_host[i];
      return fail(GR_E_BAD_ACTION, "invalid action %lld for env %lld", (long long)actions_host[i], (long long)i);
    }
  int rc = ensure_host_scratch(e);
  if (rc) return rc;
  cudaStream_t st = e->h_stream;
  HostObs* hz = obs_host ? find_host_obs(e, obs_host) : nullptr;
  if (hz && hz->dirty && (rc = host_obs_zero(e, *hz))) return rc;
  const auto t_call = hclock::now();
  CK(cudaMemcpyAsync(e->h_act_dev, actions_host, e->n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  const bool v = e->validate;
  e->validate = false;
  rc = gr_step(e, e->h_act_dev, obs_host ? e->h_obs_dev : nullptr, e->h_rew_dev, e->h_done_dev,
               newly_host ? e->h_newly_dev : nullptr, time_host ? e->h_time_dev : nullptr,
               floor_host ? e->h_floor_dev : nullptr, st);
  e->validate = v;
  if (rc) return rc;
  const int64_t ob = obs_elems_of(e) * (e->cfg.obs_mode == GR_OBS_PIXELS ? 1 : 4);
  // the small outputs first: they cross PCIe while the obs is delivered
  if (reward_host) CK(cudaMemcpyAsync(reward_host, e->h_rew_dev, e->n * sizeof(float), cudaMemcpyDeviceToHost, st));
  if (done_host) CK(cudaMemcpyAsync(done_host, e->h_done_dev, e->n, cudaMemcpyDeviceToHost, st));
  if (newly_host) CK(cudaMemcpyAsync(newly_host, e->h_newly_dev, e->n * e->d.A, cudaMemcpyDeviceToHost, st));
  if (time_host) CK(cudaMemcpyAsync(time_host, e->h_time_dev, e->n * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  if (floor_host) CK(cudaMemcpyAsync(floor_host, e->h_floor_dev, e->n, cudaMemcpyDeviceToHost, st));
  if (HostObs* ho = obs_host ? find_host_obs(e, obs_host) : nullptr) {
    rc = host_obs_deliver(e, *ho, st, t_call);
    if (rc) return rc;
  } else if (obs_host && ob && e->compact && e->cfg.obs_mode == GR_OBS_SYMBOLIC) {
    rc = host_obs_compact(e, (const uint32_t*)e->h_obs_dev, (float*)obs_host, st, t_call);
    if (rc) return rc;
  } else if (obs_host && ob && e->compact && e->cfg.obs_mode == GR_OBS_PIXELS) {
    rc = host_obs_pixrows(e, (const uint8_t*)e->h_obs_dev, (uint8_t*)obs_host, st, t_call);
    if (rc) return rc;
  } else {
    if (obs_host && ob) CK(cudaMemcpyAsync(obs_host, e->h_obs_dev, (size_t)ob * e->n, cudaMemcpyDeviceToHost, st));
    e->host_ms[0] += ms_since(t_call);
  }
  const auto t_tail = hclock::now();
  CK(cudaStreamSynchronize(st));
  e->host_ms[3] += ms_since(t_tail);
  e->host_calls += 1;
  return GR_OK;
}

// pixel frames into a plain host array: per row chunk, gather each frame's
// class rows on the device (~28 % of the frame bytes), copy them, and let
// host threads replicate them into the frames while the next chunk moves.
// frames [r0 + lo, r0 + hi) from their class rows: the frame written front to
// back in 64-byte streaming stores, each a 64-byte load from its row's class
// row (or two, blended, across a frame-row boundary); bytes before the first
// 64-byte aligned address and after the last one go by byte
__attribute__((target("avx512f,avx512bw"))) static void pix_expand_avx512(uint8_t* out, const PixRowMap& m,
                                                                            const uint8_t* stage, size_t per_env,
                                                                            int64_t r0, int64_t lo, int64_t hi) {
  const int RB = m.RB, FB = m.FB;
  for (int64_t r = lo; r < hi; ++r) {
    uint8_t* f = out + (r0 + r) * (int64_t)FB;
    const uint8_t* rows = stage + r * per_env;
    auto byte_at = [&](int b) -> uint8_t {
      const int y = b / RB;
      return rows[(size_t)m.slot_of_row[y] * RB + (b - y * RB)];
    };
    int b = (int)((64 - ((uintptr_t)f & 63)) & 63);
    if (b > FB) b = FB;
    for (int q = 0; q < b; ++q) f[q] = byte_at(q);
    int y = b / RB, o = b - y * RB;
    for (; b + 64 <= FB; b += 64) {
      const uint8_t* ra = rows + (size_t)m.slot_of_row[y] * RB + o;
      __m512i v = _mm512_loadu_si512(ra);
      const int n = RB - o;   // bytes of this block still in row y
      if (n < 64) {
        const uint8_t* rb = rows + (size_t)m.slot_of_row[y + 1] * RB - n;
        v = _mm512_mask_blend_epi8((__mmask64)(~0ull << n), v, _mm512_loadu_si512(rb));
      }
      _mm512_stream_si512((__m512i*)(f + b), v);
      o += 64;
      while (o >= RB) { o -= RB; ++y; }
    }
    for (int q = b; q < FB; ++q) f[q] = byte_at(q);
  }
  _mm_sfence();
}

static int host_obs_pixrows(gr_env* e, const uint8_t* src, uint8_t* out, cudaStream_t st, hclock::time_point t_call) {
  static const bool avx512 = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw");
  if (!e->dl_cnt_host) {
    CK(cudaHostAlloc((void**)&e->dl_cnt_host, DL_CHUNKS * sizeof(unsigned long long), cudaHostAllocDefault));
    CK(cudaMalloc((void**)&e->dl_cnt_dev, DL_CHUNKS * sizeof(unsigned long long)));
    CK(cudaStreamCreateWithFlags(&e->dl_copy, cudaStreamNonBlocking));
    for (auto& ev : e->dl_ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    for (auto& ev : e->dl_evd) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->hpool.reset(new HostPool(host_threads()));
  }
  const int C = (int)std::min<int64_t>(DL_CHUNKS, std::max<int64_t>(1, e->n / 256));
  const PixRowMap& m = e->prmap;
  const size_t per_env = (size_t)m.nused * m.RB;
  if (!e->pr_dev) {
    if (pixel_row_map(e->ext, e->cfg.tile_px, &e->prmap)) return fail(GR_E_INVALID, "no row map for this tile size");
    const size_t pe = (size_t)e->prmap.nused * e->prmap.RB;
    CK(cudaMalloc((void**)&e->pr_dev, pe * e->n));
    const int64_t rows_max = (e->n + C - 1) / C;
    // 64 bytes of slack at both ends: the expansion's 64-byte loads may run past a chunk's rows
    for (auto& p : e->pr_stage) CK(cudaHostAlloc((void**)&p, pe * rows_max + 128, cudaHostAllocDefault));
    return host_obs_pixrows(e, src, out, st, t_call);
  }
  double t_wait = 0, t_dec = 0;
  for (int c = 0; c < C; ++c) {
    const int64_t r0 = e->n * c / C, r1 = e->n * (c + 1) / C;
    launch_pix_gather(src, r0, r1, m, e->pr_dev + r0 * per_env, st);
    e->launches += 1;
    CK(cudaGetLastError());
    CK(cudaEventRecord(e->dl_ev[c], st));
  }
  e->host_ms[0] += ms_since(t_call);
  for (int c = 0; c <= C; ++c) {
    if (c < C) {   // chunk c's rows into stage c % 2 (chunk c - 2 was expanded last iteration)
      const int64_t r0 = e->n * c / C, r1 = e->n * (c + 1) / C;
      CK(cudaStreamWaitEvent(e->dl_copy, e->dl_ev[c], 0));
      CK(cudaMemcpyAsync(e->pr_stage[c & 1] + 64, e->pr_dev + r0 * per_env, (size_t)(r1 - r0) * per_env,
                         cudaMemcpyDeviceToHost, e->dl_copy));
      CK(cudaEventRecord(e->dl_evd[c], e->dl_copy));
    }
    if (c > 0) {
      const int cc = c - 1;
      const int64_t r0 = e->n * cc / C, r1 = e->n * (cc + 1) / C;
      auto t0 = hclock::now();
      CK(cudaEventSynchronize(e->dl_evd[cc]));
      t_wait += ms_since(t0);
      t0 = hclock::now();
      const uint8_t* stage = e->pr_stage[cc & 1] + 64;
      e->hpool->run(r1 - r0, [&](int64_t lo, int64_t hi) {
        if (avx512) {
          pix_expand_avx512(out, m, stage, per_env, r0, lo, hi);
          return;
        }
        for (int64_t r = lo; r < hi; ++r) {
          uint8_t* f = out + (r0 + r) * (int64_t)m.FB;
          const uint8_t* rows = stage + r * per_env;
          for (int y = 0; y < m.FH; ++y) memcpy(f + (size_t)y * m.RB, rows + (size_t)m.slot_of_row[y] * m.RB, m.RB);
        }
      }, 32);
      t_dec += ms_since(t0);
      e->host_words += (r1 - r0) * (int64_t)per_env / 4;
    }
  }
  e->host_ms[1] += t_wait;
  e->host_ms[2] += t_dec;
  return GR_OK;
}

int gr_obs_to_host(gr_env* e, const void* obs_dev, void* obs_host, void* stream) {
  if (!e || !obs_dev || !obs_host) return fail(GR_E_INVALID, "null argument");
  CK(cudaSetDevice(e->cfg.device));
  int rc = ensure_host_scratch(e);
  if (rc) return rc;
  // ordered after the caller's work on `stream` (e.g. the step that wrote obs_dev)
  CK(cudaEventRecord(e->ev_fork, (cudaStream_t)stream));
  CK(cudaStreamWaitEvent(e->h_stream, e->ev_fork, 0));
  const auto t_call = hclock::now();
  const int64_t ob = obs_elems_of(e) * (e->cfg.obs_mode == GR_OBS_PIXELS ? 1 : 4);
  if (e->compact && e->cfg.obs_mode == GR_OBS_SYMBOLIC) {
    rc = host_obs_compact(e, (const uint32_t*)obs_dev, (float*)obs_host, e->h_stream, t_call);
    if (rc) return rc;
  } else if (e->compact && e->cfg.obs_mode == GR_OBS_PIXELS) {
    rc = host_obs_pixrows(e, (const uint8_t*)obs_dev, (uint8_t*)obs_host, e->h_stream, t_call);
    if (rc) return rc;
  } else if (ob) {
    CK(cudaMemcpyAsync(obs_host, obs_dev, (size_t)ob * e->n, cudaMemcpyDeviceToHost, e->h_stream));
    e->host_ms[0] += ms_since(t_call);
  }
  const auto t_tail = hclock::now();
  CK(cudaStreamSynchronize(e->h_stream));
  e->host_ms[3] += ms_since(t_tail);
  e->host_calls += 1;
  return GR_OK;
}

int gr_host_phase_times(gr_env* e, double out[4], int64_t* calls, int64_t* words) {
  if (!e || !out) return fail(GR_E_INVALID, "null argument");
  for (int k = 0; k < 4; ++k) {
    out[k] = e->host_ms[k];
    e->host_ms[k] = 0;
  }
  if (calls) *calls = e->host_calls;
  if (words) *words = e->host_words;
  e->host_calls = 0;
  e->host_words = 0;
  return GR_OK;
}

static int materialize(gr_env* e) {
  {
    PTimer t(e, PK_OTHER, 0);
    k_materialize<<<(unsigned)e->nb, 128>>>(e->S, e->n, e->d.F, e->prev_flags);
  }
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return GR_OK;
}

int gr_export_field(gr_env* e, int32_t field, void* host_dst) {
  if (!e || !host_dst) return fail(GR_E_INVALID, "null argument");
  if (field < 0 || field >= GR_NFIELDS) return fail(GR_E_INVALID, "unknown field id %d", field);
  CK(cudaSetDevice(e->cfg.device));
  int rc = materialize(e);
  if (rc) return rc;
  const FieldDesc& fd = FIELD_TABLE[field];
  const int64_t comps = device_comps(field, e->d);
  const size_t bytes = (size_t)comps * e->n * fd.esz;
  if (fd.kind == K_MAP) {
    CK(cudaMemcpy(host_dst, e->S.f[field], bytes, cudaMemcpyDeviceToHost));
    return GR_OK;
  }
  std::vector<uint8_t> tmp(bytes);
  CK(cudaMemcpy(tmp.data(), e->S.f[field], bytes, cudaMemcpyDeviceToHost));
  uint8_t* dst = (uint8_t*)host_dst;
  if (fd.kind == K_ACH) {
    const uint32_t* w = (const uint32_t*)tmp.data();
    for (int64_t i = 0; i < e->n; ++i)
      for (int a = 0; a < e->d.A; ++a) dst[i * e->d.A + a] = (w[(size_t)(a >> 5) * e->n + i] >> (a & 31)) & 1u;
    return GR_OK;
  }
  const int es = fd.esz;
  for (int64_t c = 0; c < comps; ++c)
    for (int64_t i = 0; i < e->n; ++i)
      memcpy(dst + ((size_t)i * comps + c) * es, tmp.data() + ((size_t)c * e->n + i) * es, es);
  return GR_OK;
}

int gr_import_field(gr_env* e, int32_t field, const void* host_src) {
  if (!e || !host_src) return fail(GR_E_INVALID, "null argument");
  if (field < 0 || field >= GR_NFIELDS) return fail(GR_E_INVALID, "unknown field id %d", field);
  CK(cudaSetDevice(e->cfg.device));
  int rc = materialize(e);
  if (rc) return rc;
  const FieldDesc& fd = FIELD_TABLE[field];
  const int64_t comps = device_comps(field, e->d);
  const size_t bytes = (size_t)comps * e->n * fd.esz;
  e->have_reset = true;
  // an imported map may hold torches anywhere: disable the no-torch shortcut
  CK(cudaMemset(e->S.torch_bits, 0xFF, e->n * sizeof(uint16_t)));
  if (fd.kind == K_MAP) {
    CK(cudaMemcpy(e->S.f[field], host_src, bytes, cudaMemcpyHostToDevice));
    return GR_OK;
  }
  std::vector<uint8_t> tmp(bytes);
  const uint8_t* src = (const uint8_t*)host_src;
  if (fd.kind == K_ACH) {
    uint32_t* w = (uint32_t*)tmp.data();
    memset(w, 0, bytes);
    for (int64_t i = 0; i < e->n; ++i)
      for (int a = 0; a < e->d.A; ++a)
        if (src[i * e->d.A + a]) w[(size_t)(a >> 5) * e->n + i] |= 1u << (a & 31);
  } else {
    const int es = fd.esz;
    for (int64_t c = 0; c < comps; ++c)
      for (int64_t i = 0; i < e->n; ++i)
        memcpy(tmp.data() + ((size_t)c * e->n + i) * es, src + ((size_t)i * comps + c) * es, es);
  }
  CK(cudaMemcpy(e->S.f[field], tmp.data(), bytes, cudaMemcpyHostToDevice));
  return GR_OK;
}

int gr_observe(gr_env* e, void* obs_dev, void* stream) {
  if (!e) return fail(GR_E_INVALID, "null env");
  CK(cudaSetDevice(e->cfg.device));
  {
    PTimer t(e, PK_OTHER, (cudaStream_t)stream);
    launch_make_desc(e->ext, e->S, e->n, (cudaStream_t)stream);
  }
  return observe(e, obs_dev, (cudaStream_t)stream, true);
}

int gr_stats_get(gr_env* e, gr_stats* out) {
  if (!e || !out) return fail(GR_E_INVALID, "null argument");
  CK(cudaSetDevice(e->cfg.device));
  CK(cudaDeviceSynchronize());
  unsigned long long ep = 0, steps = 0, ach[67] = {0};
  double ret = 0;
  CK(cudaMemcpy(&ep, e->st_episodes, sizeof(ep), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&steps, e->st_steps, sizeof(steps), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&ret, e->st_return, sizeof(ret), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ach, e->st_ach, sizeof(ach), cudaMemcpyDeviceToHost));
  memset(out, 0, sizeof(*out));
  out->episodes = (int64_t)ep;
  out->total_steps = (int64_t)steps;
  out->total_return = ret;
  for (int a = 0; a < 67; ++a) out->ach_episodes[a] = (int64_t)ach[a];
  return GR_OK;
}

int gr_stats_set(gr_env* e, const gr_stats* in) {
  if (!e || !in) return fail(GR_E_INVALID, "null argument");
  if (in->episodes < 0 || in->total_steps < 0) return fail(GR_E_INVALID, "negative episode statistics");
  CK(cudaSetDevice(e->cfg.device));
  CK(cudaDeviceSynchronize());
  const unsigned long long ep = (unsigned long long)in->episodes, steps = (unsigned long long)in->total_steps;
  unsigned long long ach[67];
  for (int a = 0; a < 67; ++a) ach[a] = (unsigned long long)in->ach_episodes[a];
  CK(cudaMemcpy(e->st_episodes, &ep, sizeof(ep), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(e->st_steps, &steps, sizeof(steps), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(e->st_return, &in->total_return, sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(e->st_ach, ach, sizeof(ach), cudaMemcpyHostToDevice));
  return GR_OK;
}

int gr_export_episode(gr_env* e, double* ep_return_host, int64_t* ep_length_host) {
  if (!e) return fail(GR_E_INVALID, "null env");
  CK(cudaSetDevice(e->cfg.device));
  CK(cudaDeviceSynchronize());
  if (ep_return_host) CK(cudaMemcpy(ep_return_host, e->S.ep_return, e->n * sizeof(double), cudaMemcpyDeviceToHost));
  if (ep_length_host) {
    std::vector<int32_t> tmp(e->n);
    CK(cudaMemcpy(tmp.data(), e->S.ep_length, e->n * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < e->n; ++i) ep_length_host[i] = tmp[i];
  }
  return GR_OK;
}

int gr_import_episode(gr_env* e, const double* ep_return_host, const int64_t* ep_length_host) {
  if (!e) return fail(GR_E_INVALID, "null env");
  CK(cudaSetDevice(e->cfg.device));
  CK(cudaDeviceSynchronize());
  if (ep_return_host) CK(cudaMemcpy(e->S.ep_return, ep_return_host, e->n * sizeof(double), cudaMemcpyHostToDevice));
  if (ep_length_host) {
    std::vector<int32_t> tmp(e->n);
    for (int64_t i = 0; i < e->n; ++i) {
      if (ep_length_host[i] < 0 || ep_length_host[i] > INT32_MAX)
        return fail(GR_E_INVALID, "ep_length[%lld] out of range", (long long)i);
      tmp[i] = (int32_t)ep_length_host[i];
    }
    CK(cudaMemcpy(e->S.ep_length, tmp.data(), e->n * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  return GR_OK;
}

int gr_get_step_index(gr_env* e, int64_t* out) {
  if (!e || !out) return fail(GR_E_INVALID, "null argument");
  *out = e->step_index;
  return GR_OK;
}

int gr_set_step_index(gr_env* e, int64_t step_index) {
  if (!e || step_index < 0) return fail(GR_E_INVALID, "bad step index");
  CK(cudaSetDevice(e->cfg.device));
  CK(cudaDeviceSynchronize());
  const unsigned long long v = (unsigned long long)step_index;
  CK(cudaMemcpy(e->dstep, &v, sizeof(v), cudaMemcpyHostToDevice));
  e->step_index = step_index;
  return GR_OK;
}

void gr_levels_destroy(gr_levels* lv) {
  if (!lv) return;
  cudaSetDevice(lv->e->cfg.device);
  cudaDeviceSynchronize();
  for (void* q : lv->allocs) cudaFree(q);
  delete lv;
}

int gr_levels_create(gr_env* e, int64_t capacity, gr_levels** out) {
  if (!e || !out || capacity <= 0) return fail(GR_E_INVALID, "bad level buffer arguments");
  CK(cudaSetDevice(e->cfg.device));
  gr_levels* lv = new gr_levels();
  lv->e = e;
  lv->cap = capacity;
  const size_t mb = (size_t)capacity * e->d.F * e->d.H * e->d.W;
  auto al = [&](void** q, size_t bytes) -> bool {
    if (cudaMalloc(q, bytes) != cudaSuccess) return false;
    lv->allocs.push_back(*q);
    return cudaMemset(*q, 0, bytes) == cudaSuccess;
  };
  const bool ok = al((void**)&lv->w.blocks, mb) && al((void**)&lv->w.items, mb) &&
                  al((void**)&lv->w.meta, capacity * sizeof(WMeta)) &&
                  al((void**)&lv->p.seed, capacity * sizeof(uint64_t)) &&
                  al((void**)&lv->p.angles, capacity * 252 * sizeof(float)) &&
                  al((void**)&lv->p.floor_seed, capacity * 9 * sizeof(uint64_t));
  lv->w.cap = capacity;
  if (!ok) {
    gr_levels_destroy(lv);
    return fail(GR_E_OOM, "level buffer of %lld levels: out of device memory", (long long)capacity);
  }
  *out = lv;
  return GR_OK;
}

static int lv_range(gr_levels* lv, int64_t first, int64_t count) {
  if (!lv) return fail(GR_E_INVALID, "null level buffer");
  if (first < 0 || count < 0 || first + count > lv->cap)
    return fail(GR_E_INVALID, "levels [%lld, %lld) outside the buffer of %lld", (long long)first,
                (long long)(first + count), (long long)lv->cap);
  return GR_OK;
}

int gr_levels_set_params(gr_levels* lv, int64_t first, int64_t count, const uint64_t* seeds, const float* angles,
                         const uint64_t* floor_seeds) {
  int rc = lv_range(lv, first, count);
  if (rc) return rc;
  if (!seeds || (!angles) != (!floor_seeds)) return fail(GR_E_INVALID, "seeds required; angles and floor seeds together");
  CK(cudaSetDevice(lv->e->cfg.device));
  CK(cudaMemcpy(lv->p.seed + first, seeds, count * sizeof(uint64_t), cudaMemcpyHostToDevice));
  if (angles) {
    CK(cudaMemcpy(lv->p.angles + first * 252, angles, count * 252 * sizeof(float), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(lv->p.floor_seed + first * 9, floor_seeds, count * 9 * sizeof(uint64_t), cudaMemcpyHostToDevice));
  } else {
    launch_level_params(lv->p, first, count, 0);
    CK(cudaGetLastError());
  }
  CK(cudaDeviceSynchronize());
  return GR_OK;
}

int gr_levels_get_params(gr_levels* lv, int64_t first, int64_t count, uint64_t* seeds, float* angles,
                         uint64_t* floor_seeds) {
  int rc = lv_range(lv, first, count);
  if (rc) return rc;
  CK(cudaSetDevice(lv->e->cfg.device));
  CK(cudaDeviceSynchronize());
  if (seeds) CK(cudaMemcpy(seeds, lv->p.seed + first, count * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  if (angles) CK(cudaMemcpy(angles, lv->p.angles + first * 252, count * 252 * sizeof(float), cudaMemcpyDeviceToHost));
  if (floor_seeds)
    CK(cudaMemcpy(floor_seeds, lv->p.floor_seed + first * 9, count * 9 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return GR_OK;
}

int gr_levels_generate(gr_levels* lv, int64_t first, int64_t count) {
  int rc = lv_range(lv, first, count);
  if (rc) return rc;
  if (!count) return GR_OK;
  gr_env* e = lv->e;
  CK(cudaSetDevice(e->cfg.device));
  CK(cudaMemset(lv->w.meta + first, 0, count * sizeof(WMeta)));
  WorldJob j{};
  j.mode = 2;
  j.count = count;
  j.first = first;
  j.out = lv->w;
  j.params = lv->p;
  j.counters = e->counters;
  j.max_attempts = e->wg_attempts;
  launch_worldgen(e->ext, j, 0);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return GR_OK;
}

int gr_levels_mutate(gr_levels* lv, int32_t op, int64_t count, const int64_t* level_idx, const uint64_t* stream_key,
                     const uint64_t* stream_counter, double scale) {
  if (!lv || count < 0 || (count && (!level_idx || !stream_key || !stream_counter)))
    return fail(GR_E_INVALID, "bad mutation arguments");
  if (op != GR_MUT_NOISE && op != GR_MUT_SWAP && op != GR_MUT_RSWAP) return fail(GR_E_INVALID, "unknown mutation %d", op);
  for (int64_t k = 0; k < count; ++k)
    if (level_idx[k] < 0 || level_idx[k] >= lv->cap) return fail(GR_E_INVALID, "level %lld out of range", (long long)level_idx[k]);
  if (!count) return GR_OK;
  CK(cudaSetDevice(lv->e->cfg.device));
  DevArrays d;
  const int64_t* di = d.put(level_idx, count);
  const uint64_t* dk = d.put(stream_key, count);
  const uint64_t* dc = d.put(stream_counter, count);
  if (!di || !dk || !dc) return fail(GR_E_OOM, "mutation scratch");
  launch_mutate(lv->e->ext, op, lv->p, lv->w, di, dk, dc, count, scale, 0);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return GR_OK;
}

int gr_levels_install(gr_levels* lv, int64_t count, const int64_t* env_idx, const int64_t* level_idx,
                      const uint64_t* keys) {
  if (!lv || count < 0 || (count && (!env_idx || !level_idx || !keys))) return fail(GR_E_INVALID, "bad install arguments");
  gr_env* e = lv->e;
  for (int64_t k = 0; k < count; ++k) {
    if (env_idx[k] < 0 || env_idx[k] >= e->n) return fail(GR_E_INVALID, "env %lld out of range", (long long)env_idx[k]);
    if (level_idx[k] < 0 || level_idx[k] >= lv->cap)
      return fail(GR_E_INVALID, "level %lld out of range", (long long)level_idx[k]);
  }
  if (!count) return GR_OK;
  CK(cudaSetDevice(e->cfg.device));
  int rc = materialize(e);   // deferred cooldowns of the envs being replaced
  if (rc) return rc;
  DevArrays d;
  const int64_t* de = d.put(env_idx, count);
  const int64_t* dl = d.put(level_idx, count);
  const uint64_t* dk = d.put(keys, count);
  if (!de || !dl || !dk) return fail(GR_E_OOM, "install scratch");
  launch_install_levels(e->ext, e->S, lv->w, de, dl, dk, count, 0);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  e->have_reset = true;
  return GR_OK;
}

int gr_levels_export_world(gr_levels* lv, int64_t level, uint8_t* blocks, uint8_t* items, int16_t* spawn,
                           int16_t* ladders, int64_t* chests, uint8_t* potion) {
  int rc = lv_range(lv, level, 1);
  if (rc) return rc;
  gr_env* e = lv->e;
  CK(cudaSetDevice(e->cfg.device));
  CK(cudaDeviceSynchronize());
  const size_t mb = (size_t)e->d.F * e->d.H * e->d.W;
  if (blocks) CK(cudaMemcpy(blocks, lv->w.blocks + level * mb, mb, cudaMemcpyDeviceToHost));
  if (items) CK(cudaMemcpy(items, lv->w.items + level * mb, mb, cudaMemcpyDeviceToHost));
  WMeta m;
  CK(cudaMemcpy(&m, lv->w.meta + level, sizeof(m), cudaMemcpyDeviceToHost));
  const int F = e->d.F;
  if (spawn) { spawn[0] = m.spawn[0]; spawn[1] = m.spawn[1]; }
  if (ladders)
    for (int f = 0; f < F; ++f) {
      ladders[4 * f] = m.ld[f][0]; ladders[4 * f + 1] = m.ld[f][1];
      ladders[4 * f + 2] = m.lu[f][0]; ladders[4 * f + 3] = m.lu[f][1];
    }
  if (chests)
    for (int f = 0; f < F; ++f)
      for (int jj = 0; jj < 6; ++jj)
        for (int q = 0; q < 4; ++q)
          chests[(f * 6 + jj) * 4 + q] = (e->ext && jj < m.nch[f]) ? (int64_t)m.chest[f][jj][q] : -1;
  if (potion)
    for (int k = 0; k < 6; ++k) potion[k] = m.potion[k];
  return GR_OK;
}

int gr_levels_world_info(gr_levels* lv, int64_t level, uint64_t* seed, uint32_t* template_floors) {
  int rc = lv_range(lv, level, 1);
  if (rc) return rc;
  CK(cudaSetDevice(lv->e->cfg.device));
  CK(cudaDeviceSynchronize());
  WMeta m;
  CK(cudaMemcpy(&m, lv->w.meta + level, sizeof(m), cudaMemcpyDeviceToHost));
  if (seed) *seed = m.seed;
  if (template_floors) *template_floors = (m.flags >> 8) & 0x1ffu;
  return GR_OK;
}

int gr_levels_import_world(gr_levels* lv, int64_t level, uint64_t seed, const uint8_t* blocks, const uint8_t* items,
                           const int16_t* spawn, const int16_t* ladders, const int64_t* chests, const uint8_t* potion,
                           uint32_t template_floors) {
  int rc = lv_range(lv, level, 1);
  if (rc) return rc;
  if (!blocks || !items || !spawn || !ladders || !chests || !potion) return fail(GR_E_INVALID, "null argument");
  gr_env* e = lv->e;
  const int F = e->d.F, H = e->d.H, W = e->d.W;
  WMeta m;
  memset(&m, 0, sizeof(m));
  m.spawn[0] = spawn[0];
  m.spawn[1] = spawn[1];
  for (int f = 0; f < F; ++f) {
    m.ld[f][0] = ladders[4 * f];
    m.ld[f][1] = ladders[4 * f + 1];
    m.lu[f][0] = ladders[4 * f + 2];
    m.lu[f][1] = ladders[4 * f + 3];
    int k = 0;
    for (int j = 0; j < 6; ++j) {
      const int64_t* c = chests + (f * 6 + j) * 4;
      if (c[0] < 0) continue;
      if (!e->ext) return fail(GR_E_INVALID, "the classic tier has no chests");
      if (c[0] >= H || c[1] < 0 || c[1] >= W) return fail(GR_E_INVALID, "chest outside the map");
      for (int q = 0; q < 4; ++q) m.chest[f][k][q] = (int16_t)c[q];
      ++k;
    }
    m.nch[f] = (uint8_t)k;
  }
  for (int q = 0; q < 6; ++q) {
    if (potion[q] > 5) return fail(GR_E_INVALID, "potion permutation entry %d out of range", (int)potion[q]);
    m.potion[q] = potion[q];
  }
  m.seed = seed;
  m.flags = ((template_floors & 0x1ffu) << 8) | (template_floors ? WG_FLAG_TEMPLATE : 0u);
  CK(cudaSetDevice(e->cfg.device));
  CK(cudaDeviceSynchronize());
  const size_t mb = (size_t)F * H * W;
  CK(cudaMemcpy(lv->w.blocks + level * mb, blocks, mb, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(lv->w.items + level * mb, items, mb, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(lv->w.meta + level, &m, sizeof(m), cudaMemcpyHostToDevice));
  return GR_OK;
}

int gr_episodes_completed(gr_env* e, int64_t* out) {
  if (!e || !out) return fail(GR_E_INVALID, "null argument");
  unsigned long long ep = 0;
  CK(cudaMemcpy(&ep, e->st_episodes, sizeof(ep), cudaMemcpyDeviceToHost));
  *out = (int64_t)ep;
  return GR_OK;
}

int gr_level_seeds(gr_env* e, uint64_t* host_dst) { return gr_export_field(e, GR_F_PARAMS_SEED, host_dst); }

int gr_set_profiling(gr_env* e, int32_t on) {
  if (!e) return fail(GR_E_INVALID, "null env");
  e->prof.on = on != 0;
  return GR_OK;
}

// per kernel class: summed device milliseconds and launch counts since the
// last call (classes: step, scan, info, worldgen, install, obs, policy, other)
int gr_kernel_times(gr_env* e, double* ms, int64_t* counts, int32_t n) {
  if (!e) return fail(GR_E_INVALID, "null env");
  CK(cudaSetDevice(e->cfg.device));
  CK(cudaDeviceSynchronize());
  for (int c = 0; c < PK_N; ++c) {
    double tot = 0;
    for (auto& p : e->prof.ev[c]) {
      float x = 0;
      cudaEventElapsedTime(&x, p.first, p.second);
      tot += x;
      e->prof.pool.push_back(p.first);
      e->prof.pool.push_back(p.second);
    }
    if (c < n) {
      if (ms) ms[c] = tot;
      if (counts) counts[c] = (int64_t)e->prof.ev[c].size();
    }
    e->prof.ev[c].clear();
  }
  return GR_OK;
}

int gr_set_worldgen_attempts(gr_env* e, int32_t max_attempts) {
  if (!e || max_attempts < 0) return fail(GR_E_INVALID, "max_attempts must be >= 0");
  CK(cudaSetDevice(e->cfg.device));
  CK(cudaDeviceSynchronize());
  e->wg_attempts = max_attempts;
  for (auto& g : e->step_graphs) cudaGraphExecDestroy(g.exec);   // they captured the old value
  e->step_graphs.clear();
  return GR_OK;
}

int gr_selftest_sincos64(const float* x, double* s, double* c, int64_t n, void* stream) {
  if (n < 0 || (n && (!x || !s || !c))) return fail(GR_E_INVALID, "bad self-test arguments");
  if (!n) return GR_OK;
  k_selftest_sincos64<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, s, c, n);
  CK(cudaGetLastError());
  return GR_OK;
}

int gr_selftest_argsort6(const float* keys, uint8_t* idx, int64_t n, void* stream) {
  if (n < 0 || (n && (!keys || !idx))) return fail(GR_E_INVALID, "bad self-test arguments");
  if (!n) return GR_OK;
  k_selftest_argsort6<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(keys, idx, n);
  CK(cudaGetLastError());
  return GR_OK;
}

int gr_worldgen_counters(gr_env* e, int64_t out[5]) {
  if (!e || !out) return fail(GR_E_INVALID, "null argument");
  unsigned long long c[5];
  CK(cudaMemcpy(c, e->counters, sizeof(c), cudaMemcpyDeviceToHost));
  for (int k = 0; k < 5; ++k) out[k] = (int64_t)c[k];
  return GR_OK;
}

}  // extern "C"
