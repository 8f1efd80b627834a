// gr_obs.cu -- observation rendering: the symbolic one-hot vector
// (obs.encode_symbolic_batch, obs.py:191-386) and the RGB tile frame
// (tiles.render_tiles, tiles.py:85-186).
//
// Both writers start from the env's 256-byte observation descriptor
// (gr_desc.cuh, written by the step / install kernels) plus the egocentric
// window of its block / item maps, and write every output byte exactly
// once with full-line stores (write-only, no read-for-ownership).
#include <cstdint>
#include <algorithm>
#include "gr_device.cuh"
#include "gr_state.cuh"
#include "gr_kernels.cuh"
#include "gr_desc.cuh"

namespace gr {

template <bool EXT>
struct OT {
  static constexpr int F = EXT ? 9 : 1, H = EXT ? 48 : 64, W = H, HW = H * W;
  static constexpr int VR = EXT ? 9 : 7, VC = EXT ? 11 : 9, T = VR * VC;
  static constexpr int BCH = EXT ? 37 : 15, ICH = EXT ? 5 : 0, CCH = EXT ? 36 : 5;
  static constexpr int STRIDE = BCH + ICH + CCH + 1;
  static constexpr int L = EXT ? 8268 : 1345;
  static constexpr int NINV = EXT ? 50 : 18;
};


// obs._CLASSIC_BLOCK_LOCAL (obs.py:46-57): block id -> classic channel,
// 4 bits per block packed in registers (lanes index it by their own tile's
// block: a __constant__ table would serialise)
__device__ __forceinline__ uint32_t classic_local(uint32_t b) {
  const uint64_t w = b < 16 ? 0xdcba987650432100ull : b < 32 ? 0xeull : 0x0ull;
  return (uint32_t)(w >> (4 * (b & 15))) & 15u;
}

// the window of env i's current floor: lane t (+32q) holds tile t's block and item
template <bool EXT>
__device__ __forceinline__ void load_window(const DS& S, int64_t i, uint32_t pos, uint32_t fl, int lane,
                                            uint8_t (&bq)[(OT<EXT>::T + 31) / 32],
                                            uint8_t (&iq)[(OT<EXT>::T + 31) / 32]) {
  using O = OT<EXT>;
  const int pr = (int16_t)(pos & 0xFFFF), pc = (int16_t)(pos >> 16), pf = fl & 0xFF;
  const uint8_t* blk = (const uint8_t*)S.f[GR_F_BLOCKS] + ((size_t)i * O::F + pf) * O::HW;
  const uint8_t* itm = (const uint8_t*)S.f[GR_F_ITEMS] + ((size_t)i * O::F + pf) * O::HW;
  const int r0 = pr - O::VR / 2, c0 = pc - O::VC / 2;
#pragma unroll
  for (int q = 0; q < (O::T + 31) / 32; ++q) {
    const int t = lane + 32 * q;
    const int r = r0 + t / O::VC, c = c0 + t % O::VC;
    const bool inb = t < O::T && r >= 0 && r < O::H && c >= 0 && c < O::W;
    bq[q] = inb ? __ldg(blk + r * O::W + c) : B_OOB;
    iq[q] = inb && EXT ? __ldg(itm + r * O::W + c) : 0;
  }
}

// ----------------------------------------------------------------- pixels
__constant__ uint8_t C_PALETTE[37][3] = {
    {0, 0, 0}, {10, 10, 10}, {64, 160, 66}, {48, 92, 190}, {120, 120, 120}, {28, 100, 38}, {134, 97, 55},
    {160, 140, 110}, {60, 60, 64}, {188, 168, 152}, {130, 220, 228}, {168, 120, 50}, {150, 80, 60},
    {216, 200, 130}, {230, 90, 16}, {96, 190, 90}, {180, 210, 70}, {84, 78, 76}, {4, 4, 4}, {86, 110, 76},
    {142, 134, 128}, {60, 110, 230}, {210, 40, 80}, {196, 150, 40}, {110, 170, 220}, {190, 110, 40},
    {180, 220, 240}, {100, 96, 90}, {150, 60, 20}, {140, 190, 210}, {240, 140, 90}, {150, 200, 255},
    {90, 20, 120}, {130, 130, 140}, {118, 118, 130}, {106, 106, 120}, {200, 60, 230}};
__constant__ uint8_t C_ITEMC[5][3] = {{255, 255, 255}, {255, 220, 90}, {20, 20, 25}, {235, 235, 240}, {70, 30, 30}};
__constant__ uint8_t C_BARC[5][3] = {{220, 60, 60}, {220, 160, 60}, {70, 130, 230}, {240, 230, 90}, {150, 90, 220}};
__constant__ uint8_t C_GEARC[7][3] = {{200, 200, 210}, {160, 160, 170}, {120, 140, 200}, {240, 220, 90},
                                      {90, 220, 140}, {220, 90, 90}, {140, 120, 240}};

__device__ __forceinline__ uint32_t creature_rgb(bool ext, int ch) {
  int kind;
  if (!ext) {
    if (ch == 4) return 0xFAFAFAu;
    kind = ch == 1 ? 0 : ch == 2 ? 2 : 1;
  } else {
    if (ch >= 20) return 0xFAFAFAu;
    kind = ch - 1;
  }
  uint32_t r, g, b;
  if (kind == 0) { r = 80; g = 200; b = 90; }
  else if (kind == 1) { r = 230; g = 230; b = 215; }
  else if (kind == 2) { r = 240; g = 190; b = 160; }
  else { r = 40 + 11 * kind; g = 255 - 12 * kind; b = 60 + 9 * kind; }
  return (r << 16) | (g << 8) | b;
}

template <bool EXT>
struct PixSmem {
  uint32_t tile_rgb[OT<EXT>::T];   // shaded tile colour
  uint32_t inset_rgb[OT<EXT>::T];  // 0xFF000000 = none
  int fill[12];                    // bar fills: 5 strip + 7 side
};

// frame geometry of one tier and tile size (tiles.py:85-133)
template <bool EXT, int PX>
struct PG {
  using O = OT<EXT>;
  static constexpr int FH = (O::VR + 2) * PX, FW = (O::VC + (EXT ? 2 : 0)) * PX;
  static constexpr int RB = FW * 3, FB = FH * RB;                  // bytes per frame row / frame
  static constexpr int INSET = PX / 4 > 1 ? PX / 4 : 1;
  static constexpr int NS = EXT ? 5 : 4;
  static constexpr int BAR_H = (2 * PX) / (NS + 1) > 2 ? (2 * PX) / (NS + 1) : 2;
  static constexpr int Y0 = O::VR * PX;
  static constexpr int NCLASS = O::VR * 4 + 6;                     // row classes (see row_class)
  // class-row stride: 32-word segments 37 words apart (see pix_word) over
  // the RB bytes plus the 8 the last chunk's funnel shift may read beyond
  static constexpr int PS = ((RB + 8 + 3) / 4 + 31) / 32 * 37 * 4;
  static constexpr int SMEM = NCLASS * PS;
  static_assert(NCLASS * PS < 65536, "row offsets are 16-bit");
};

// Pattern (class) rows are stored as 32-word segments 37 words apart; the 4
// words after a segment repeat the first 4 of the next one.  So the 5 words
// a 16-byte chunk is shifted out of sit at 5 consecutive addresses (one base
// + immediate offsets, no per-word fix-up), and lanes reading words 16 bytes
// apart (consecutive chunks) hit distinct banks (37 = 5 mod 32).  Logical
// word L sits at pix_word(L); its repeat (first 4 words of a segment) 5
// words before.
__device__ __forceinline__ int pix_word(int L) { return L + 5 * (L >> 5); }
__device__ __forceinline__ int pix_off(int B) { return 4 * pix_word(B >> 2) + (B & 3); }
__device__ __forceinline__ void put_word(uint32_t* w, int L, uint32_t v) {
  const int a = pix_word(L);
  w[a] = v;
  if ((L & 31) < 4 && L >= 32) w[a - 5] = v;
}
__device__ __forceinline__ void put_byte(uint8_t* p, int B, uint8_t v) {
  const int a = pix_off(B);
  p[a] = v;
  if (((B >> 2) & 31) < 4 && B >= 128) p[a - 20] = v;
}
// the 4 bytes at logical byte offset off >= 0 of a pattern row
__device__ __forceinline__ uint32_t pat_word(const uint32_t* w, int off) {
  const int L = off >> 2;
  const uint32_t* x = w + pix_word(L);
  return __funnelshift_r(x[0], x[1], (off & 3) * 8);
}

// The frame rows fall into a few classes that depend on the geometry only:
// within a tile row, the rows outside / inside the inset squares, with or
// without the side-panel gear bar; in the bottom strip, each vital bar and
// the blank rows.  Rows of one class are byte-identical.
template <bool EXT, int PX>
__host__ __device__ __forceinline__ int row_class(int y) {
  using G = PG<EXT, PX>;
  if (y < G::Y0) {
    const int R = y / PX, iy = y % PX;
    const bool ins = iy >= G::INSET && iy < PX - G::INSET;
    const bool bar = EXT && R < 7 && iy >= 1 && iy < PX - 1;
    return R * 4 + (ins ? 1 : 0) + (bar ? 2 : 0);
  }
  const int r = y - G::Y0 - 1;
  if (r >= 0 && r / G::BAR_H < G::NS && r % G::BAR_H < G::BAR_H - 1) return OT<EXT>::VR * 4 + r / G::BAR_H;
  return OT<EXT>::VR * 4 + 5;
}

// The 12 bar fills (f64, rounded half-even like Python round): bar k is
// computed by lane k of the warp, so the state loads and the float64
// divisions of the 12 bars overlap instead of running one after another.
// Split into the loads (issued early, beside the map-window loads) and the
// arithmetic: vital bars (tiles.py:147-166), gear panel (:169-186).
struct BarIn {
  float num;                 // vital bar: health / food / drink / energy / mana
  int isum;                  // gear bar: sword, pick, armour sum or xp
  float str_, dex, intel;
};
template <bool EXT>
__device__ __forceinline__ BarIn bar_load(const DS& S, int64_t i, int lane) {
  BarIn b{0.0f, 0, 0.0f, 0.0f, 0.0f};
  if (lane >= (EXT ? 12 : 5)) return b;
  b.str_ = (float)GR_AT(S, GR_F_STR, uint8_t, 0, i);
  b.dex = (float)GR_AT(S, GR_F_DEX, uint8_t, 0, i);
  b.intel = (float)GR_AT(S, GR_F_INTEL, uint8_t, 0, i);
  if (lane < 5) {
    if (lane == 0) b.num = GR_AT(S, GR_F_HEALTH, float, 0, i);
    else if (lane == 4) b.num = EXT ? GR_AT(S, GR_F_MANA, float, 0, i) : 0.0f;
    else b.num = GR_AT(S, lane == 1 ? GR_F_FOOD : lane == 2 ? GR_F_DRINK : GR_F_ENERGY, float, 0, i);
  } else {
    const int k = lane - 5;
    if (k == 0) b.isum = GR_AT(S, GR_F_SWORD_TIER, uint8_t, 0, i);
    else if (k == 1) b.isum = GR_AT(S, GR_F_PICK_TIER, uint8_t, 0, i);
    else if (k == 2)
      b.isum = GR_AT(S, GR_F_ARMOUR, uint8_t, 0, i) + GR_AT(S, GR_F_ARMOUR, uint8_t, 1, i) +
               GR_AT(S, GR_F_ARMOUR, uint8_t, 2, i) + GR_AT(S, GR_F_ARMOUR, uint8_t, 3, i);
    else if (k == 3) b.isum = GR_AT(S, GR_F_XP, uint8_t, 0, i);
  }
  return b;
}
template <bool EXT>
__device__ __forceinline__ int bar_compute(const BarIn& b, int px, int lane) {
  using O = OT<EXT>;
  double x;
  int width;
  if (lane < 5) {
    if (lane == 0) x = (double)b.num / (double)__fadd_rn(9.0f, b.str_);
    else if (lane == 4) x = EXT ? (double)b.num / (double)__fadd_rn(16.0f, b.intel) : 0.0;
    else x = (double)b.num / (double)__fadd_rn(12.0f, b.dex);
    width = O::VC * px - 2;
  } else {
    const int k = lane - 5;
    if (k == 0 || k == 1) x = (double)b.isum / 4.0;
    else if (k == 2 || k == 3) x = (double)b.isum / 8.0;
    else x = (double)(k == 4 ? b.dex : k == 5 ? b.str_ : b.intel) / 5.0;
    width = 2 * px - 2;
  }
  const double f = x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x);
  return (int)rint(__dmul_rn(f, (double)width));
}

// Per-env pixel inputs, written by k_pixprep into global scratch and read
// by k_pixels with one 16-byte-vector copy: shaded tile colours, inset
// colours (0xFF000000 = none) and the 12 bar fills.
template <bool EXT>
__host__ __device__ constexpr int pix_words() { return pix_scratch_words(EXT); }

// One warp per env: the view (obs.view_window / light_window / creature
// grid) from the env's 256-byte descriptor (k_step / install write it) and
// its map window, the shaded tile colours (tiles.py:113-133) and the bar
// fills.  A separate, massively parallel pass so the frame writer never
// waits on these dependent state loads.
// (no register cap: 64 registers; fitting 10 or 12 resident CTAs spills and is slower)
template <bool EXT>
__global__ void __launch_bounds__(128) k_pixprep(DS S, ObsArgs a) {
  using O = OT<EXT>;
  constexpr int TQ = (O::T + 31) / 32;
  __shared__ float light_s[4][O::T];
  __shared__ uint8_t cre_s[4][O::T];
  // colour tables in shared memory: lanes index them by their own tile's
  // block / item, which a __constant__ table would serialise
  __shared__ float pal[37][3];
  __shared__ uint32_t itemc[5];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < 37 * 3; k += blockDim.x) pal[k / 3][k % 3] = (float)C_PALETTE[k / 3][k % 3];
  if (threadIdx.x < 5)
    itemc[threadIdx.x] = ((uint32_t)C_ITEMC[threadIdx.x][0] << 16) | ((uint32_t)C_ITEMC[threadIdx.x][1] << 8) |
                         C_ITEMC[threadIdx.x][2];
  __syncthreads();
  float* light = light_s[warp];
  uint8_t* cre = cre_s[warp];
  const int64_t count = a.sel == 2 ? (int64_t)a.info->k_local : a.n;
  const int64_t stride = (int64_t)gridDim.x * 4;
  // software pipeline (extended): the next env's index, done flag and
  // descriptor are in flight while this env is built, so per env only the
  // map-window and bar-field loads (issued together) are exposed (ext 10 px:
  // 0.079 -> 0.068 ms; the classic pass, half the work per env, measured
  // no faster and its step 0.7 % slower, so it fetches each env in turn)
  constexpr bool PF = EXT;
  auto fetch = [&](int64_t jj, int64_t& ii, int& dn, uint2& dw) {
    ii = a.sel == 2 ? (int64_t)a.list[jj] : jj;   // sel 2: reset envs only
    dn = a.sel == 1 ? (int)__ldcg(a.done + ii) : 0;
    dw = reinterpret_cast<const uint2*>(S.desc + (size_t)ii * DESC_WORDS)[lane];
  };
  int64_t j = (int64_t)blockIdx.x * 4 + warp, i_n = 0;
  int dn_n = 0;
  uint2 dw_n = make_uint2(0u, 0u);
  if (PF && j < count) fetch(j, i_n, dn_n, dw_n);
  for (; j < count; j += stride) {
    if (!PF) fetch(j, i_n, dn_n, dw_n);
    const int64_t i = i_n;
    const uint2 dw = dw_n;
    const int dn = dn_n;
    if (PF && j + stride < count) fetch(j + stride, i_n, dn_n, dw_n);
    if (dn) continue;   // warp-uniform env filter (sel 1: reset this step)
    PixSmem<EXT>* dst = reinterpret_cast<PixSmem<EXT>*>(a.pix + (size_t)i * pix_words<EXT>());
    const BarIn bi = bar_load<EXT>(S, i, lane);   // independent loads, in flight with the window's
    const uint32_t pos = __shfl_sync(0xffffffffu, dw.y, D_POS / 2), fl = __shfl_sync(0xffffffffu, dw.x, D_FLAGS / 2);
    const float base = __uint_as_float(__shfl_sync(0xffffffffu, dw.x, D_BASE / 2));
    const int pr = (int16_t)(pos & 0xFFFF), pc = (int16_t)(pos >> 16), pf = fl & 0xFF;
    uint8_t bq[TQ], iq[TQ];
    load_window<EXT>(S, i, pos, fl, lane, bq, iq);
#pragma unroll
    for (int q = 0; q < TQ; ++q) {
      const int t = lane + 32 * q;
      if (t < O::T) { light[t] = base; cre[t] = 0; }
    }
    __syncwarp();
    // render_tiles sees a one-env batch: glow iff this env's floor is dark
    // (and only floors this env ever put a torch on can have one)
    if (EXT && C_FLOOR_AMB[pf] < 1.0f && ((fl >> 9) & 1u)) {
      const uint8_t* itm = (const uint8_t*)S.f[GR_F_ITEMS] + ((size_t)i * O::F + pf) * O::HW;
      constexpr int WR = O::VR + 6, WC = O::VC + 6;
      const int r0 = pr - O::VR / 2, c0 = pc - O::VC / 2;
      for (int t = lane; t < WR * WC; t += 32) {
        const int wr = t / WC - 3, wc = t % WC - 3;
        const int r = r0 + wr, c = c0 + wc;
        if (r < 0 || r >= O::H || c < 0 || c >= O::W || itm[r * O::W + c] != I_TORCH) continue;
        for (int aa = max(wr - 3, 0); aa <= min(wr + 3, O::VR - 1); ++aa)
          for (int bb = max(wc - 3, 0); bb <= min(wc + 3, O::VC - 1); ++bb) {
            const int d = max(abs(aa - wr), abs(bb - wc));
            atomicMax(reinterpret_cast<int*>(&light[aa * O::VC + bb]), __float_as_int(1.0f - 0.25f * (float)d));
          }
      }
      __syncwarp();
    }
    // creature cells: slot lane < NSLOT; the highest slot wins a cell
    constexpr int NSLOT = EXT ? 14 : 11;
    uint32_t sl = 0xFFFFu;
    {
      // gather descriptor word D_CRE + (lane >> 1) into every lane
      const int wi = D_CRE + ((lane < NSLOT ? lane : 0) >> 1);
      const uint32_t lo = __shfl_sync(0xffffffffu, dw.x, wi >> 1), hi = __shfl_sync(0xffffffffu, dw.y, wi >> 1);
      const uint32_t word = (wi & 1) ? hi : lo;
      if (lane < NSLOT) sl = (word >> (16 * (lane & 1))) & 0xFFFFu;
    }
    const int cell = sl == 0xFFFFu ? -1 : (int)(sl >> 8);
    bool win = cell >= 0;
    for (int s = 1; s < NSLOT; ++s) {
      const int oc = __shfl_down_sync(0xffffffffu, cell, s);
      if (lane + s < NSLOT && oc == cell) win = false;
    }
    if (win) cre[cell] = (uint8_t)(sl & 0xFF);
    const bool sleeping = (fl >> 8) & 1;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < TQ; ++q) {
      const int t = lane + 32 * q;
      if (t >= O::T) continue;
      const float l = sleeping ? 0.0f : light[t];
      const float sh = l < 0.0f ? 0.0f : (l > 1.0f ? 1.0f : l);
      const bool dark = l < 0.05f;
      const int b = bq[q];
      uint32_t rgb = 0;
      if (!dark)
        for (int k = 0; k < 3; ++k)
          rgb |= (uint32_t)(uint8_t)(int)__fmul_rn(pal[b][k], sh) << (16 - 8 * k);
      dst->tile_rgb[t] = rgb;
      uint32_t ins = 0xFF000000u;
      if (!dark) {
        const int it = iq[q];
        if (it) ins = itemc[it];
        if (cre[t]) ins = creature_rgb(EXT, cre[t]);
      }
      if (t == (O::VR / 2) * O::VC + O::VC / 2) ins = 0xFA3C3Cu;   // the player
      dst->inset_rgb[t] = ins;
    }
    if (lane < (EXT ? 12 : 5)) dst->fill[lane] = bar_compute<EXT>(bi, a.tile_px, lane);
    __syncwarp();
  }
}

// The frame writer: one CTA per env at a time, software-pipelined over the
// CTA's envs.
//  1. one byte row per row class present (<= 31 rows, ~1/4 of the frame):
//     tile rows per tile segment, side panel and bottom strip per pixel
//  2. the frame streamed out as 16-byte stores of the globally 16-byte
//     aligned chunks of the env's byte range (frames are 42,900 / 11,907 B,
//     not 16-byte multiples), each the funnel shift of 5 words of its class
//     row (stored with a pad word per 32 so the lanes' loads are free of
//     bank conflicts); the <= 1 chunk per frame-row boundary that straddles
//     two rows and the head / tail bytes outside the aligned chunks are a
//     separate, small pass.  A warp store covers 512 contiguous bytes;
//     meanwhile the next env's inputs (k_pixprep scratch) arrive in the
//     other buffer by cp.async.  (4-byte words per lane measured slower:
//     4x the loop overhead.)
// threads per frame CTA: large frames stream faster with more (extended 10 px:
// 128 -> 384 took the writer from 0.95 to 0.84 ms; 512+ slower), small
// frames prefer 128 (classic 7 px: 384 was 10 % slower)
#ifndef GR_PIX_MINB
#define GR_PIX_MINB 4   // resident frame CTAs per SM the registers are fitted to (ext px10: 40 registers, 4 CTAs/SM)
#endif
#ifndef GR_PIX_STREAM_INC
#define GR_PIX_STREAM_INC 1   // incremental (row, offset) walk in the chunk stream (0: divide per chunk)
#endif
template <bool EXT, int PX>
// (end of round 2, 65,536 envs: classic 7 px with 96 threads 0.350 -> 0.343
// ms per step; classic 10 px and extended 7 px lose with 96 or fewer, 64 and
// 32 lose everywhere)
__host__ __device__ constexpr int pix_threads() {
  return !EXT && PX == 7 ? 96 : PG<EXT, PX>::FB >= 32768 ? 384 : 128;
}

template <bool EXT, int PX>
__global__ void __launch_bounds__(pix_threads<EXT, PX>(), GR_PIX_MINB) k_pixels(DS S, ObsArgs a) {
  using O = OT<EXT>;
  using G = PG<EXT, PX>;
  constexpr int PW = pix_words<EXT>();
  static_assert(sizeof(PixSmem<EXT>) <= PW * 4, "scratch layout");
  extern __shared__ uint4 pix_dyn[];
  uint8_t* pat = reinterpret_cast<uint8_t*>(pix_dyn);   // [NCLASS][PS]
  __shared__ __align__(16) uint32_t pmw[2][PW];
  __shared__ uint8_t rowcls[G::FH];
  __shared__ uint16_t rowoff[G::FH];   // byte offset of frame row y's class row
  __shared__ int16_t rep[G::NCLASS];
  __shared__ uint8_t ucls[G::NCLASS];
  __shared__ int nused;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // row class of every frame row, one representative row per class and the
  // list of classes present (geometry only: once per CTA); rows of a class
  // are identical, so any representative will do
  for (int c = threadIdx.x; c < G::NCLASS; c += blockDim.x) rep[c] = -1;
  __syncthreads();
  for (int y = threadIdx.x; y < G::FH; y += blockDim.x) {
    const int c = row_class<EXT, PX>(y);
    rowcls[y] = (uint8_t)c;
    rowoff[y] = (uint16_t)(c * G::PS);
    rep[c] = (int16_t)y;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int u = 0;
    for (int c = 0; c < G::NCLASS; ++c)
      if (rep[c] >= 0) ucls[u++] = (uint8_t)c;
    nused = u;
  }
  const int64_t count = a.sel == 2 ? (int64_t)a.info->k_local : a.n;
  const int64_t stride = gridDim.x;
  // the CTA's next env at or after list position jj (-1: none)
  auto next_env = [&](int64_t jj) -> int64_t {
    for (; jj < count; jj += stride) {
      const int64_t ii = a.sel == 2 ? (int64_t)a.list[jj] : jj;
      if (a.sel == 1 && a.done[ii]) continue;   // CTA-uniform env filter
      return jj;
    }
    return -1;
  };
  auto env_of = [&](int64_t jj) -> int64_t { return a.sel == 2 ? (int64_t)a.list[jj] : jj; };
  // env ii's scratch -> pmw[b] (warp 0, asynchronous)
  auto fetch = [&](int64_t ii, int b) {
    const char* src = reinterpret_cast<const char*>(a.pix + (size_t)ii * PW);
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&pmw[b][0]);
    for (int q = lane; q < PW / 4; q += 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * q), "l"(src + 16 * q) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int64_t j = next_env(blockIdx.x);
  if (j >= 0 && warp == 0) {
    fetch(env_of(j), 0);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  int cur = 0;
  // frame offsets are taken from the 16-byte-aligned address at or below
  // the buffer, so the "aligned" chunks are aligned in absolute terms for
  // any buffer alignment (a uint8 tensor view may start anywhere)
  const int mis = (int)(reinterpret_cast<uintptr_t>(a.out) & 15u);
  uint8_t* out = (uint8_t*)a.out - mis;
  while (j >= 0) {
    const int64_t i = env_of(j);
    // the next env: its done flag is loaded now and only looked at after
    // the class rows are built, so the load's latency hides under the build
    // (resolving it here stalled every frame's start on a global load)
    const int64_t cand = j + stride;
    const bool cand_ok = cand < count;
    const uint8_t cand_done = (a.sel == 1 && cand_ok) ? __ldcg(a.done + cand) : (uint8_t)0;
    const PixSmem<EXT>& pm = *reinterpret_cast<const PixSmem<EXT>*>(&pmw[cur][0]);
    // 1. class rows
    {
      const int nu = nused;
      constexpr int NTC = O::VR * 4;   // tile-row classes are [0, NTC)
      // tile segments, as 4-byte words: GS consecutive segments (3*PX*GS
      // bytes, a multiple of 4) per task, each word assembled in registers
      // from the segments' tile / inset colours (byte positions are
      // compile-time after unrolling); the < GS segments left at the row
      // end are written byte by byte
      // (odd PX would need 4-segment groups: too few, too long tasks for the
      // 128-thread classic CTAs -- classic 7 px measured 0.295 -> 0.326 ms --
      // so those stay on the byte path; ext 10 px: 0.857 -> 0.809 ms)
      constexpr int SEGB = 3 * PX;
      constexpr int GS = SEGB % 4 == 0 ? 1 : SEGB % 2 == 0 ? 2 : 4;
      constexpr int GW = SEGB * GS / 4, NGR = GS <= 2 ? O::VC / GS : 0;
      for (int q = threadIdx.x; q < nu * NGR; q += blockDim.x) {
        const int c = ucls[q / NGR], g = q % NGR;
        if (c >= NTC) continue;
        uint32_t ct[GS], ci[GS];
#pragma unroll
        for (int k = 0; k < GS; ++k) {
          const int t = (c >> 2) * O::VC + g * GS + k;
          ct[k] = pm.tile_rgb[t];
          const uint32_t ic = pm.inset_rgb[t];
          ci[k] = (c & 1) && ic != 0xFF000000u ? ic : ct[k];
        }
        uint32_t* wp = reinterpret_cast<uint32_t*>(pat + c * G::PS);
        const int L0 = g * GW;
#pragma unroll
        for (int w = 0; w < GW; ++w) {
          uint32_t v = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int gb = 4 * w + j, k = gb / SEGB, sb = gb % SEGB, ix = sb / 3, ch = sb % 3;
            const uint32_t rgb = ix >= G::INSET && ix < PX - G::INSET ? ci[k] : ct[k];
            v |= ((rgb >> (8 * (2 - ch))) & 0xFFu) << (8 * j);
          }
          put_word(wp, L0 + w, v);
        }
      }
      constexpr int LEFT = O::VC - NGR * GS;
      if constexpr (LEFT > 0)
      for (int q = threadIdx.x; q < nu * LEFT; q += blockDim.x) {
        const int c = ucls[q / LEFT], C = NGR * GS + q % LEFT;
        if (c >= NTC) continue;
        const int t = (c >> 2) * O::VC + C;
        const uint32_t tc = pm.tile_rgb[t], ic = pm.inset_rgb[t];
        const bool ins = (c & 1) && ic != 0xFF000000u;
        uint8_t* p = pat + c * G::PS;
        const int B0 = 3 * PX * C;
#pragma unroll
        for (int ix = 0; ix < PX; ++ix) {
          const uint32_t rgb = ins && ix >= G::INSET && ix < PX - G::INSET ? ic : tc;
          put_byte(p, B0 + 3 * ix, (uint8_t)(rgb >> 16));
          put_byte(p, B0 + 3 * ix + 1, (uint8_t)(rgb >> 8));
          put_byte(p, B0 + 3 * ix + 2, (uint8_t)rgb);
        }
      }
      // side panel of the tile-row classes (gear bar k = tile row, per
      // pixel, byte stores: the panel is not word-aligned) ...
      constexpr int SW = G::FW - O::VC * PX;   // side panel width (0 classic)
      for (int q = threadIdx.x; q < nu * SW; q += blockDim.x) {
        const int c = ucls[q / SW], xx = q % SW;
        if (c >= NTC) continue;
        const int k = c >> 2;
        uint32_t rgb = 0u;
        if ((c & 2) && xx >= 1 && xx < 2 * PX - 1)   // (c & 2): a gear-bar row (row_class)
          rgb = xx < 1 + pm.fill[5 + k] ? ((uint32_t)C_GEARC[k][0] << 16) | ((uint32_t)C_GEARC[k][1] << 8) | C_GEARC[k][2]
                                        : 0x1E1E1Eu;
        uint8_t* p = pat + c * G::PS;
        const int B0 = 3 * (O::VC * PX + xx);
        put_byte(p, B0, (uint8_t)(rgb >> 16));
        put_byte(p, B0 + 1, (uint8_t)(rgb >> 8));
        put_byte(p, B0 + 2, (uint8_t)rgb);
      }
      // ... and the bottom-strip classes (vital bar k, or blank), 4 pixels
      // -> 3 words per task
      constexpr int NG = (G::FW + 3) / 4;
      for (int q = threadIdx.x; q < 6 * NG; q += blockDim.x) {
        const int k = q / NG, x0 = 4 * (q - k * NG), c = NTC + k;
        if (rep[c] < 0) continue;
        const uint32_t barc = k < G::NS ? ((uint32_t)C_BARC[k][0] << 16) | ((uint32_t)C_BARC[k][1] << 8) | C_BARC[k][2] : 0u;
        const int fl = k < G::NS ? pm.fill[k] : 0;
        uint32_t cl[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int x = x0 + m;
          cl[m] = k < G::NS && x >= 1 && x < 1 + O::VC * PX - 2 ? (x < 1 + fl ? barc : 0x1E1E1Eu) : 0u;
        }
        // bytes r0 g0 b0 r1 | g1 b1 r2 g2 | b2 r3 g3 b3 (little-endian words)
        uint32_t* p = reinterpret_cast<uint32_t*>(pat + c * G::PS);
        const int L0 = 3 * x0 / 4;   // 3 * x0 is a multiple of 4
        put_word(p, L0, __byte_perm(cl[0], cl[1], 0x6012));
        put_word(p, L0 + 1, __byte_perm(cl[1], cl[2], 0x5601));
        put_word(p, L0 + 2, __byte_perm(cl[2], cl[3], 0x4560));
      }
    }
    __syncthreads();
    const int64_t jn = !cand_ok ? -1 : cand_done ? next_env(cand + stride) : cand;
    if (warp == 0 && jn >= 0) fetch(env_of(jn), cur ^ 1);   // the next env's inputs, under this env's stores
    // 2. stream the frame: bytes [f0, f0 + FB) of the output
    const int64_t f0 = i * (int64_t)G::FB + mis;
    const int64_t c0 = (f0 + 15) & ~(int64_t)15, c1 = (f0 + G::FB) & ~(int64_t)15;
    const int nchunk = (int)((c1 - c0) >> 4);
    auto byte_at = [&](int b) -> uint32_t {
      const int y = b / G::RB;
      return pat[rowcls[y] * G::PS + pix_off(b - y * G::RB)];
    };
    // straddling chunks (one per frame-row boundary not on a 16-byte
    // boundary) and the head / tail bytes
    for (int q = threadIdx.x; q < G::FH - 1 + 32; q += blockDim.x) {
      if (q < G::FH - 1) {
        const int64_t bnd = f0 + (int64_t)(q + 1) * G::RB;
        const int64_t c = bnd & ~(int64_t)15;
        if (c == bnd || c < c0 || c >= c1) continue;
        // n bytes from the tail of row q, the rest from the head of row q + 1
        const int b = (int)(c - f0), o = b - q * G::RB, n = G::RB - o;
        const uint32_t* wa = reinterpret_cast<const uint32_t*>(pat + rowcls[q] * G::PS);
        const uint32_t* wb = reinterpret_cast<const uint32_t*>(pat + rowcls[q + 1] * G::PS);
        uint32_t wv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int m = n - 4 * k;   // bytes of word k from row q
          if (m >= 4) {
            wv[k] = pat_word(wa, o + 4 * k);
          } else if (m <= 0) {
            wv[k] = pat_word(wb, -m);
          } else {
            const uint32_t keep = 0xFFFFFFFFu >> (32 - 8 * m);
            wv[k] = (pat_word(wa, o + 4 * k) & keep) | (wb[pix_word(0)] << (8 * m));
          }
        }
        *reinterpret_cast<uint4*>(out + c) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      } else {
        const int r = q - (G::FH - 1);
        const int head = (int)(c0 - f0), tail = (int)(f0 + G::FB - c1);
        if (r < 16) {
          if (r < head) out[f0 + r] = (uint8_t)byte_at(r);
        } else if (r - 16 < tail) {
          out[c1 + r - 16] = (uint8_t)byte_at((int)(c1 - f0) + r - 16);
        }
      }
    }
    // the aligned chunks inside one frame row: lane-consecutive, so a warp
    // store covers 512 contiguous bytes; a chunk at row offset o is the
    // funnel shift of the 5 pattern words from o & ~3 (padded layout: the
    // lanes' loads hit distinct banks)
#if GR_PIX_STREAM_INC
    {
      // (row, offset) of each thread's chunk advance by a constant per pass
      // (NT * 16 bytes = DY rows + DO bytes), so no division per chunk; the
      // pattern is addressed in words with the pad word per 32 folded in
      constexpr int NT = pix_threads<EXT, PX>();
      constexpr int DY = NT * 16 / G::RB, DO = NT * 16 - DY * G::RB;
      // shared-space addresses (32-bit, laundered through a mov so they stay
      // in registers instead of being re-derived from the CTA id every
      // chunk): per chunk one row-offset load, 5 pattern loads at immediate
      // offsets, 4 funnel shifts and the store
      uint32_t pat_s, row_s;
      asm volatile("mov.u32 %0, %1;" : "=r"(pat_s) : "r"((uint32_t)__cvta_generic_to_shared(pat)));
      asm volatile("mov.u32 %0, %1;" : "=r"(row_s) : "r"((uint32_t)__cvta_generic_to_shared(rowoff)));
      int b = (int)(c0 - f0) + 16 * (int)threadIdx.x;
      int y = b / G::RB, o = b - y * G::RB;
      uint4* dst = reinterpret_cast<uint4*>(out + c0) + threadIdx.x;
#pragma unroll 2
      for (int q = threadIdx.x; q < nchunk; q += NT) {
        if (o <= G::RB - 16) {
          uint32_t ro, x0, x1, x2, x3, x4;
          asm volatile("ld.shared.u16 %0, [%1];" : "=r"(ro) : "r"(row_s + 2u * (uint32_t)y));
          const uint32_t ad = pat_s + ro + (uint32_t)(o & ~3) + 20u * (uint32_t)(o >> 7);
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x0) : "r"(ad));
          asm volatile("ld.shared.u32 %0, [%1+4];" : "=r"(x1) : "r"(ad));
          asm volatile("ld.shared.u32 %0, [%1+8];" : "=r"(x2) : "r"(ad));
          asm volatile("ld.shared.u32 %0, [%1+12];" : "=r"(x3) : "r"(ad));
          asm volatile("ld.shared.u32 %0, [%1+16];" : "=r"(x4) : "r"(ad));
          const uint32_t sh = (uint32_t)(o & 3) * 8u;
          *dst = make_uint4(__funnelshift_r(x0, x1, sh), __funnelshift_r(x1, x2, sh), __funnelshift_r(x2, x3, sh),
                            __funnelshift_r(x3, x4, sh));
        }
        dst += NT;
        y += DY;
        o += DO;
        if (o >= G::RB) { o -= G::RB; ++y; }
      }
    }
#else
    for (int q = threadIdx.x; q < nchunk; q += blockDim.x) {
      const int b = (int)(c0 - f0) + 16 * q;
      const int y = b / G::RB, o = b - y * G::RB;
      if (o + 16 <= G::RB) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(pat + rowcls[y] * G::PS);
        const int L = o >> 2, sh = (o & 3) * 8;
        uint32_t x[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) x[k] = w[pix_word(L + k)];
        const uint4 val = make_uint4(__funnelshift_r(x[0], x[1], sh), __funnelshift_r(x[1], x[2], sh),
                                     __funnelshift_r(x[2], x[3], sh), __funnelshift_r(x[3], x[4], sh));
        *reinterpret_cast<uint4*>(out + c0 + 16 * (int64_t)q) = val;
      }
    }
#endif
    if (warp == 0) asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    j = jn;
    cur ^= 1;
  }
}

template <bool EXT, int PX>
static void launch_pixels_px(const DS& S, const ObsArgs& a, int sms, cudaStream_t st) {
  constexpr int smem = PG<EXT, PX>::SMEM;
  static PerDeviceOnce once;
  static int occ[64];
  int dev = 0;
  cudaGetDevice(&dev);
  once([&](int d) {
    int o = 0;
    cudaFuncSetAttribute(k_pixels<EXT, PX>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_pixels<EXT, PX>, pix_threads<EXT, PX>(), smem);
    occ[d] = o < 1 ? 1 : o;
  });
  const int per_sm = occ[dev & 63];
  // persistent grid: every CTA resident from the start (k_pixprep ran before, launch_pixprep)
  k_pixels<EXT, PX><<<(int)std::min<int64_t>(a.n, (int64_t)sms * per_sm), pix_threads<EXT, PX>(), smem, st>>>(S, a);
}

// ---------------------------------------------------- symbolic writer
// One warp per env.  The 256-byte descriptor (k_step / install write it)
// plus the egocentric window of the block / item maps become, per tile, the
// <= 3 one-hot channel targets (pre-masked by the light threshold) and the
// light scalar.  The row is ~95% zeros: each warp keeps one zero-initialised
// copy of a row in shared memory, scatters the non-zeros into it, streams it
// out (one TMA bulk store for extended rows, 16-byte stores otherwise) and
// scatters the zeros back -- O(non-zeros) shared-memory work per env and
// every global byte written exactly once.
//
// The loop is software-pipelined: the descriptor of the next env is loaded
// while the current one is built, and the next env's map window is loaded
// while the current row drains, so the two dependent global loads per env
// (descriptor -> window) overlap the store instead of serialising with it.
template <bool EXT>
struct TileSmem {
  uint32_t tgt[OT<EXT>::T];   // on-channels: 3 x 8 bits (0xFF = none)
  float light[OT<EXT>::T];
  uint32_t desc[DESC_WORDS];
};

#ifndef GR_OBS_WIN_EARLY
#define GR_OBS_WIN_EARLY 1   // symbolic writer: next env's window loads issued before the scatter
#endif
template <bool EXT>
#ifndef GR_CLS_WARPS
#define GR_CLS_WARPS 4   // classic symbolic writer: warps (rows in flight) per CTA (4 x 8 CTAs/SM: 0.1378 -> 0.1370 ms/step at 65,536 envs against 8 x 4)
#endif
#ifndef GR_CLS_CTAS
#define GR_CLS_CTAS 8    // classic symbolic writer: CTAs per SM (8 x 5, 4 x 10, 16 x 2 measured slower)
#endif
__host__ __device__ constexpr int stage_warps() { return EXT ? 2 : GR_CLS_WARPS; }
// one stage = one whole row + up to 3 floats of alignment shift
template <bool EXT>
__host__ __device__ constexpr int stage_floats() { return EXT ? 8272 : 1352; }

template <bool EXT>
__global__ void __launch_bounds__(stage_warps<EXT>() * 32) k_symbolic_stage(DS S, ObsArgs a) {
  using O = OT<EXT>;
  constexpr int NW = stage_warps<EXT>();
  constexpr int SC = stage_floats<EXT>();
  constexpr int TQ = (O::T + 31) / 32;
  static_assert(SC >= O::L + 3, "a stage holds a whole row");
  extern __shared__ float4 dyn_smem[];
  __shared__ TileSmem<EXT> views[NW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  TileSmem<EXT>& v = views[warp];
  float* stage = reinterpret_cast<float*>(dyn_smem) + (size_t)warp * SC;
  for (int q = lane; q < SC / 4; q += 32) reinterpret_cast<float4*>(stage)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncwarp();
  const bool glow = EXT && a.flags && (a.flags[0] & 4u);
  const bool tma = EXT && a.tma;
  const int64_t count = a.sel == 2 ? (int64_t)a.info->k_local : a.n;
  const int64_t stride = (int64_t)gridDim.x * NW;
  // env at list position jj and its descriptor words 2*lane, 2*lane+1; the
  // done flag (sel 1 skips the envs reset this step) is loaded beside the
  // descriptor and only checked once the descriptor is needed (settle)
  auto issue = [&](int64_t jj, int64_t& ii, uint2& dw, int& dn) {
    ii = a.sel == 2 ? (int64_t)a.list[jj] : jj;
    dn = a.sel == 1 ? a.done[ii] : 0;
    dw = reinterpret_cast<const uint2*>(S.desc + (size_t)ii * DESC_WORDS)[lane];
  };
  auto settle = [&](int64_t& jj, int64_t& ii, uint2& dw, int& dn) -> bool {
    while (jj < count && dn) {   // warp-uniform
      jj += stride;
      if (jj < count) issue(jj, ii, dw, dn);
    }
    return jj < count;
  };
  int64_t jn = (int64_t)blockIdx.x * NW + warp, in = 0;
  uint2 dwn = make_uint2(0, 0);
  int dn = 0;
  uint8_t bqn[TQ], iqn[TQ];
  if (jn < count) issue(jn, in, dwn, dn);
  bool have = settle(jn, in, dwn, dn);
  if (have)
    load_window<EXT>(S, in, __shfl_sync(0xffffffffu, dwn.y, D_POS / 2), __shfl_sync(0xffffffffu, dwn.x, D_FLAGS / 2),
                     lane, bqn, iqn);
  while (have) {
    const int64_t i = in;
    uint8_t bq[TQ], iq[TQ];
#pragma unroll
    for (int q = 0; q < TQ; ++q) { bq[q] = bqn[q]; iq[q] = iqn[q]; }
    v.desc[2 * lane] = dwn.x;
    v.desc[2 * lane + 1] = dwn.y;
    // the descriptor of the next env is in flight while this one is built
    jn += stride;
    if (jn < count) issue(jn, in, dwn, dn);
    __syncwarp();
    const uint32_t pos = v.desc[D_POS], fl = v.desc[D_FLAGS];
    const int pr = (int16_t)(pos & 0xFFFF), pc = (int16_t)(pos >> 16), pf = fl & 0xFF;
    const bool sleeping = (fl >> 8) & 1;
    const float base = __uint_as_float(v.desc[D_BASE]);
    const int r0 = pr - O::VR / 2, c0 = pc - O::VC / 2;
#pragma unroll
    for (int q = 0; q < TQ; ++q) {
      const int t = lane + 32 * q;
      if (t < O::T) v.light[t] = base;
    }
    __syncwarp();
    if (glow && ((fl >> 9) & 1u)) {   // only floors this env ever put a torch on
      const uint8_t* itm = (const uint8_t*)S.f[GR_F_ITEMS] + ((size_t)i * O::F + pf) * O::HW;
      constexpr int WR = O::VR + 6, WC = O::VC + 6;
      for (int t = lane; t < WR * WC; t += 32) {
        const int wr = t / WC - 3, wc = t % WC - 3;
        const int r = r0 + wr, c = c0 + wc;
        if (r < 0 || r >= O::H || c < 0 || c >= O::W || itm[r * O::W + c] != I_TORCH) continue;
        for (int aa = max(wr - 3, 0); aa <= min(wr + 3, O::VR - 1); ++aa)
          for (int bb = max(wc - 3, 0); bb <= min(wc + 3, O::VC - 1); ++bb) {
            const int d = max(abs(aa - wr), abs(bb - wc));
            atomicMax(reinterpret_cast<int*>(&v.light[aa * O::VC + bb]), __float_as_int(1.0f - 0.25f * (float)d));
          }
      }
      __syncwarp();
    }
    // creature cells: slot lane < NSLOT; the highest slot wins a cell
    constexpr int NSLOT = EXT ? 14 : 11;
    uint32_t sl = 0xFFFFu;
    if (lane < NSLOT) sl = (v.desc[D_CRE + (lane >> 1)] >> (16 * (lane & 1))) & 0xFFFFu;
    const int cell = sl == 0xFFFFu ? -1 : (int)(sl >> 8);
    bool win = cell >= 0;
    for (int s = 1; s < NSLOT; ++s) {
      const int oc = __shfl_down_sync(0xffffffffu, cell, s);
      if (lane + s < NSLOT && oc == cell) win = false;
    }
#pragma unroll
    for (int q = 0; q < TQ; ++q) {
      const int t = lane + 32 * q;
      if (t < O::T) {
        if (sleeping) v.light[t] = 0.0f;
        const bool lit = v.light[t] >= 0.05f;
        const uint32_t bc = EXT ? bq[q] : classic_local(bq[q]);
        const uint32_t ic = EXT ? (uint32_t)(O::BCH + iq[q]) : 0xFFu;
        v.tgt[t] = lit ? (bc | ic << 8 | (uint32_t)(O::BCH + O::ICH) << 16) : 0xFFFFFFu;
      }
    }
    __syncwarp();
    if (win && (v.tgt[cell] >> 16) != 0xFFu)
      v.tgt[cell] = (v.tgt[cell] & 0xFFFFu) | ((uint32_t)(O::BCH + O::ICH + (sl & 0xFF)) << 16);
    __syncwarp();
    // element p of the row sits at stage[p + shift]: shift aligns the
    // 16-byte groups of the stage with those of the destination
    float* row = (float*)a.out + (size_t)i * O::L;
    const int shift = (int)((reinterpret_cast<uintptr_t>(row) & 15u) >> 2);
    float* sr = stage + shift;
#if GR_OBS_WIN_EARLY
    // the next env's window loads are issued before this row's scatter (its
    // descriptor had the whole build to arrive), so they overlap the
    // scatter, the drain and the unscatter
    have = settle(jn, in, dwn, dn);
    if (have)
      load_window<EXT>(S, in, __shfl_sync(0xffffffffu, dwn.y, D_POS / 2),
                       __shfl_sync(0xffffffffu, dwn.x, D_FLAGS / 2), lane, bqn, iqn);
#endif
    for (int t = lane; t < O::T; t += 32) {
      const uint32_t g = v.tgt[t];
      float* tv = sr + t * O::STRIDE;
      if ((g & 0xFF) != 0xFF) {
        tv[g & 0xFF] = 1.0f;
        if (EXT) tv[(g >> 8) & 0xFF] = 1.0f;
        tv[g >> 16] = 1.0f;
      }
      tv[O::STRIDE - 1] = v.light[t];
    }
    for (int k = lane; k < O::NINV; k += 32) sr[O::T * O::STRIDE + k] = __uint_as_float(v.desc[D_INV + k]);
#if !GR_OBS_WIN_EARLY
    have = settle(jn, in, dwn, dn);
#endif
    if (tma) {
      // extended rows are 33,072 B = a 16-byte multiple at 16-byte aligned
      // addresses: one TMA bulk store (cp.async.bulk) per row, issued by one
      // lane; the warp waits only until the stage has been read
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const uint32_t saddr = (uint32_t)__cvta_generic_to_shared(sr);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     :: "l"(row), "r"(saddr), "r"((uint32_t)(O::L * 4)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
#if !GR_OBS_WIN_EARLY
      // the next env's window loads overlap the drain of this row
      if (have)
        load_window<EXT>(S, in, __shfl_sync(0xffffffffu, dwn.y, D_POS / 2),
                         __shfl_sync(0xffffffffu, dwn.x, D_FLAGS / 2), lane, bqn, iqn);
#endif
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
    } else {
#if !GR_OBS_WIN_EARLY
      if (have)
        load_window<EXT>(S, in, __shfl_sync(0xffffffffu, dwn.y, D_POS / 2),
                         __shfl_sync(0xffffffffu, dwn.x, D_FLAGS / 2), lane, bqn, iqn);
#endif
      __syncwarp();
      const int head = (4 - shift) & 3;
      if (lane < head) row[lane] = sr[lane];
      const int nv = (O::L - head) >> 2;
      const float4* s4 = reinterpret_cast<const float4*>(sr + head);
      float4* g4 = reinterpret_cast<float4*>(row + head);
      for (int q = lane; q < nv; q += 32) g4[q] = s4[q];
      const int tl = head + nv * 4;
      if (tl + lane < O::L) row[tl + lane] = sr[tl + lane];
      __syncwarp();
    }
    for (int t = lane; t < O::T; t += 32) {
      const uint32_t g = v.tgt[t];
      float* tv = sr + t * O::STRIDE;
      if ((g & 0xFF) != 0xFF) {
        tv[g & 0xFF] = 0.0f;
        if (EXT) tv[(g >> 8) & 0xFF] = 0.0f;
        tv[g >> 16] = 0.0f;
      }
      tv[O::STRIDE - 1] = 0.0f;
    }
    for (int k = lane; k < O::NINV; k += 32) sr[O::T * O::STRIDE + k] = 0.0f;
    __syncwarp();
  }
  // bulk stores must complete before the CTA retires
  if (tma && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// the per-env pass before the pixel writer (k_pixprep); persistent grid,
// 4 envs per CTA
void launch_pixprep(bool ext, const DS& S, const ObsArgs& a, cudaStream_t st) {
  if (a.n <= 0 || !a.pix) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>((a.n + 3) / 4, (int64_t)sms * 16);
  if (ext) k_pixprep<true><<<grid, 128, 0, st>>>(S, a);
  else k_pixprep<false><<<grid, 128, 0, st>>>(S, a);
}

void launch_symbolic(bool ext, const DS& S, const ObsArgs& a, cudaStream_t st) {
  if (a.n <= 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (ext) {
    constexpr int NW = stage_warps<true>();
    const size_t smem = (size_t)NW * stage_floats<true>() * sizeof(float);
    static PerDeviceOnce once;
    once([&](int) { cudaFuncSetAttribute(k_symbolic_stage<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
    const int per_sm = a.ctas_per_sm > 0 ? a.ctas_per_sm : 3;
    const int grid = (int)std::min<int64_t>((a.n + NW - 1) / NW, (int64_t)sms * per_sm);
    k_symbolic_stage<true><<<grid, NW * 32, smem, st>>>(S, a);
  } else {
    constexpr int NW = stage_warps<false>();
    const size_t smem = (size_t)NW * stage_floats<false>() * sizeof(float);
    static PerDeviceOnce once;
    once([&](int) { cudaFuncSetAttribute(k_symbolic_stage<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
    const int grid = (int)std::min<int64_t>((a.n + NW - 1) / NW, (int64_t)sms * GR_CLS_CTAS);
    k_symbolic_stage<false><<<grid, NW * 32, smem, st>>>(S, a);
  }
}

// ---- pixel frames to the host, packed by row class ------------------------
// Rows of one class are byte-identical in every frame (k_pixels only ever
// renders the class rows), so a frame is determined by its class rows: the
// transfer to a host array moves one representative row per class present
// (~12 KB of a 42.9 KB extended 10 px frame) and host threads replicate them.
template <bool EXT, int PX>
static void row_map_px(PixRowMap* m) {
  using G = PG<EXT, PX>;
  m->FH = G::FH;
  m->RB = G::RB;
  m->FB = G::FB;
  int slot[64];
  for (int c = 0; c < 64; ++c) slot[c] = -1;
  m->nused = 0;
  for (int y = 0; y < G::FH; ++y) {
    const int c = row_class<EXT, PX>(y);
    if (slot[c] < 0) {
      slot[c] = m->nused;
      m->rep[m->nused++] = (int16_t)y;
    }
    m->slot_of_row[y] = (int16_t)slot[c];
  }
}

int pixel_row_map(bool ext, int px, PixRowMap* m) {
  switch ((ext ? 100 : 0) + px) {
    case 7: row_map_px<false, 7>(m); return 0;
    case 10: row_map_px<false, 10>(m); return 0;
    case 16: row_map_px<false, 16>(m); return 0;
    case 107: row_map_px<true, 7>(m); return 0;
    case 110: row_map_px<true, 10>(m); return 0;
    case 116: row_map_px<true, 16>(m); return 0;
    default: return -1;
  }
}

// one CTA per env: the representative rows of frames [r0, r1) -> out[env - r0][slot][RB]
__global__ void __launch_bounds__(256) k_pix_gather(const uint8_t* __restrict__ frames, int64_t r0, int64_t r1, int FB,
                                                     int RB, int nused, PixRowMap map, uint8_t* __restrict__ out) {
  for (int64_t r = r0 + blockIdx.x; r < r1; r += gridDim.x) {
    const uint8_t* f = frames + r * (int64_t)FB;
    uint8_t* o = out + (r - r0) * (int64_t)nused * RB;   // out is this chunk's region
    for (int q = threadIdx.x; q < nused * RB; q += blockDim.x) {
      const int k = q / RB, b = q - k * RB;
      o[q] = __ldcg(f + map.rep[k] * RB + b);
    }
  }
}

void launch_pix_gather(const uint8_t* frames, int64_t r0, int64_t r1, const PixRowMap& m, uint8_t* out,
                       cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(r1 - r0, (int64_t)sms * 8);
  if (grid > 0) k_pix_gather<<<grid, 256, 0, st>>>(frames, r0, r1, m.FB, m.RB, m.nused, m, out);
}

void launch_pixels(bool ext, const DS& S, const ObsArgs& a, cudaStream_t st) {
  if (a.n <= 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  switch ((ext ? 100 : 0) + a.tile_px) {
    case 7: launch_pixels_px<false, 7>(S, a, sms, st); break;
    case 10: launch_pixels_px<false, 10>(S, a, sms, st); break;
    case 16: launch_pixels_px<false, 16>(S, a, sms, st); break;
    case 107: launch_pixels_px<true, 7>(S, a, sms, st); break;
    case 110: launch_pixels_px<true, 10>(S, a, sms, st); break;
    case 116: launch_pixels_px<true, 16>(S, a, sms, st); break;
    default: break;   // gr_create admits 7, 10, 16 only
  }
}

}  // namespace gr
