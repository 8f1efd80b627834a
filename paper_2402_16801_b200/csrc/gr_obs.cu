// gr_obs.cu -- observation rendering: the symbolic one-hot vector
// (obs.encode_symbolic_batch, obs.py:191-386) and the RGB tile frame
// (tiles.render_tiles, tiles.py:85-186), one warp per environment.
//
// Per env the warp first builds the egocentric view in shared memory
// (block / item / creature channel and light per tile: obs.view_window,
// light_window, _creature_channel_grid) and the scaled inventory, then
// streams the row out: each lane writes consecutive 16-byte vectors, so a
// warp instruction covers 512 contiguous bytes and every obs byte is
// written exactly once (write-only, no read-for-ownership of the output).
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

constexpr int OBS_WARPS = 4;

template <bool EXT>
struct ViewSmem {
  uint8_t blk[OT<EXT>::T];     // block id (global)
  uint8_t itm[OT<EXT>::T];
  uint8_t cre[OT<EXT>::T];
  float light[OT<EXT>::T];
  float inv[OT<EXT>::NINV];
};


__constant__ int8_t C_CLASSIC_LOCAL[37] = {0, 0, 1, 2, 3, 4, 0, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 0, 0,
                                           0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};

// build the view of env i into v (whole warp); glow: batch-wide torch flag
template <bool EXT>
__device__ void build_view(const DS& S, int64_t i, bool glow, ViewSmem<EXT>& v) {
  using O = OT<EXT>;
  const int lane = threadIdx.x & 31;
  const int pf = EXT ? GR_AT(S, GR_F_PFLOOR, uint8_t, 0, i) : 0;
  const int pr = GR_AT(S, GR_F_PROW, int16_t, 0, i), pc = GR_AT(S, GR_F_PCOL, int16_t, 0, i);
  const uint32_t time = GR_AT(S, GR_F_TIME, uint32_t, 0, i);
  const bool sleeping = GR_AT(S, GR_F_SLEEPING, uint8_t, 0, i);
  const uint8_t* blk = (const uint8_t*)S.f[GR_F_BLOCKS] + ((size_t)i * O::F + pf) * O::HW;
  const uint8_t* itm = (const uint8_t*)S.f[GR_F_ITEMS] + ((size_t)i * O::F + pf) * O::HW;
  const float base = pf == 0 ? daylight(time) : C_FLOOR_AMB[pf];
  const int r0 = pr - O::VR / 2, c0 = pc - O::VC / 2;
  for (int t = lane; t < O::T; t += 32) {
    const int r = r0 + t / O::VC, c = c0 + t % O::VC;
    const bool inb = r >= 0 && r < O::H && c >= 0 && c < O::W;
    const uint8_t b = inb ? blk[r * O::W + c] : B_OOB;
    v.blk[t] = b;
    v.itm[t] = inb && EXT ? itm[r * O::W + c] : 0;
    v.cre[t] = 0;
    v.light[t] = base;
  }
  __syncwarp();
  if (EXT && glow) {
    // obs._torch_light over the (VR+6)x(VC+6) item window: each torch lights
    // view tiles within Chebyshev 3 at 1 - d/4
    constexpr int WR = O::VR + 6, WC = O::VC + 6;
    for (int t = lane; t < WR * WC; t += 32) {
      const int wr = t / WC - 3, wc = t % WC - 3;   // view coordinates
      const int r = r0 + wr, c = c0 + wc;
      if (r < 0 || r >= O::H || c < 0 || c >= O::W || itm[r * O::W + c] != I_TORCH) continue;
      for (int a = max(wr - 3, 0); a <= min(wr + 3, O::VR - 1); ++a)
        for (int b = max(wc - 3, 0); b <= min(wc + 3, O::VC - 1); ++b) {
          const int d = max(abs(a - wr), abs(b - wc));
          const float g = 1.0f - 0.25f * (float)d;   // exact: 1, .75, .5, .25
          atomicMax(reinterpret_cast<int*>(&v.light[a * O::VC + b]), __float_as_int(g));
        }
    }
    __syncwarp();
  }
  if (sleeping)
    for (int t = lane; t < O::T; t += 32) v.light[t] = 0.0f;
  // creature channels (obs.py:263-296): lane s loads slot s in parallel
  // (melee 0-2, ranged 3-4, passive 5-7, enemy proj 8-10, player proj 11-13);
  // the paint order -- later slots overwrite earlier ones -- is kept by
  // letting the highest slot index win each cell
  {
    constexpr int NSLOT = EXT ? 14 : 11;
    int cell = -1, ch = 0;
    if (lane < NSLOT) {
      int r = 0, c = 0, alive = 0;
      if (lane < 8) {
        const int cls = lane < 3 ? 0 : lane < 5 ? 1 : 2;
        const int l = lane - (cls == 0 ? 0 : cls == 1 ? 3 : 5), cap = cls == 1 ? 2 : 3;
        const int fp = cls == 0 ? GR_F_MEL_POS : cls == 1 ? GR_F_RAN_POS : GR_F_PAS_POS;
        const int fa = cls < 2 ? fp + 3 : fp + 2, ft = cls < 2 ? fp + 4 : fp + 3;
        const int li = pf * cap + l;
        r = GR_AT(S, fp, int16_t, 2 * li, i);
        c = GR_AT(S, fp, int16_t, 2 * li + 1, i);
        alive = GR_AT(S, fa, uint8_t, li, i);
        const int ty = GR_AT(S, ft, uint8_t, li, i);
        ch = EXT ? ty + 1 : (ty == 0 ? 1 : ty == 2 ? 2 : ty == 1 ? 3 : 0);
      } else {
        const bool ep = lane < 11;
        const int l = ep ? lane - 8 : lane - 11;
        const int fp = ep ? GR_F_EPROJ_POS : GR_F_PPROJ_POS;
        r = GR_AT(S, fp, int16_t, 2 * l, i);
        c = GR_AT(S, fp, int16_t, 2 * l + 1, i);
        alive = GR_AT(S, ep ? GR_F_EPROJ_ALIVE : GR_F_PPROJ_ALIVE, uint8_t, l, i);
        ch = EXT ? GR_AT(S, ep ? GR_F_EPROJ_TYPE : GR_F_PPROJ_TYPE, uint8_t, l, i) + 20 : 4;
      }
      const int wr = r - r0, wc = c - c0;
      if (alive && wr >= 0 && wr < O::VR && wc >= 0 && wc < O::VC) cell = wr * O::VC + wc;
    }
    // later slots win: a slot paints unless a higher slot targets the same cell
    bool win = cell >= 0;
    for (int s = 1; s < NSLOT; ++s) {
      const int oc = __shfl_down_sync(0xffffffffu, cell, s);
      if (lane + s < NSLOT && oc == cell) win = false;
    }
    if (win) v.cre[cell] = (uint8_t)ch;
  }
  // inventory section (obs._scaled_inventory, obs.py:300-340)
  for (int k = lane; k < O::NINV; k += 32) {
    auto sq = [](uint8_t n) { return __fdiv_rn(__fsqrt_rn((float)n), 10.0f); };
    auto u8 = [&](int fid, int c) { return GR_AT(S, fid, uint8_t, c, i); };
    auto f32 = [&](int fid) { return GR_AT(S, fid, float, 0, i); };
    const uint8_t facing = u8(GR_F_FACING, 0);
    const float day = __fdiv_rn((float)(time % 300u), 300.0f);
    float x = 0.0f;
    if (!EXT) {
      switch (k) {
        case 0: x = sq(u8(GR_F_INV_WOOD, 0)); break;
        case 1: x = sq(u8(GR_F_INV_STONE, 0)); break;
        case 2: x = sq(u8(GR_F_INV_COAL, 0)); break;
        case 3: x = sq(u8(GR_F_INV_IRON, 0)); break;
        case 4: x = sq(u8(GR_F_INV_DIAMOND, 0)); break;
        case 5: x = sq(u8(GR_F_INV_SAPLING, 0)); break;
        case 6: x = __fdiv_rn((float)u8(GR_F_PICK_TIER, 0), 4.0f); break;
        case 7: x = __fdiv_rn((float)u8(GR_F_SWORD_TIER, 0), 4.0f); break;
        case 8: x = __fdiv_rn(f32(GR_F_HEALTH), 10.0f); break;
        case 9: x = __fdiv_rn(f32(GR_F_FOOD), 10.0f); break;
        case 10: x = __fdiv_rn(f32(GR_F_DRINK), 10.0f); break;
        case 11: x = __fdiv_rn(f32(GR_F_ENERGY), 10.0f); break;
        case 12: case 13: case 14: case 15: x = facing == k - 12 ? 1.0f : 0.0f; break;
        case 16: x = day; break;
        default: x = sleeping ? 1.0f : 0.0f; break;
      }
    } else {
      if (k < 10) {
        const int fids[10] = {GR_F_INV_WOOD, GR_F_INV_STONE, GR_F_INV_COAL, GR_F_INV_IRON, GR_F_INV_DIAMOND,
                              GR_F_INV_SAPPHIRE, GR_F_INV_RUBY, GR_F_INV_SAPLING, GR_F_INV_TORCH, GR_F_INV_ARROW};
        x = sq(u8(fids[k], 0));
      } else if (k < 16) {
        x = sq(u8(GR_F_INV_POTION, k - 10));
      } else if (k == 16) {
        x = __fdiv_rn((float)u8(GR_F_INV_BOOK, 0), 2.0f);
      } else if (k == 17) {
        x = __fdiv_rn((float)u8(GR_F_PICK_TIER, 0), 4.0f);
      } else if (k == 18) {
        x = __fdiv_rn((float)u8(GR_F_SWORD_TIER, 0), 4.0f);
      } else if (k == 19) {
        x = (float)u8(GR_F_SWORD_ENCH, 0);
      } else if (k == 20) {
        x = (float)u8(GR_F_HAS_BOW, 0);
      } else if (k < 25) {
        x = __fdiv_rn((float)u8(GR_F_ARMOUR, k - 21), 2.0f);
      } else if (k < 29) {
        x = (float)u8(GR_F_ARMOUR_ENCH, k - 25);
      } else if (k < 34) {
        const int fids[5] = {GR_F_HEALTH, GR_F_FOOD, GR_F_DRINK, GR_F_ENERGY, GR_F_MANA};
        x = __fdiv_rn(f32(fids[k - 29]), 10.0f);
      } else if (k < 38) {
        const int fids[4] = {GR_F_XP, GR_F_DEX, GR_F_STR, GR_F_INTEL};
        x = __fdiv_rn((float)u8(fids[k - 34], 0), 10.0f);
      } else if (k < 42) {
        x = facing == k - 38 ? 1.0f : 0.0f;
      } else if (k == 42) {
        x = day;
      } else if (k == 43) {
        x = sleeping ? 1.0f : 0.0f;
      } else if (k == 44) {
        x = (float)u8(GR_F_RESTING, 0);
      } else if (k == 45) {
        x = (float)u8(GR_F_LEARNED_FIRE, 0);
      } else if (k == 46) {
        x = (float)u8(GR_F_LEARNED_ICE, 0);
      } else if (k == 47) {
        x = __fdiv_rn((float)pf, 10.0f);
      } else if (k == 48) {
        x = (float)u8(GR_F_FLOOR_CLEARED, pf);
      } else {
        x = (float)u8(GR_F_BOSS_VULN, 0);
      }
    }
    v.inv[k] = x;
  }
  __syncwarp();
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

template <bool EXT>
__global__ void __launch_bounds__(128) k_pixels(DS S, ObsArgs a) {
  using O = OT<EXT>;
  __shared__ ViewSmem<EXT> view;
  __shared__ PixSmem<EXT> pm;
  const int px = a.tile_px;
  const int side = EXT ? 2 : 0;
  const int FH = (O::VR + 2) * px, FW = (O::VC + side) * px;
  const int inset = max(1, px / 4);
  const int64_t frame = (int64_t)FH * FW * 3;
  const int64_t count = a.sel == 2 ? (int64_t)a.info->k_local : a.n;
  for (int64_t j = blockIdx.x; j < count; j += gridDim.x) {
    const int64_t i = a.sel == 2 ? (int64_t)a.list[j] : j;   // sel 2: reset envs only
    if (a.sel == 1 && a.done[i]) continue;                      // CTA-uniform env filter
    if (threadIdx.x < 32) {
      // render_tiles sees a one-env batch: glow iff this env's floor is dark
      const int pf = EXT ? GR_AT(S, GR_F_PFLOOR, uint8_t, 0, i) : 0;
      build_view<EXT>(S, i, EXT && C_FLOOR_AMB[pf] < 1.0f, view);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < O::T; t += blockDim.x) {
      const float l = view.light[t];
      const float sh = l < 0.0f ? 0.0f : (l > 1.0f ? 1.0f : l);
      const bool dark = l < 0.05f;
      const int b = view.blk[t];
      uint32_t rgb = 0;
      if (!dark)
        for (int k = 0; k < 3; ++k)
          rgb |= (uint32_t)(uint8_t)(int)__fmul_rn((float)C_PALETTE[b][k], sh) << (16 - 8 * k);
      pm.tile_rgb[t] = rgb;
      uint32_t ins = 0xFF000000u;
      if (!dark) {
        const int it = view.itm[t];
        if (it) ins = ((uint32_t)C_ITEMC[it][0] << 16) | ((uint32_t)C_ITEMC[it][1] << 8) | C_ITEMC[it][2];
        if (view.cre[t]) ins = creature_rgb(EXT, view.cre[t]);
      }
      if (t == (O::VR / 2) * O::VC + O::VC / 2) ins = 0xFA3C3Cu;   // the player
      pm.inset_rgb[t] = ins;
    }
    if (threadIdx.x == 0) {
      // vital bars (tiles.py:147-166) and gear panel (:169-186), float64
      const float str_ = (float)GR_AT(S, GR_F_STR, uint8_t, 0, i), dex = (float)GR_AT(S, GR_F_DEX, uint8_t, 0, i);
      const float intel = (float)GR_AT(S, GR_F_INTEL, uint8_t, 0, i);
      const double hmax = (double)__fadd_rn(9.0f, str_), fmax = (double)__fadd_rn(12.0f, dex);
      double st[5] = {(double)GR_AT(S, GR_F_HEALTH, float, 0, i) / hmax, (double)GR_AT(S, GR_F_FOOD, float, 0, i) / fmax,
                      (double)GR_AT(S, GR_F_DRINK, float, 0, i) / fmax, (double)GR_AT(S, GR_F_ENERGY, float, 0, i) / fmax,
                      EXT ? (double)GR_AT(S, GR_F_MANA, float, 0, i) / (double)__fadd_rn(16.0f, intel) : 0.0};
      const int width = O::VC * px - 2;
      for (int k = 0; k < 5; ++k) {
        const double f = st[k] < 0.0 ? 0.0 : (st[k] > 1.0 ? 1.0 : st[k]);
        pm.fill[k] = (int)rint(__dmul_rn(f, (double)width));
      }
      if (EXT) {
        const int arm = GR_AT(S, GR_F_ARMOUR, uint8_t, 0, i) + GR_AT(S, GR_F_ARMOUR, uint8_t, 1, i) +
                        GR_AT(S, GR_F_ARMOUR, uint8_t, 2, i) + GR_AT(S, GR_F_ARMOUR, uint8_t, 3, i);
        double g[7] = {(double)GR_AT(S, GR_F_SWORD_TIER, uint8_t, 0, i) / 4.0,
                       (double)GR_AT(S, GR_F_PICK_TIER, uint8_t, 0, i) / 4.0, (double)arm / 8.0,
                       (double)GR_AT(S, GR_F_XP, uint8_t, 0, i) / 8.0, (double)dex / 5.0, (double)str_ / 5.0,
                       (double)intel / 5.0};
        for (int k = 0; k < 7; ++k) {
          const double f = g[k] < 0.0 ? 0.0 : (g[k] > 1.0 ? 1.0 : g[k]);
          pm.fill[5 + k] = (int)rint(__dmul_rn(f, (double)(2 * px - 2)));
        }
      }
    }
    __syncthreads();
    uint8_t* out = (uint8_t*)a.out + (size_t)i * frame;
    const int ns = EXT ? 5 : 4;
    const int bar_h = max(2, (2 * px) / (ns + 1));
    const int y0 = O::VR * px;
    for (int64_t byte = threadIdx.x; byte < frame; byte += blockDim.x) {
      const int p = (int)(byte / 3), ch = (int)(byte % 3);
      const int y = p / FW, x = p % FW;
      uint32_t rgb = 0;
      if (y < O::VR * px && x < O::VC * px) {
        const int t = (y / px) * O::VC + x / px, iy = y % px, ix = x % px;
        rgb = pm.tile_rgb[t];
        if (iy >= inset && iy < px - inset && ix >= inset && ix < px - inset && pm.inset_rgb[t] != 0xFF000000u)
          rgb = pm.inset_rgb[t];
      } else if (y >= y0 && x < O::VC * px) {
        const int k = (y - y0 - 1) / bar_h, yy = (y - y0 - 1) % bar_h;
        if (y - y0 - 1 >= 0 && k < ns && yy < bar_h - 1 && x >= 1 && x < 1 + O::VC * px - 2) {
          rgb = x < 1 + pm.fill[k]
                    ? ((uint32_t)C_BARC[k][0] << 16) | ((uint32_t)C_BARC[k][1] << 8) | C_BARC[k][2]
                    : 0x1E1E1Eu;
        }
      } else if (EXT && x >= O::VC * px) {
        const int k = y / px, yy = y % px, xx = x - O::VC * px;
        if (k < 7 && k * px + px <= FH && yy >= 1 && yy < px - 1 && xx >= 1 && xx < 2 * px - 1) {
          rgb = xx < 1 + pm.fill[5 + k]
                    ? ((uint32_t)C_GEARC[k][0] << 16) | ((uint32_t)C_GEARC[k][1] << 8) | C_GEARC[k][2]
                    : 0x1E1E1Eu;
        }
      }
      out[byte] = (uint8_t)(rgb >> (16 - 8 * ch));
    }
    __syncthreads();
  }
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

template <bool EXT>
__host__ __device__ constexpr int stage_warps() { return EXT ? 2 : 8; }
// one stage = one whole row + up to 3 floats of alignment shift
template <bool EXT>
__host__ __device__ constexpr int stage_floats() { return EXT ? 8272 : 1352; }

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
        const uint32_t bc = EXT ? bq[q] : (uint32_t)C_CLASSIC_LOCAL[bq[q]];
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
    have = settle(jn, in, dwn, dn);
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
      // the next env's window loads overlap the drain of this row
      if (have)
        load_window<EXT>(S, in, __shfl_sync(0xffffffffu, dwn.y, D_POS / 2),
                         __shfl_sync(0xffffffffu, dwn.x, D_FLAGS / 2), lane, bqn, iqn);
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
    } else {
      if (have)
        load_window<EXT>(S, in, __shfl_sync(0xffffffffu, dwn.y, D_POS / 2),
                         __shfl_sync(0xffffffffu, dwn.x, D_FLAGS / 2), lane, bqn, iqn);
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

void launch_symbolic(bool ext, const DS& S, const ObsArgs& a, cudaStream_t st) {
  if (a.n <= 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (ext) {
    constexpr int NW = stage_warps<true>();
    const size_t smem = (size_t)NW * stage_floats<true>() * sizeof(float);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_symbolic_stage<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    const int per_sm = a.ctas_per_sm > 0 ? a.ctas_per_sm : 3;
    const int grid = (int)std::min<int64_t>((a.n + NW - 1) / NW, (int64_t)sms * per_sm);
    k_symbolic_stage<true><<<grid, NW * 32, smem, st>>>(S, a);
  } else {
    constexpr int NW = stage_warps<false>();
    const size_t smem = (size_t)NW * stage_floats<false>() * sizeof(float);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_symbolic_stage<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    const int grid = (int)std::min<int64_t>((a.n + NW - 1) / NW, (int64_t)sms * 4);
    k_symbolic_stage<false><<<grid, NW * 32, smem, st>>>(S, a);
  }
}

void launch_pixels(bool ext, const DS& S, const ObsArgs& a, cudaStream_t st) {
  if (a.n <= 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(a.n, (int64_t)sms * 16);
  if (ext) k_pixels<true><<<grid, 128, 0, st>>>(S, a);
  else k_pixels<false><<<grid, 128, 0, st>>>(S, a);
}

}  // namespace gr
