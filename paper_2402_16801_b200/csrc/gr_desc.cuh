// gr_desc.cuh -- the per-env observation descriptor.
//
// The symbolic observation (obs.encode_symbolic_batch, obs.py:343-386) of
// one env is a pure function of: its view window of blocks/items (read by
// the writer kernel straight from the maps), the base light and sleeping
// flag (obs.light_window, :227-250), the creature/projectile cells painted
// into the view (obs._creature_channel_grid, :253-297) and the scaled
// inventory section (obs._scaled_inventory, :300-340).  Everything except
// the maps is folded into 64 words per env by whoever last wrote the env's
// state -- the step kernel (thread per env, from registers) or the install
// kernel (reset constants) -- so the bandwidth-bound writer kernel reads
// one contiguous 256-byte record per env instead of ~100 scattered fields.
#pragma once
#include <cstdint>
#include "gr_device.cuh"

namespace gr {

constexpr int DESC_WORDS = 64;
// word layout
constexpr int D_INV = 0;        // [0, 50): inventory section (float bits)
constexpr int D_BASE = 50;      // base light (float bits)
constexpr int D_POS = 51;       // (uint16)prow | (uint16)pcol << 16
constexpr int D_FLAGS = 52;     // pfloor | sleeping << 8 | torch-possible-on-this-floor << 9
constexpr int D_CRE = 53;       // 14 x u16 slot (cell << 8 | channel), 0xFFFF = none

// obs.daylight (obs.py:191-195): float32, numpy's SIMD sin
__device__ __forceinline__ float daylight(uint32_t time) {
  float phase = __fdiv_rn((float)(time % 300u), 300.0f);
  float m = phase < 0.5f ? phase : 0.5f;
  float arg = __fmul_rn(__fmul_rn(3.14159274101257324f, m), 2.0f);
  float lift = np_sincosf(arg, false);
  return __fadd_rn(0.150000006f, __fmul_rn(0.850000024f, lift > 0.0f ? lift : 0.0f));
}

// everything _scaled_inventory reads
struct InvSrc {
  uint8_t wood, stone, coal, iron, diamond, sapphire, ruby, sapling, torch, arrow, book;
  uint8_t potion[6];
  uint8_t pick, sword, sword_ench, has_bow, armour[4], armour_ench[4];
  uint8_t xp, dex, str_, intel, facing, sleeping, resting, learned_fire, learned_ice, pf, cleared, boss_vuln;
  float health, food, drink, energy, mana;
  uint32_t time;
};

__device__ __forceinline__ float sq10(uint8_t n) { return __fdiv_rn(__fsqrt_rn((float)n), 10.0f); }

// The observation values of small integer arguments come from one table,
// computed once per handle on the device by the exact expressions below
// (k_init_lut), so every entry is bit-identical to evaluating them: the
// descriptor writers then spend a load instead of an IEEE div / sqrt (20-40
// instructions each, ~1,000 per env in the step kernel) or numpy's sin.
constexpr int LUT_SQ10 = 0;          // sqrt(n) / 10, n < 256          (obs.py:98)
constexpr int LUT_DIV10 = 256;       // n / 10, n < 256                (obs.py:105-121)
constexpr int LUT_DAY = 512;         // (t % 300) / 300, t < 300       (obs.py:113)
constexpr int LUT_DAYLIGHT = 812;    // daylight(t), t < 300           (obs.py:191-195)
constexpr int LUT_N = 1112;

__device__ __forceinline__ float lut_value_exact(int k) {
  if (k < LUT_DIV10) return sq10((uint8_t)k);
  if (k < LUT_DAY) return __fdiv_rn((float)(k - LUT_DIV10), 10.0f);
  if (k < LUT_DAYLIGHT) return __fdiv_rn((float)(k - LUT_DAY), 300.0f);
  return daylight((uint32_t)(k - LUT_DAYLIGHT));
}

__device__ __forceinline__ float lut_daylight(const float* lut, uint32_t time) {
  return __ldg(lut + LUT_DAYLIGHT + time % 300u);
}

// obs._scaled_inventory in inventory_fields order (obs.py:87-122); the
// divisions by 2 and 4 are exact scalings
template <bool EXT>
__device__ __forceinline__ void inv_section(const InvSrc& s, float* v, const float* lut) {
  auto q = [&](uint8_t n) { return __ldg(lut + LUT_SQ10 + n); };
  auto d10 = [&](uint8_t n) { return __ldg(lut + LUT_DIV10 + n); };
  const float day = __ldg(lut + LUT_DAY + s.time % 300u);
  int k = 0;
  if (!EXT) {
    v[k++] = q(s.wood); v[k++] = q(s.stone); v[k++] = q(s.coal);
    v[k++] = q(s.iron); v[k++] = q(s.diamond); v[k++] = q(s.sapling);
    v[k++] = __fmul_rn((float)s.pick, 0.25f); v[k++] = __fmul_rn((float)s.sword, 0.25f);
    v[k++] = __fdiv_rn(s.health, 10.0f); v[k++] = __fdiv_rn(s.food, 10.0f);
    v[k++] = __fdiv_rn(s.drink, 10.0f); v[k++] = __fdiv_rn(s.energy, 10.0f);
    for (int d = 0; d < 4; ++d) v[k++] = s.facing == d ? 1.0f : 0.0f;
    v[k++] = day;
    v[k++] = s.sleeping ? 1.0f : 0.0f;
    return;
  }
  v[k++] = q(s.wood); v[k++] = q(s.stone); v[k++] = q(s.coal); v[k++] = q(s.iron);
  v[k++] = q(s.diamond); v[k++] = q(s.sapphire); v[k++] = q(s.ruby); v[k++] = q(s.sapling);
  v[k++] = q(s.torch); v[k++] = q(s.arrow);
  for (int p = 0; p < 6; ++p) v[k++] = q(s.potion[p]);
  v[k++] = __fmul_rn((float)s.book, 0.5f);
  v[k++] = __fmul_rn((float)s.pick, 0.25f);
  v[k++] = __fmul_rn((float)s.sword, 0.25f);
  v[k++] = (float)s.sword_ench;
  v[k++] = (float)s.has_bow;
  for (int p = 0; p < 4; ++p) v[k++] = __fmul_rn((float)s.armour[p], 0.5f);
  for (int p = 0; p < 4; ++p) v[k++] = (float)s.armour_ench[p];
  v[k++] = __fdiv_rn(s.health, 10.0f); v[k++] = __fdiv_rn(s.food, 10.0f);
  v[k++] = __fdiv_rn(s.drink, 10.0f); v[k++] = __fdiv_rn(s.energy, 10.0f);
  v[k++] = __fdiv_rn(s.mana, 10.0f); v[k++] = d10(s.xp);
  v[k++] = d10(s.dex); v[k++] = d10(s.str_);
  v[k++] = d10(s.intel);
  for (int d = 0; d < 4; ++d) v[k++] = s.facing == d ? 1.0f : 0.0f;
  v[k++] = day;
  v[k++] = (float)s.sleeping; v[k++] = (float)s.resting;
  v[k++] = (float)s.learned_fire; v[k++] = (float)s.learned_ice;
  v[k++] = d10(s.pf);
  v[k++] = (float)s.cleared;
  v[k++] = (float)s.boss_vuln;
}

// classic creature channel of a kind (obs.py:59-60): zombie 1, cow 2, skeleton 3
__device__ __forceinline__ int classic_channel(int kind) { return kind == 0 ? 1 : kind == 2 ? 2 : kind == 1 ? 3 : 0; }

// one painted slot: view cell (0xFF invisible or dead) and channel
template <bool EXT>
__device__ __forceinline__ uint32_t cre_slot(int r, int c, bool alive, int ch, int pr, int pc) {
  constexpr int VR = EXT ? 9 : 7, VC = EXT ? 11 : 9;
  const int wr = r - (pr - VR / 2), wc = c - (pc - VC / 2);
  if (!alive || wr < 0 || wr >= VR || wc < 0 || wc >= VC) return 0xFFFFu;
  return (uint32_t)((wr * VC + wc) << 8 | (ch & 0xFF));
}

}  // namespace gr
