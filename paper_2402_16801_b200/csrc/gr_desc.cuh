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

// obs._scaled_inventory in inventory_fields order (obs.py:87-122)
template <bool EXT>
__device__ __forceinline__ void inv_section(const InvSrc& s, float* v) {
  const float day = __fdiv_rn((float)(s.time % 300u), 300.0f);
  int k = 0;
  if (!EXT) {
    v[k++] = sq10(s.wood); v[k++] = sq10(s.stone); v[k++] = sq10(s.coal);
    v[k++] = sq10(s.iron); v[k++] = sq10(s.diamond); v[k++] = sq10(s.sapling);
    v[k++] = __fdiv_rn((float)s.pick, 4.0f); v[k++] = __fdiv_rn((float)s.sword, 4.0f);
    v[k++] = __fdiv_rn(s.health, 10.0f); v[k++] = __fdiv_rn(s.food, 10.0f);
    v[k++] = __fdiv_rn(s.drink, 10.0f); v[k++] = __fdiv_rn(s.energy, 10.0f);
    for (int d = 0; d < 4; ++d) v[k++] = s.facing == d ? 1.0f : 0.0f;
    v[k++] = day;
    v[k++] = s.sleeping ? 1.0f : 0.0f;
    return;
  }
  v[k++] = sq10(s.wood); v[k++] = sq10(s.stone); v[k++] = sq10(s.coal); v[k++] = sq10(s.iron);
  v[k++] = sq10(s.diamond); v[k++] = sq10(s.sapphire); v[k++] = sq10(s.ruby); v[k++] = sq10(s.sapling);
  v[k++] = sq10(s.torch); v[k++] = sq10(s.arrow);
  for (int p = 0; p < 6; ++p) v[k++] = sq10(s.potion[p]);
  v[k++] = __fdiv_rn((float)s.book, 2.0f);
  v[k++] = __fdiv_rn((float)s.pick, 4.0f);
  v[k++] = __fdiv_rn((float)s.sword, 4.0f);
  v[k++] = (float)s.sword_ench;
  v[k++] = (float)s.has_bow;
  for (int p = 0; p < 4; ++p) v[k++] = __fdiv_rn((float)s.armour[p], 2.0f);
  for (int p = 0; p < 4; ++p) v[k++] = (float)s.armour_ench[p];
  v[k++] = __fdiv_rn(s.health, 10.0f); v[k++] = __fdiv_rn(s.food, 10.0f);
  v[k++] = __fdiv_rn(s.drink, 10.0f); v[k++] = __fdiv_rn(s.energy, 10.0f);
  v[k++] = __fdiv_rn(s.mana, 10.0f); v[k++] = __fdiv_rn((float)s.xp, 10.0f);
  v[k++] = __fdiv_rn((float)s.dex, 10.0f); v[k++] = __fdiv_rn((float)s.str_, 10.0f);
  v[k++] = __fdiv_rn((float)s.intel, 10.0f);
  for (int d = 0; d < 4; ++d) v[k++] = s.facing == d ? 1.0f : 0.0f;
  v[k++] = day;
  v[k++] = (float)s.sleeping; v[k++] = (float)s.resting;
  v[k++] = (float)s.learned_fire; v[k++] = (float)s.learned_ice;
  v[k++] = __fdiv_rn((float)s.pf, 10.0f);
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
