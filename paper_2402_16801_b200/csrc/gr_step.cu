// gr_step.cu -- the game-logic step kernel: one thread per environment.
//
// Restates engine.step_batch (engine.py:706-746) with its phases
//   player actions  engine.py:568-633   (move, DO, sleep, place, craft,
//                                        rest, ladders, bow, spells,
//                                        potions, books, level-ups)
//   projectiles     creatures.py:182-231
//   creatures       creatures.py:287-382
//   survival        engine.py:640-700
//   spawn/despawn   creatures.py:387-452  (+ boss waves :455-520)
//   plants          creatures.py:525-541
//   time / achievements / reward / done   engine.py:729-746
// followed by the batch bookkeeping of batch.batch_step (batch.py:206-209).
//
// Each thread loads its env's scalars and the *active floor's* creature
// lanes from the struct-of-arrays state (coalesced across the warp), runs
// the phases in registers, and stores everything back once.
//
// Batch-coupled corners of the reference reproduced exactly:
//  * creatures.py:312,345 decrement cooldowns on *dead* lanes too, but only
//    when some env of the batch has a live lane of that class.  The flag is
//    known only after every env's projectile phase, so the dead-lane
//    decrement is deferred: the lanes are marked in cd_pending and the
//    decrement is applied at the start of the next step (or at export) once
//    the batch-wide flag of this step is known.  Live lanes decrement
//    immediately (their own liveness makes the flag true).
//  * obs.py:236 torch glow is batch-coupled; this kernel publishes the
//    "some env stands on a dark floor" bit for the observation kernel.
#include <cstdint>
#include "gr_device.cuh"
#include "gr_state.cuh"
#include "gr_kernels.cuh"
#include "gr_desc.cuh"
#include "gr_tail.cuh"

namespace gr {

template <bool EXT>
struct TD {
  static constexpr int F = EXT ? 9 : 1, H = EXT ? 48 : 64, W = EXT ? 48 : 64;
  static constexpr int A = EXT ? 67 : 22, NA = EXT ? 43 : 17;
  static constexpr int HW = H * W;
};

// per-env working copy: scalars + the active floor's creature lanes.  k_step
// keeps one per thread in shared memory (Ctx-per-thread array, stride an odd
// number of words: bank-conflict free); members sorted by size so the struct
// packs with 4-byte alignment.  The env's map planes are at
// s_blk_base / s_itm_base + i * F * H * W (CTA-wide bases, set by the kernel).
struct Ctx {
  // 4-byte members
  uint32_t i;
  float health, food, drink, energy, mana;
  int lf;   // lanes of floor `lf`: class 0 melee (3), 1 ranged (2), 2 passive (3)
  float lhp[8];
  float ppdmg[3][3];
  float epdmg[3][3];
  uint32_t ach[3];
  uint32_t time;
  uint32_t key_lo;   // low word of rng_key: the only part the step uses (_kern.py:38-46)
  float boss_hp;
  uint32_t unlock[3];   // workspace (_kern.Workspace)
  float health0;
  uint32_t base;
  // 2-byte members
  int16_t prow, pcol;
  int16_t lr[8], lc[8];
  int16_t ppr[3], ppc[3];
  int16_t epr[3], epc[3];
  int16_t plr[10], plc[10];
  uint16_t plage[10];
  uint16_t visited, cleared;
  uint16_t torch;     // floors that may hold a torch (DS.torch_bits)
  uint16_t clocks[6];
  int16_t nr, nc;     // necro_pos
  // 1-byte members
  uint8_t pfloor, facing, xp, dex, str_, intel, sword_tier, pick_tier, has_bow, sword_ench, bow_ench;
  uint8_t armour[4], armour_ench[4];
  uint8_t learned_fire, learned_ice, sleeping, resting;
  uint8_t inv_wood, inv_stone, inv_coal, inv_iron, inv_diamond, inv_sapphire, inv_ruby, inv_sapling,
      inv_torch, inv_arrow, inv_book;
  uint8_t inv_potion[6];
  uint8_t lcd[8], lal[8], lty[8];
  uint8_t ppdir[3], pptype[3], ppttl[3], ppal[3];
  uint8_t epdir[3], eptype[3], epttl[3], epal[3];
  uint8_t plal[10];
  uint8_t boss_wave, boss_vuln, boss_timer;
  bool hurt;
  uint8_t act, pend, lflags;   // k_step's action-sorted phase: action in, pending cooldowns / lane flags out
  uint8_t pad_[5];
};
static_assert(alignof(Ctx) == 4, "Ctx packs at 4-byte alignment");
static_assert((sizeof(Ctx) / 4) % 2 == 1, "Ctx stride must be an odd number of words (shared-memory banks)");

// CTA-wide map plane bases (k_step / k_make_desc set them before any access)
__shared__ uint8_t* s_blk_base;
__shared__ uint8_t* s_itm_base;

// code-size knobs (dev A/B): GR_STEP_NI on the once-called phase / action
// handlers, GR_STEP_NI2 on the many-call-site lane helpers
#ifndef GR_STEP_NI
#define GR_STEP_NI
#endif
#ifndef GR_STEP_NI2
#define GR_STEP_NI2
#endif

// lane slot layout inside Ctx: melee 0..2, ranged 3..4, passive 5..7
__host__ __device__ constexpr int l0_of(int cls) { return cls == 0 ? 0 : cls == 1 ? 3 : 5; }
__host__ __device__ constexpr int cap_of(int cls) { return cls == 1 ? 2 : 3; }
#define L0 l0_of
#define LCAP cap_of

template <bool EXT>
__device__ __forceinline__ uint8_t gblock(const Ctx& e, int f, int r, int c) {
  using T = TD<EXT>;
  if (r < 0 || r >= T::H || c < 0 || c >= T::W) return B_OOB;
  return s_blk_base[(size_t)e.i * (T::F * T::HW) + f * T::HW + r * T::W + c];
}
template <bool EXT>
__device__ __forceinline__ uint8_t gitem(const Ctx& e, int f, int r, int c) {
  using T = TD<EXT>;
  if (r < 0 || r >= T::H || c < 0 || c >= T::W) return 0;
  return s_itm_base[(size_t)e.i * (T::F * T::HW) + f * T::HW + r * T::W + c];
}
template <bool EXT>
__device__ __forceinline__ void sblock(Ctx& e, int f, int r, int c, uint8_t v) {
  using T = TD<EXT>;
  s_blk_base[(size_t)e.i * (T::F * T::HW) + f * T::HW + r * T::W + c] = v;
}

template <bool EXT>
__device__ __forceinline__ void award(Ctx& e, int a) {
  if (a < TD<EXT>::A) e.unlock[a >> 5] |= 1u << (a & 31);
}

__device__ __forceinline__ float fmaxd(float a, float b) { return a > b ? a : b; }
__device__ __forceinline__ float fmind(float a, float b) { return a < b ? a : b; }
__device__ __forceinline__ float food_max(const Ctx& e) { return __fadd_rn(12.0f, (float)e.dex); }
__device__ __forceinline__ float health_max(const Ctx& e) { return __fadd_rn(9.0f, (float)e.str_); }
__device__ __forceinline__ float mana_max(const Ctx& e) { return __fadd_rn(16.0f, (float)e.intel); }
__device__ __forceinline__ uint8_t add_cap(uint8_t v, int d) { int x = v + d; return (uint8_t)(x < 99 ? x : 99); }
__device__ __forceinline__ float draw(const Ctx& e, int sub, int lane) { return u32f(e.base, (uint32_t)(sub * 64 + lane)); }

// _kern.hurt_player
__device__ __forceinline__ void hurt(Ctx& e, float amount) {
  if (!(amount > 0.0f)) return;
  e.health = __fsub_rn(e.health, amount);
  e.health = q1(fmaxd(e.health, 0.0f));
  e.hurt = true;
}

// _kern.player_defense
__device__ __forceinline__ void player_defense(const Ctx& e, float d[3]) {
  float phys = __fmul_rn((float)(e.armour[0] + e.armour[1] + e.armour[2] + e.armour[3]), 10.0f);
  int nf = 0, ni = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    nf += e.armour[k] > 0 && e.armour_ench[k] == 1;
    ni += e.armour[k] > 0 && e.armour_ench[k] == 2;
  }
  d[0] = fmind(phys, 80.0f);
  d[1] = fmind(__fmul_rn((float)nf, 20.0f), 80.0f);
  d[2] = fmind(__fmul_rn((float)ni, 20.0f), 80.0f);
}

// ----------------------------------------------------------- lane I/O
template <bool EXT>
__device__ void load_lanes(Ctx& e, const DS& S, int f) {
  e.lf = f;
  const int64_t i = e.i;
#pragma unroll
  for (int cls = 0; cls < 3; ++cls) {
    const int fp = cls == 0 ? GR_F_MEL_POS : cls == 1 ? GR_F_RAN_POS : GR_F_PAS_POS;
    const int cap = LCAP(cls);
#pragma unroll
    for (int l = 0; l < cap; ++l) {
      const int s = L0(cls) + l, lane = f * cap + l;
      e.lr[s] = GR_AT(S, fp, int16_t, lane * 2, i);
      e.lc[s] = GR_AT(S, fp, int16_t, lane * 2 + 1, i);
      e.lhp[s] = GR_AT(S, fp + 1, float, lane, i);
      if (cls < 2) {
        e.lcd[s] = GR_AT(S, fp + 2, uint8_t, lane, i);
        e.lal[s] = GR_AT(S, fp + 3, uint8_t, lane, i);
        e.lty[s] = GR_AT(S, fp + 4, uint8_t, lane, i);
      } else {
        e.lcd[s] = 0;
        e.lal[s] = GR_AT(S, fp + 2, uint8_t, lane, i);
        e.lty[s] = GR_AT(S, fp + 3, uint8_t, lane, i);
      }
    }
  }
}

template <bool EXT>
__device__ void store_lanes(const Ctx& e, const DS& S) {
  const int f = e.lf;
  const int64_t i = e.i;
#pragma unroll
  for (int cls = 0; cls < 3; ++cls) {
    const int fp = cls == 0 ? GR_F_MEL_POS : cls == 1 ? GR_F_RAN_POS : GR_F_PAS_POS;
    const int cap = LCAP(cls);
#pragma unroll
    for (int l = 0; l < cap; ++l) {
      const int s = L0(cls) + l, lane = f * cap + l;
      GR_AT(S, fp, int16_t, lane * 2, i) = e.lr[s];
      GR_AT(S, fp, int16_t, lane * 2 + 1, i) = e.lc[s];
      GR_AT(S, fp + 1, float, lane, i) = e.lhp[s];
      if (cls < 2) {
        GR_AT(S, fp + 2, uint8_t, lane, i) = e.lcd[s];
        GR_AT(S, fp + 3, uint8_t, lane, i) = e.lal[s];
        GR_AT(S, fp + 4, uint8_t, lane, i) = e.lty[s];
      } else {
        GR_AT(S, fp + 2, uint8_t, lane, i) = e.lal[s];
        GR_AT(S, fp + 3, uint8_t, lane, i) = e.lty[s];
      }
    }
  }
}

template <bool EXT>
__device__ void load_env(Ctx& e, const DS& S) {
  using T = TD<EXT>;
  const int64_t i = e.i;
#define LD(fid, T_, c) GR_AT(S, fid, T_, c, i)
  e.pfloor = EXT ? LD(GR_F_PFLOOR, uint8_t, 0) : 0;
  e.prow = LD(GR_F_PROW, int16_t, 0);
  e.pcol = LD(GR_F_PCOL, int16_t, 0);
  e.facing = LD(GR_F_FACING, uint8_t, 0);
  e.health = LD(GR_F_HEALTH, float, 0);
  e.food = LD(GR_F_FOOD, float, 0);
  e.drink = LD(GR_F_DRINK, float, 0);
  e.energy = LD(GR_F_ENERGY, float, 0);
  e.mana = LD(GR_F_MANA, float, 0);
  e.xp = LD(GR_F_XP, uint8_t, 0);
  e.dex = LD(GR_F_DEX, uint8_t, 0);
  e.str_ = LD(GR_F_STR, uint8_t, 0);
  e.intel = LD(GR_F_INTEL, uint8_t, 0);
  e.sword_tier = LD(GR_F_SWORD_TIER, uint8_t, 0);
  e.pick_tier = LD(GR_F_PICK_TIER, uint8_t, 0);
  e.has_bow = LD(GR_F_HAS_BOW, uint8_t, 0);
  e.sword_ench = LD(GR_F_SWORD_ENCH, uint8_t, 0);
  e.bow_ench = LD(GR_F_BOW_ENCH, uint8_t, 0);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    e.armour[k] = LD(GR_F_ARMOUR, uint8_t, k);
    e.armour_ench[k] = LD(GR_F_ARMOUR_ENCH, uint8_t, k);
  }
  e.learned_fire = LD(GR_F_LEARNED_FIRE, uint8_t, 0);
  e.learned_ice = LD(GR_F_LEARNED_ICE, uint8_t, 0);
  e.sleeping = LD(GR_F_SLEEPING, uint8_t, 0);
  e.resting = LD(GR_F_RESTING, uint8_t, 0);
  e.inv_wood = LD(GR_F_INV_WOOD, uint8_t, 0);
  e.inv_stone = LD(GR_F_INV_STONE, uint8_t, 0);
  e.inv_coal = LD(GR_F_INV_COAL, uint8_t, 0);
  e.inv_iron = LD(GR_F_INV_IRON, uint8_t, 0);
  e.inv_diamond = LD(GR_F_INV_DIAMOND, uint8_t, 0);
  e.inv_sapphire = LD(GR_F_INV_SAPPHIRE, uint8_t, 0);
  e.inv_ruby = LD(GR_F_INV_RUBY, uint8_t, 0);
  e.inv_sapling = LD(GR_F_INV_SAPLING, uint8_t, 0);
  e.inv_torch = LD(GR_F_INV_TORCH, uint8_t, 0);
  e.inv_arrow = LD(GR_F_INV_ARROW, uint8_t, 0);
  e.inv_book = LD(GR_F_INV_BOOK, uint8_t, 0);
#pragma unroll
  for (int k = 0; k < 6; ++k) e.inv_potion[k] = LD(GR_F_INV_POTION, uint8_t, k);
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    if (EXT) {
      e.ppr[l] = LD(GR_F_PPROJ_POS, int16_t, 2 * l);
      e.ppc[l] = LD(GR_F_PPROJ_POS, int16_t, 2 * l + 1);
      e.ppdir[l] = LD(GR_F_PPROJ_DIR, uint8_t, l);
      e.pptype[l] = LD(GR_F_PPROJ_TYPE, uint8_t, l);
      e.ppttl[l] = LD(GR_F_PPROJ_TTL, uint8_t, l);
      e.ppal[l] = LD(GR_F_PPROJ_ALIVE, uint8_t, l);
#pragma unroll
      for (int k = 0; k < 3; ++k) e.ppdmg[l][k] = LD(GR_F_PPROJ_DMG, float, 3 * l + k);
    }
    e.epr[l] = LD(GR_F_EPROJ_POS, int16_t, 2 * l);
    e.epc[l] = LD(GR_F_EPROJ_POS, int16_t, 2 * l + 1);
    e.epdir[l] = LD(GR_F_EPROJ_DIR, uint8_t, l);
    e.eptype[l] = LD(GR_F_EPROJ_TYPE, uint8_t, l);
    e.epttl[l] = LD(GR_F_EPROJ_TTL, uint8_t, l);
    e.epal[l] = LD(GR_F_EPROJ_ALIVE, uint8_t, l);
#pragma unroll
    for (int k = 0; k < 3; ++k) e.epdmg[l][k] = LD(GR_F_EPROJ_DMG, float, 3 * l + k);
  }
#pragma unroll
  for (int l = 0; l < 10; ++l) {
    e.plr[l] = LD(GR_F_PLANT_POS, int16_t, 2 * l);
    e.plc[l] = LD(GR_F_PLANT_POS, int16_t, 2 * l + 1);
    e.plage[l] = LD(GR_F_PLANT_AGE, uint16_t, l);
    e.plal[l] = LD(GR_F_PLANT_ALIVE, uint8_t, l);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) e.ach[k] = LD(GR_F_ACH, uint32_t, k);
  e.time = LD(GR_F_TIME, uint32_t, 0);
  e.key_lo = (uint32_t)LD(GR_F_RNG_KEY, uint64_t, 0);
  e.torch = EXT ? S.torch_bits[i] : 0;
  e.visited = 0;
  e.cleared = 0;
  if (EXT) {
    // accumulate in registers: 18 independent loads in flight, not 9 load ->
    // local-store round trips
    uint32_t vis = 0, clr = 0;
#pragma unroll
    for (int f = 0; f < T::F; ++f) {
      vis |= LD(GR_F_FLOORS_VISITED, uint8_t, f) ? 1u << f : 0u;
      clr |= LD(GR_F_FLOOR_CLEARED, uint8_t, f) ? 1u << f : 0u;
    }
    e.visited = (uint16_t)vis;
    e.cleared = (uint16_t)clr;
    e.boss_hp = LD(GR_F_BOSS_HP, float, 0);
    e.boss_wave = LD(GR_F_BOSS_WAVE, uint8_t, 0);
    e.boss_vuln = LD(GR_F_BOSS_VULN, uint8_t, 0);
    e.boss_timer = LD(GR_F_BOSS_TIMER, uint8_t, 0);
    e.nr = LD(GR_F_NECRO_POS, int16_t, 0);
    e.nc = LD(GR_F_NECRO_POS, int16_t, 1);
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) e.clocks[k] = LD(GR_F_CLOCKS, uint16_t, k);
#undef LD
}

template <bool EXT>
__device__ void store_env(const Ctx& e, const DS& S) {
  using T = TD<EXT>;
  const int64_t i = e.i;
#define ST(fid, T_, c, v) GR_AT(S, fid, T_, c, i) = (v)
  if (EXT) ST(GR_F_PFLOOR, uint8_t, 0, e.pfloor);
  ST(GR_F_PROW, int16_t, 0, e.prow);
  ST(GR_F_PCOL, int16_t, 0, e.pcol);
  ST(GR_F_FACING, uint8_t, 0, e.facing);
  ST(GR_F_HEALTH, float, 0, e.health);
  ST(GR_F_FOOD, float, 0, e.food);
  ST(GR_F_DRINK, float, 0, e.drink);
  ST(GR_F_ENERGY, float, 0, e.energy);
  ST(GR_F_MANA, float, 0, e.mana);
  ST(GR_F_XP, uint8_t, 0, e.xp);
  ST(GR_F_DEX, uint8_t, 0, e.dex);
  ST(GR_F_STR, uint8_t, 0, e.str_);
  ST(GR_F_INTEL, uint8_t, 0, e.intel);
  ST(GR_F_SWORD_TIER, uint8_t, 0, e.sword_tier);
  ST(GR_F_PICK_TIER, uint8_t, 0, e.pick_tier);
  ST(GR_F_HAS_BOW, uint8_t, 0, e.has_bow);
  ST(GR_F_SWORD_ENCH, uint8_t, 0, e.sword_ench);
  ST(GR_F_BOW_ENCH, uint8_t, 0, e.bow_ench);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    ST(GR_F_ARMOUR, uint8_t, k, e.armour[k]);
    ST(GR_F_ARMOUR_ENCH, uint8_t, k, e.armour_ench[k]);
  }
  ST(GR_F_LEARNED_FIRE, uint8_t, 0, e.learned_fire);
  ST(GR_F_LEARNED_ICE, uint8_t, 0, e.learned_ice);
  ST(GR_F_SLEEPING, uint8_t, 0, e.sleeping);
  ST(GR_F_RESTING, uint8_t, 0, e.resting);
  ST(GR_F_INV_WOOD, uint8_t, 0, e.inv_wood);
  ST(GR_F_INV_STONE, uint8_t, 0, e.inv_stone);
  ST(GR_F_INV_COAL, uint8_t, 0, e.inv_coal);
  ST(GR_F_INV_IRON, uint8_t, 0, e.inv_iron);
  ST(GR_F_INV_DIAMOND, uint8_t, 0, e.inv_diamond);
  ST(GR_F_INV_SAPPHIRE, uint8_t, 0, e.inv_sapphire);
  ST(GR_F_INV_RUBY, uint8_t, 0, e.inv_ruby);
  ST(GR_F_INV_SAPLING, uint8_t, 0, e.inv_sapling);
  ST(GR_F_INV_TORCH, uint8_t, 0, e.inv_torch);
  ST(GR_F_INV_ARROW, uint8_t, 0, e.inv_arrow);
  ST(GR_F_INV_BOOK, uint8_t, 0, e.inv_book);
#pragma unroll
  for (int k = 0; k < 6; ++k) ST(GR_F_INV_POTION, uint8_t, k, e.inv_potion[k]);
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    if (EXT) {
      ST(GR_F_PPROJ_POS, int16_t, 2 * l, e.ppr[l]);
      ST(GR_F_PPROJ_POS, int16_t, 2 * l + 1, e.ppc[l]);
      ST(GR_F_PPROJ_DIR, uint8_t, l, e.ppdir[l]);
      ST(GR_F_PPROJ_TYPE, uint8_t, l, e.pptype[l]);
      ST(GR_F_PPROJ_TTL, uint8_t, l, e.ppttl[l]);
      ST(GR_F_PPROJ_ALIVE, uint8_t, l, e.ppal[l]);
#pragma unroll
      for (int k = 0; k < 3; ++k) ST(GR_F_PPROJ_DMG, float, 3 * l + k, e.ppdmg[l][k]);
    }
    ST(GR_F_EPROJ_POS, int16_t, 2 * l, e.epr[l]);
    ST(GR_F_EPROJ_POS, int16_t, 2 * l + 1, e.epc[l]);
    ST(GR_F_EPROJ_DIR, uint8_t, l, e.epdir[l]);
    ST(GR_F_EPROJ_TYPE, uint8_t, l, e.eptype[l]);
    ST(GR_F_EPROJ_TTL, uint8_t, l, e.epttl[l]);
    ST(GR_F_EPROJ_ALIVE, uint8_t, l, e.epal[l]);
#pragma unroll
    for (int k = 0; k < 3; ++k) ST(GR_F_EPROJ_DMG, float, 3 * l + k, e.epdmg[l][k]);
  }
#pragma unroll
  for (int l = 0; l < 10; ++l) {
    ST(GR_F_PLANT_POS, int16_t, 2 * l, e.plr[l]);
    ST(GR_F_PLANT_POS, int16_t, 2 * l + 1, e.plc[l]);
    ST(GR_F_PLANT_AGE, uint16_t, l, e.plage[l]);
    ST(GR_F_PLANT_ALIVE, uint8_t, l, e.plal[l]);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) ST(GR_F_ACH, uint32_t, k, e.ach[k]);
  ST(GR_F_TIME, uint32_t, 0, e.time);
  if (EXT) {
    S.torch_bits[i] = e.torch;
#pragma unroll
    for (int f = 0; f < T::F; ++f) {
      ST(GR_F_FLOORS_VISITED, uint8_t, f, (uint8_t)((e.visited >> f) & 1));
      ST(GR_F_FLOOR_CLEARED, uint8_t, f, (uint8_t)((e.cleared >> f) & 1));
    }
    ST(GR_F_BOSS_HP, float, 0, e.boss_hp);
    ST(GR_F_BOSS_WAVE, uint8_t, 0, e.boss_wave);
    ST(GR_F_BOSS_VULN, uint8_t, 0, e.boss_vuln);
    ST(GR_F_BOSS_TIMER, uint8_t, 0, e.boss_timer);
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) ST(GR_F_CLOCKS, uint16_t, k, e.clocks[k]);
#undef ST
}

// ----------------------------------------------------- player actions

// engine._melee_damage_at (engine.py:91-100)
__device__ __forceinline__ void melee_damage(const Ctx& e, float d[3]) {
  float phys = q1(__fmul_rn(C_SWORD_BASE[e.sword_tier], __fadd_rn(0.5f, __fmul_rn((float)e.str_, 0.5f))));
  float elem = q1(__fmul_rn(phys, 0.5f));
  d[0] = phys;
  d[1] = e.sword_ench == 1 ? elem : 0.0f;
  d[2] = e.sword_ench == 2 ? elem : 0.0f;
}

__device__ __forceinline__ bool occupied(const Ctx& e, int r, int c) {
  bool o = false;
#pragma unroll
  for (int s = 0; s < 8; ++s) o |= e.lal[s] && e.lr[s] == r && e.lc[s] == c;
  return o;
}

// creatures.damage_creatures_at for one lane; `write` false reproduces the
// extended tier's discarded act0 copy (engine.py:573, creatures.py:90-94)
template <bool EXT>
GR_STEP_NI __device__ void damage_lane(Ctx& e, int s, const float d[3], bool write) {
  int kind = e.lty[s];
  float dealt = resolve(d[0], d[1], d[2], C_DEF[kind][0], C_DEF[kind][1], C_DEF[kind][2]);
  float hp = q1(__fsub_rn(e.lhp[s], dealt));
  bool died = hp <= 0.0f && e.lal[s] && dealt > 0.0f;
  if (write) {
    e.lhp[s] = hp;
    if (died) e.lal[s] = 0;
  }
  if (!died) return;
  award<EXT>(e, C_DEFEAT_ACH[kind]);
  float meat = C_EAT[kind];
  if (meat > 0.0f) {
    float fm = food_max(e);
    e.food = __fadd_rn(e.food, meat);
    e.food = q1(fmind(e.food, fm));
  }
}

// creatures._check_boss_death
template <bool EXT>
GR_STEP_NI __device__ void check_boss_death(Ctx& e) {
  if (!(e.boss_vuln && e.boss_hp <= 0.0f)) return;
  award<EXT>(e, 49);
  e.cleared |= 1u << 8;
  e.boss_vuln = 0;
  sblock<EXT>(e, 8, e.nr, e.nc, B_PATH);
}

// engine._open_chests (engine.py:240-272)
template <bool EXT>
GR_STEP_NI __device__ void open_chest(Ctx& e, const DS& S, int af, int tr, int tc) {
  const int64_t i = e.i;
  int lane = -1;
  for (int j = 0; j < 6; ++j) {
    uint8_t loot = GR_AT(S, GR_F_CHEST_LOOT, uint8_t, af * 6 + j, i);
    if (loot != LOOT_NOTHING && GR_AT(S, GR_F_CHEST_POS, int16_t, (af * 6 + j) * 2, i) == tr &&
        GR_AT(S, GR_F_CHEST_POS, int16_t, (af * 6 + j) * 2 + 1, i) == tc) {
      lane = j;
      break;
    }
  }
  if (lane < 0) return;
  int c = af * 6 + lane;
  uint8_t loot = GR_AT(S, GR_F_CHEST_LOOT, uint8_t, c, i);
  uint8_t qty = GR_AT(S, GR_F_CHEST_QTY, uint8_t, c, i);
  uint8_t aux = GR_AT(S, GR_F_CHEST_AUX, uint8_t, c, i);
  if (loot == LOOT_BOW) { e.has_bow = 1; award<EXT>(e, 52); }
  if (loot == LOOT_BOOK) e.inv_book = (uint8_t)(e.inv_book + qty);
  if (loot == LOOT_POTION) e.inv_potion[aux] = (uint8_t)(e.inv_potion[aux] + qty);
  if (loot == LOOT_ARROWS) e.inv_arrow = (uint8_t)(e.inv_arrow + qty);
  if (loot == LOOT_TORCHES) e.inv_torch = (uint8_t)(e.inv_torch + qty);
  if (e.inv_book > 99) e.inv_book = 99;
#pragma unroll
  for (int k = 0; k < 6; ++k) if (e.inv_potion[k] > 99) e.inv_potion[k] = 99;
  if (e.inv_arrow > 99) e.inv_arrow = 99;
  if (e.inv_torch > 99) e.inv_torch = 99;
  GR_AT(S, GR_F_CHEST_LOOT, uint8_t, c, i) = LOOT_NOTHING;
  sblock<EXT>(e, af, tr, tc, B_PATH);
  award<EXT>(e, 61);
}

// engine._do_interact (engine.py:143-237)
template <bool EXT>
GR_STEP_NI __device__ void do_interact(Ctx& e, const DS& S, int af) {
  int tr = e.prow + C_DIR[e.facing][0], tc = e.pcol + C_DIR[e.facing][1];
#pragma unroll
  for (int cls = 0; cls < 3; ++cls) {
    int hit = -1;
    for (int l = LCAP(cls) - 1; l >= 0; --l) {
      int s = L0(cls) + l;
      if (e.lal[s] && e.lr[s] == tr && e.lc[s] == tc) hit = s;
    }
    if (hit >= 0) {
      float d[3];
      melee_damage(e, d);
      damage_lane<EXT>(e, hit, d, !EXT);
      return;
    }
  }
  uint8_t tb = gblock<EXT>(e, af, tr, tc);
  if (tb == B_TREE || tb == B_FIRE_TREE || tb == B_ICE_SHRUB) {
    e.inv_wood = add_cap(e.inv_wood, 1);
    award<EXT>(e, 0);
  } else if (tb == B_GRASS) {
    if (draw(e, 1, 0) < 0.1f) {
      e.inv_sapling = add_cap(e.inv_sapling, 1);
      award<EXT>(e, 3);
    }
  } else if (tb == B_WATER || tb == B_FOUNTAIN) {
    e.drink = q1(fmind(__fadd_rn(e.drink, 1.0f), food_max(e)));
    award<EXT>(e, 4);
    if (tb == B_FOUNTAIN) e.mana = q1(fmind(__fadd_rn(e.mana, 1.0f), mana_max(e)));
  } else if (tb == B_RIPE_PLANT) {
    e.food = q1(fmind(__fadd_rn(e.food, 4.0f), food_max(e)));
    award<EXT>(e, 11);
    sblock<EXT>(e, af, tr, tc, B_PLANT);
#pragma unroll
    for (int l = 0; l < 10; ++l)
      if (e.plal[l] && e.plr[l] == tr && e.plc[l] == tc) e.plage[l] = 0;
  } else {
    // MINEABLE (constants.py:450-458)
    int req = -1, ach = -1;
    uint8_t* inv = nullptr;
    switch (tb) {
      case B_STONE: req = 1; ach = 9; inv = &e.inv_stone; break;
      case B_COAL: req = 1; ach = 17; inv = &e.inv_coal; break;
      case B_STALAGMITE: req = 1; inv = &e.inv_stone; break;
      case B_IRON: req = 2; ach = 18; inv = &e.inv_iron; break;
      case B_DIAMOND: req = 3; ach = 19; inv = &e.inv_diamond; break;
      case B_SAPPHIRE: req = 3; ach = 54; inv = &e.inv_sapphire; break;
      case B_RUBY: req = 4; ach = 59; inv = &e.inv_ruby; break;
      default: break;
    }
    if (req >= 0 && e.pick_tier >= req) {
      *inv = add_cap(*inv, 1);
      sblock<EXT>(e, af, tr, tc, B_PATH);
      if (ach >= 0) award<EXT>(e, ach);
    } else if (EXT && tb == B_CHEST) {
      open_chest<EXT>(e, S, af, tr, tc);
    } else if (EXT && tb == B_NECROMANCER_VULN && e.boss_vuln) {
      float d[3];
      melee_damage(e, d);
      float dealt = resolve(d[0], d[1], d[2], 0.0f, 0.0f, 0.0f);
      e.boss_hp = __fsub_rn(e.boss_hp, dealt);
      award<EXT>(e, 48);
      check_boss_death<EXT>(e);
    }
  }
}

// engine._place_actions (engine.py:275-336)
template <bool EXT>
GR_STEP_NI __device__ void place_action(Ctx& e, int a, int af) {
  using T = TD<EXT>;
  int tr = e.prow + C_DIR[e.facing][0], tc = e.pcol + C_DIR[e.facing][1];
  uint8_t tb = gblock<EXT>(e, af, tr, tc);
  uint8_t ti = gitem<EXT>(e, af, tr, tc);
  bool open = ti == I_EMPTY && !occupied(e, tr, tc);
  if (!open) return;
  if (a == 7 && e.inv_stone > 0 && in_set(PLACE_STONE_SET, tb)) {
    sblock<EXT>(e, af, tr, tc, B_STONE); award<EXT>(e, 10); e.inv_stone -= 1;
  } else if (a == 8 && e.inv_wood > 0 && in_set(PLACE_SOLID_SET, tb)) {
    sblock<EXT>(e, af, tr, tc, B_TABLE); award<EXT>(e, 1); e.inv_wood -= 1;
  } else if (a == 9 && e.inv_stone > 0 && in_set(PLACE_SOLID_SET, tb)) {
    sblock<EXT>(e, af, tr, tc, B_FURNACE); award<EXT>(e, 16); e.inv_stone -= 1;
  } else if (a == 10 && e.inv_sapling > 0 && tb == B_GRASS && af == 0) {
    int slot = -1;
    for (int l = 9; l >= 0; --l) if (!e.plal[l]) slot = l;
    if (slot >= 0) {
      sblock<EXT>(e, af, tr, tc, B_PLANT); award<EXT>(e, 7);
      e.plr[slot] = (int16_t)tr; e.plc[slot] = (int16_t)tc;
      e.plage[slot] = 0; e.plal[slot] = 1;
      e.inv_sapling -= 1;
    }
  } else if (EXT && a == 28 && e.inv_torch > 0 && in_set(WALK_SET, tb)) {
    s_itm_base[(size_t)e.i * (T::F * T::HW) + af * T::HW + tr * T::W + tc] = I_TORCH;
    e.torch |= (uint16_t)(1u << af);
    e.inv_torch -= 1;
    award<EXT>(e, 24);
  }
}

// engine._craft_actions (engine.py:346-457)
template <bool EXT>
GR_STEP_NI __device__ void craft_action(Ctx& e, int a, int af) {
  bool near_table = false, near_furnace = false, near_fire = false, near_ice = false;
#pragma unroll
  for (int dr = -1; dr <= 1; ++dr)
#pragma unroll
    for (int dc = -1; dc <= 1; ++dc) {
      uint8_t b = gblock<EXT>(e, af, e.prow + dr, e.pcol + dc);
      near_table |= b == B_TABLE;
      near_furnace |= b == B_FURNACE;
      near_fire |= b == B_ENCHANT_FIRE;
      near_ice |= b == B_ENCHANT_ICE;
    }
  // the eight tool recipes (engine.py:54-77)
  int pick = -1, level = 0, w = 0, st = 0, co = 0, ir = 0, di = 0, fur = 0, ach = 0;
  switch (a) {
    case 11: pick = 1; level = 1; w = 1; ach = 5; break;
    case 12: pick = 1; level = 2; w = 1; st = 1; ach = 13; break;
    case 13: pick = 1; level = 3; w = 1; co = 1; ir = 1; fur = 1; ach = 20; break;
    case 20: pick = 1; level = 4; w = 1; di = 2; ach = 60; break;
    case 14: pick = 0; level = 1; w = 1; ach = 6; break;
    case 15: pick = 0; level = 2; w = 1; st = 1; ach = 14; break;
    case 16: pick = 0; level = 3; w = 1; co = 1; ir = 1; fur = 1; ach = 21; break;
    case 21: pick = 0; level = 4; w = 1; di = 2; ach = 25; break;
    default: break;
  }
  if (pick >= 0) {
    uint8_t& tool = pick ? e.pick_tier : e.sword_tier;
    if (tool < level && near_table && (!fur || near_furnace) && e.inv_wood >= w && e.inv_stone >= st &&
        e.inv_coal >= co && e.inv_iron >= ir && e.inv_diamond >= di) {
      e.inv_wood -= w; e.inv_stone -= st; e.inv_coal -= co; e.inv_iron -= ir; e.inv_diamond -= di;
      tool = (uint8_t)level;
      award<EXT>(e, ach);
    }
    return;
  }
  if (!EXT) return;
  if (a == 25) {
    if (near_table && e.inv_wood >= 1 && e.inv_stone >= 1) {
      e.inv_wood -= 1; e.inv_stone -= 1;
      e.inv_arrow = add_cap(e.inv_arrow, 2);
      award<EXT>(e, 22);
    }
  } else if (a == 38) {
    if (e.inv_wood >= 1 && e.inv_coal >= 1) {
      e.inv_wood -= 1; e.inv_coal -= 1;
      e.inv_torch = add_cap(e.inv_torch, 4);
      award<EXT>(e, 23);
    }
  } else if (a == 22 || a == 23) {
    int need = a == 22 ? 1 : 2;
    bool ok = a == 22 ? (near_table && near_furnace && e.inv_iron >= 2 && e.inv_coal >= 1)
                      : (near_table && e.inv_diamond >= 2);
    if (ok) {
      int slot = 0;
#pragma unroll
      for (int k = 1; k < 4; ++k) if (e.armour[k] < e.armour[slot]) slot = k;
      if (e.armour[slot] < need) {
        e.armour[slot] = (uint8_t)need;
        if (a == 22) { e.inv_iron -= 2; e.inv_coal -= 1; award<EXT>(e, 26); }
        else { e.inv_diamond -= 2; award<EXT>(e, 27); }
      }
    }
  } else if (a == 36 || a == 37 || a == 42) {
    bool can_fire = near_fire && e.inv_ruby >= 1 && e.mana >= 2.0f;
    bool can_ice = near_ice && e.inv_sapphire >= 1 && e.mana >= 2.0f;
    uint8_t* slot = nullptr;
    if (a == 36 && e.sword_tier > 0) slot = &e.sword_ench;
    if (a == 42 && e.has_bow) slot = &e.bow_ench;
    if (a == 37) {
      for (int k = 3; k >= 0; --k) if (e.armour[k] > 0 && e.armour_ench[k] == 0) slot = &e.armour_ench[k];
    }
    if (slot && (can_fire || can_ice)) {
      if (can_fire) { *slot = 1; e.inv_ruby -= 1; }
      else { *slot = 2; e.inv_sapphire -= 1; }
      e.mana = __fsub_rn(e.mana, 2.0f);
      if (a == 36) award<EXT>(e, 63);
      if (a == 37) award<EXT>(e, 64);
    }
  }
}

// engine._spawn_player_projectile
__device__ __forceinline__ bool spawn_pproj(Ctx& e, int kind, float d0, float d1, float d2) {
  int slot = -1;
  for (int l = 2; l >= 0; --l) if (!e.ppal[l]) slot = l;
  if (slot < 0) return false;
  e.ppr[slot] = e.prow; e.ppc[slot] = e.pcol;
  e.ppdir[slot] = e.facing; e.pptype[slot] = (uint8_t)kind; e.ppttl[slot] = 6;
  e.ppdmg[slot][0] = d0; e.ppdmg[slot][1] = d1; e.ppdmg[slot][2] = d2;
  e.ppal[slot] = 1;
  return true;
}

// engine._ladder_moves (engine.py:533-565)
template <bool EXT>
GR_STEP_NI __device__ void ladder_move(Ctx& e, const DS& S, int a) {
  using T = TD<EXT>;
  uint8_t here = gitem<EXT>(e, e.pfloor, e.prow, e.pcol);
  bool down = a == 18 && here == I_LADDER_DOWN && e.pfloor + 1 < T::F;
  bool up = a == 19 && here == I_LADDER_UP && e.pfloor > 0;
  if (!down && !up) return;
  int nf = e.pfloor + (down ? 1 : -1);
  e.pfloor = (uint8_t)nf;
  const int fid = down ? GR_F_LADDER_UP : GR_F_LADDER_DOWN;
  e.prow = GR_AT(S, fid, int16_t, nf * 2, e.i);
  e.pcol = GR_AT(S, fid, int16_t, nf * 2 + 1, e.i);
#pragma unroll
  for (int l = 0; l < 3; ++l) { e.ppal[l] = 0; e.epal[l] = 0; }
  if (!((e.visited >> nf) & 1)) {
    e.visited |= 1u << nf;
    uint8_t x = (uint8_t)(e.xp + 1);
    e.xp = x < 255 ? x : 255;
    if (C_ENTER_ACH[nf] != 255) award<EXT>(e, C_ENTER_ACH[nf]);
  }
}

template <bool EXT>
__device__ void player_actions(Ctx& e, const DS& S, int action) {
  int eff = (e.sleeping || e.resting) ? 0 : action;
  int af = e.pfloor;
  if (eff >= 1 && eff <= 4) {
    e.facing = (uint8_t)(eff - 1);
    int tr = e.prow + C_DIR[e.facing][0], tc = e.pcol + C_DIR[e.facing][1];
    uint8_t tb = gblock<EXT>(e, af, tr, tc);
    if (in_set(WALK_SET, tb) && !occupied(e, tr, tc)) { e.prow = (int16_t)tr; e.pcol = (int16_t)tc; }
    return;
  }
  if (eff == 5) { do_interact<EXT>(e, S, af); return; }
  if (eff == 6) {
    if (!e.sleeping && e.energy < food_max(e)) e.sleeping = 1;
    return;
  }
  if ((eff >= 7 && eff <= 10) || (EXT && eff == 28)) { place_action<EXT>(e, eff, af); return; }
  if ((eff >= 11 && eff <= 16) ||
      (EXT && (eff == 20 || eff == 21 || eff == 22 || eff == 23 || eff == 25 || eff == 38 || eff == 36 ||
               eff == 37 || eff == 42))) {
    craft_action<EXT>(e, eff, af);
    return;
  }
  if (!EXT) return;
  if (eff == 17) { e.resting = 1; return; }
  if (eff == 18 || eff == 19) { ladder_move<EXT>(e, S, eff); return; }
  if (eff == 24) {
    if (e.has_bow && e.inv_arrow > 0) {
      float phys = q1(__fadd_rn(3.0f, (float)e.dex));
      float elem = q1(__fmul_rn(phys, 0.5f));
      if (spawn_pproj(e, 0, phys, e.bow_ench == 1 ? elem : 0.0f, e.bow_ench == 2 ? elem : 0.0f)) {
        e.inv_arrow -= 1;
        award<EXT>(e, 53);
      }
    }
    return;
  }
  if (eff == 26 || eff == 27) {
    bool learned = eff == 26 ? e.learned_fire : e.learned_ice;
    if (learned && e.mana >= 2.0f) {
      float v = __fadd_rn(6.0f, (float)e.intel);
      if (spawn_pproj(e, eff == 26 ? 1 : 2, 0.0f, eff == 26 ? v : 0.0f, eff == 27 ? v : 0.0f)) {
        e.mana = q1(__fsub_rn(e.mana, 2.0f));
        award<EXT>(e, eff == 26 ? 56 : 58);
      }
    }
    return;
  }
  // engine._consumables (engine.py:473-517)
  if (eff >= 29 && eff <= 34) {
    int color = eff - 29;
    if (e.inv_potion[color] > 0) {
      e.inv_potion[color] -= 1;
      int effect = GR_AT(S, GR_F_POTION_MAP, uint8_t, color, e.i);
      switch (effect) {
        case 0: e.health = q1(fmind(__fadd_rn(e.health, 8.0f), health_max(e))); break;
        case 1: e.mana = q1(fmind(__fadd_rn(e.mana, 8.0f), mana_max(e))); break;
        case 2: e.energy = q1(fmind(__fadd_rn(e.energy, 8.0f), food_max(e))); break;
        case 3: hurt(e, 3.0f); break;
        case 4: e.mana = q1(fmaxd(__fsub_rn(e.mana, 3.0f), 0.0f)); break;
        default:
          e.food = q1(fmind(__fadd_rn(e.food, 4.0f), food_max(e)));
          e.drink = q1(fmind(__fadd_rn(e.drink, 4.0f), food_max(e)));
          break;
      }
      award<EXT>(e, 62);
    }
    return;
  }
  if (eff == 35) {
    if (e.inv_book > 0) {
      bool lf = !e.learned_fire, li = e.learned_fire && !e.learned_ice;
      if (lf || li) e.inv_book -= 1;
      if (lf) { e.learned_fire = 1; award<EXT>(e, 55); }
      if (li) { e.learned_ice = 1; award<EXT>(e, 57); }
    }
    return;
  }
  // engine._level_ups (engine.py:520-530)
  if (eff >= 39 && eff <= 41 && e.xp >= 1) {
    uint8_t& attr = eff == 39 ? e.dex : eff == 40 ? e.str_ : e.intel;
    if (attr < 5) { attr += 1; e.xp -= 1; }
  }
}

// ---------------------------------------------------------- projectiles
template <bool EXT>
GR_STEP_NI __device__ void advance_projectiles(Ctx& e) {
  const int af = e.pfloor;
  if (EXT) {
#pragma unroll
    for (int l = 0; l < 3; ++l)
      if (e.ppal[l]) { e.ppr[l] += C_DIR[e.ppdir[l]][0]; e.ppc[l] += C_DIR[e.ppdir[l]][1]; }
#pragma unroll 1
    for (int l = 0; l < 3; ++l) {
      if (!e.ppal[l]) continue;
      int r = e.ppr[l], c = e.ppc[l];
      bool live = true;
#pragma unroll 1
      for (int cls = 0; cls < 3; ++cls) {
        if (!live) break;
        int hit = -1;
#pragma unroll 1
        for (int k = LCAP(cls) - 1; k >= 0; --k) {
          int s = L0(cls) + k;
          if (e.lal[s] && e.lr[s] == r && e.lc[s] == c) hit = s;
        }
        if (hit >= 0) {
          damage_lane<EXT>(e, hit, e.ppdmg[l], true);
          live = false;
        }
      }
      if (live && e.boss_vuln && r == e.nr && c == e.nc) {
        e.boss_hp = __fsub_rn(e.boss_hp, resolve(e.ppdmg[l][0], e.ppdmg[l][1], e.ppdmg[l][2], 0.f, 0.f, 0.f));
        award<EXT>(e, 48);
        check_boss_death<EXT>(e);
      }
      uint8_t b = gblock<EXT>(e, af, r, c);
      bool stopped = !live || in_set(PROJ_STOP_SET, b) || e.ppttl[l] <= 1;
      e.ppttl[l] -= 1;
      if (stopped) e.ppal[l] = 0;
    }
  }
  if (!(e.epal[0] | e.epal[1] | e.epal[2])) return;
  bool at[3];
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    if (e.epal[l]) { e.epr[l] += C_DIR[e.epdir[l]][0]; e.epc[l] += C_DIR[e.epdir[l]][1]; }
    at[l] = e.epal[l] && e.epr[l] == e.prow && e.epc[l] == e.pcol;
  }
  if (at[0] || at[1] || at[2]) {
    float pd[3], d[3];
    player_defense(e, pd);
#pragma unroll
    for (int l = 0; l < 3; ++l)
      d[l] = at[l] ? resolve(e.epdmg[l][0], e.epdmg[l][1], e.epdmg[l][2], pd[0], pd[1], pd[2]) : 0.0f;
    hurt(e, __fadd_rn(__fadd_rn(d[0], d[1]), d[2]));
#pragma unroll
    for (int l = 0; l < 3; ++l) if (at[l]) e.epal[l] = 0;
  }
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    if (!e.epal[l]) continue;
    if (in_set(PROJ_STOP_SET, gblock<EXT>(e, af, e.epr[l], e.epc[l]))) { e.epal[l] = 0; continue; }
    e.epttl[l] -= 1;
    if (e.epttl[l] == 0) e.epal[l] = 0;
  }
}

// ------------------------------------------------------------ creatures
__device__ __forceinline__ int isgn(int x) { return (x > 0) - (x < 0); }

template <bool EXT>
__device__ __forceinline__ uint64_t walk_set_of(const Ctx& e, int s) {
  if (!EXT) return coll_set(0);
  return coll_set(C_COLL[e.lty[s]]);
}

template <bool EXT>
GR_STEP_NI2 __device__ void move_lane(Ctx& e, int s, int sr, int sc) {
  int tr = e.lr[s] + sr, tc = e.lc[s] + sc;
  if (in_set(walk_set_of<EXT>(e, s), gblock<EXT>(e, e.lf, tr, tc)) && !(tr == e.prow && tc == e.pcol)) {
    e.lr[s] = (int16_t)tr; e.lc[s] = (int16_t)tc;
  }
}

template <bool EXT>
GR_STEP_NI2 __device__ void chase_move(Ctx& e, int s, int dr, int dc) {
  int sr = isgn(dr), sc = isgn(dc);
  bool row_first = abs(dr) >= abs(dc);
  int pr = row_first ? sr : 0, pc = row_first ? 0 : sc;
  int qr = sr - pr, qc = sc - pc;
  uint64_t ws = walk_set_of<EXT>(e, s);
  int t1r = e.lr[s] + pr, t1c = e.lc[s] + pc, t2r = e.lr[s] + qr, t2c = e.lc[s] + qc;
  bool ok1 = in_set(ws, gblock<EXT>(e, e.lf, t1r, t1c)) && !(t1r == e.prow && t1c == e.pcol);
  bool ok2 = in_set(ws, gblock<EXT>(e, e.lf, t2r, t2c)) && !(t2r == e.prow && t2c == e.pcol);
  if (ok1) { e.lr[s] = (int16_t)t1r; e.lc[s] = (int16_t)t1c; }
  else if (ok2) { e.lr[s] = (int16_t)t2r; e.lc[s] = (int16_t)t2c; }
}

// creatures.creatures_act (creatures.py:287-382).  Dead-lane cooldown
// decrements are recorded in *pending (see file header).
template <bool EXT>
__device__ void creatures_act(Ctx& e, uint8_t* pending) {
  // melee
  {
    int dr[3], dc[3], cb[3];
    bool adj[3], attack[3];
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      dr[l] = e.prow - e.lr[l]; dc[l] = e.pcol - e.lc[l];
      cb[l] = max(abs(dr[l]), abs(dc[l]));
      adj[l] = abs(dr[l]) + abs(dc[l]) == 1;
      attack[l] = e.lal[l] && adj[l] && e.lcd[l] == 0;
    }
    if (attack[0] || attack[1] || attack[2]) {
      float d[3];
      if (!EXT) {
#pragma unroll
        for (int l = 0; l < 3; ++l) d[l] = attack[l] ? C_DEALT_BARE[e.lty[l]] : 0.0f;
      } else {
        float pd[3];
        player_defense(e, pd);
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          int k = e.lty[l];
          d[l] = attack[l] ? resolve(C_DMG[k][0], C_DMG[k][1], C_DMG[k][2], pd[0], pd[1], pd[2]) : 0.0f;
        }
      }
      hurt(e, __fadd_rn(__fadd_rn(d[0], d[1]), d[2]));
    }
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      if (e.lal[l]) {
        if (e.lcd[l] > 0) e.lcd[l] -= 1;
      } else if (e.lcd[l] > 0) {
        *pending |= (uint8_t)(1u << l);
      }
      if (attack[l]) e.lcd[l] = 2;
    }
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      if (!e.lal[l] || adj[l]) continue;
      if (cb[l] <= 6) {
        chase_move<EXT>(e, l, dr[l], dc[l]);
      } else {
        float u = draw(e, 2, l);
        if (u < 0.25f) {
          int d = min((int)__fmul_rn(u, 16.0f) % 4, 3);
          move_lane<EXT>(e, l, C_DIR[d][0], C_DIR[d][1]);
        }
      }
    }
  }
  // ranged
  {
    int dr[2], dc[2], cb[2];
    bool shoot[2];
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      const int s = 3 + l;
      dr[l] = e.prow - e.lr[s]; dc[l] = e.pcol - e.lc[s];
      cb[l] = max(abs(dr[l]), abs(dc[l]));
      bool aligned = (dr[l] == 0 || dc[l] == 0) && cb[l] >= 1;
      shoot[l] = e.lal[s] && aligned && cb[l] <= 5 && e.lcd[s] == 0;
      if (shoot[l]) {
        int sr = isgn(dr[l]), sc = isgn(dc[l]);
        for (int k = 1; k < 5 && k < cb[l]; ++k)
          if (in_set(PROJ_STOP_SET, gblock<EXT>(e, e.lf, e.lr[s] + sr * k, e.lc[s] + sc * k))) { shoot[l] = false; break; }
      }
    }
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      const int s = 3 + l;
      if (e.lal[s]) {
        if (e.lcd[s] > 0) e.lcd[s] -= 1;
      } else if (e.lcd[s] > 0) {
        *pending |= (uint8_t)(1u << (3 + l));
      }
      if (shoot[l]) e.lcd[s] = 6;
    }
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      if (!shoot[l]) continue;
      const int s = 3 + l;
      int slot = -1;
      for (int k = 2; k >= 0; --k) if (!e.epal[k]) slot = k;
      if (slot < 0) continue;
      int kind = e.lty[s];
      e.epr[slot] = e.lr[s]; e.epc[slot] = e.lc[s];
      e.epdir[slot] = dr[l] == 0 ? (dc[l] > 0 ? 1 : 0) : (dr[l] > 0 ? 3 : 2);
      e.eptype[slot] = C_RANGED_PROJ[kind];
      e.epttl[slot] = 6;
      e.epdmg[slot][0] = C_DMG[kind][0]; e.epdmg[slot][1] = C_DMG[kind][1]; e.epdmg[slot][2] = C_DMG[kind][2];
      e.epal[slot] = 1;
    }
#pragma unroll
    for (int l = 0; l < 2; ++l)
      if (e.lal[3 + l] && !shoot[l] && cb[l] <= 6 && cb[l] > 2) chase_move<EXT>(e, 3 + l, dr[l], dc[l]);
  }
  // passive
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const int s = 5 + l;
    if (!e.lal[s]) continue;
    float u = draw(e, 3, l);
    if (!(u < 0.5f)) continue;
    int d = min((int)__fmul_rn(u, 16.0f) % 4, 3);
    move_lane<EXT>(e, s, C_DIR[d][0], C_DIR[d][1]);
  }
}

// engine._survival_tick (engine.py:640-700)
template <bool EXT>
GR_STEP_NI __device__ void survival_tick(Ctx& e) {
  const uint16_t dex = e.dex;
  const float hmax = health_max(e), fmax = food_max(e);
#pragma unroll
  for (int k = 0; k < 4; ++k) e.clocks[k] = (uint16_t)(e.clocks[k] + 1);
  bool due0 = e.clocks[0] >= (uint16_t)(30 * dex), due1 = e.clocks[1] >= (uint16_t)(20 * dex),
       due2 = e.clocks[2] >= (uint16_t)(40 * dex);
  bool tire = due2;
  if (e.sleeping) {
    tire = false;
    if (e.clocks[2] >= 2) { e.energy = fmind(__fadd_rn(e.energy, 1.0f), fmax); e.clocks[2] = 0; }
  }
  if (due0) e.food = __fsub_rn(e.food, 1.0f);
  if (due1) e.drink = __fsub_rn(e.drink, 1.0f);
  if (tire) e.energy = __fsub_rn(e.energy, 1.0f);
  if (due0) e.clocks[0] = 0;
  if (due1) e.clocks[1] = 0;
  if (due2) e.clocks[2] = 0;
  if (due0 || due1 || due2) {
    e.food = fmaxd(e.food, 0.0f); e.drink = fmaxd(e.drink, 0.0f); e.energy = fmaxd(e.energy, 0.0f);
  }
  if (e.clocks[3] >= 10) { e.mana = fmind(__fadd_rn(e.mana, 1.0f), mana_max(e)); e.clocks[3] = 0; }
  float depleted = __fadd_rn(__fadd_rn((float)(e.food <= 0.0f), (float)(e.drink <= 0.0f)), (float)(e.energy <= 0.0f));
  bool starving = depleted > 0.0f;
  e.clocks[4] = starving ? (uint16_t)(e.clocks[4] + 1) : (uint16_t)0;
  if (e.clocks[4] >= 10) { hurt(e, depleted); e.clocks[4] = 0; }
  bool healthy = !starving && e.health < hmax && e.health > 0.0f;
  e.clocks[5] = healthy ? (uint16_t)(e.clocks[5] + 1) : (uint16_t)0;
  if (e.clocks[5] >= 30) { e.health = q1(fmind(__fadd_rn(e.health, 1.0f), hmax)); e.clocks[5] = 0; }
  if (e.sleeping) {
    if (e.energy >= fmax) { e.sleeping = 0; award<EXT>(e, 15); }
    if (e.hurt) e.sleeping = 0;
  }
  if (EXT && e.resting) {
    if (e.hurt) e.resting = 0;
    if (e.health >= hmax || starving) e.resting = 0;
  }
}

// creatures._spawn_class (creatures.py:387-423)
template <bool EXT>
GR_STEP_NI2 __device__ void spawn_class(Ctx& e, int cls, int kind, double prob, int sub, uint8_t* pending) {
  const int cap = LCAP(cls), s0 = L0(cls);
  int n_alive = 0;
  for (int l = 0; l < cap; ++l) n_alive += e.lal[s0 + l];
  float u = draw(e, sub, 0);
  if (!((double)u < prob) || !(n_alive < cap) || kind < 0) return;
  float u1 = draw(e, sub, 1), u2 = draw(e, sub, 2);
  int off_r = (int)(int16_t)(int)__fmul_rn(u1, 21.0f) - 10;
  int off_c = (int)(int16_t)(int)__fmul_rn(u2, 21.0f) - 10;
  int dist = max(abs(off_r), abs(off_c));
  if (!(dist >= 5 && dist <= 10)) return;
  int r = e.prow + off_r, c = e.pcol + off_c;
  uint8_t b = gblock<EXT>(e, e.lf, r, c);
  uint64_t ws = coll_set(C_COLL[kind]);
  if (!in_set(ws, b)) return;
  if (cls == 1 && !(b == B_PATH || e.lf != 0)) return;
  int slot = -1;
  for (int l = cap - 1; l >= 0; --l) if (!e.lal[s0 + l]) slot = l;
  const int s = s0 + slot;
  e.lr[s] = (int16_t)r; e.lc[s] = (int16_t)c;
  e.lhp[s] = C_HP[kind];
  e.lty[s] = (uint8_t)kind;
  if (cls != 2) {
    e.lcd[s] = 0;
    *pending &= (uint8_t)~(1u << (s0 + slot));
  }
  e.lal[s] = 1;
}

// creatures._spawn_wave (creatures.py:455-486); the active floor is 8
template <bool EXT>
GR_STEP_NI __device__ void spawn_wave(Ctx& e, int wf, uint8_t* pending) {
  using T = TD<EXT>;
  uint8_t mk = (uint8_t)C_MEL_KIND[wf], rk = (uint8_t)C_RAN_KIND[wf];
#pragma unroll
  for (int l = 0; l < 2; ++l) {
    int r = e.nr + 2, c = e.nc + (l == 0 ? -2 : 2);
    if (r == e.prow && c == e.pcol) c += 1;
    e.lr[l] = (int16_t)r; e.lc[l] = (int16_t)c;
    e.lhp[l] = C_HP[mk]; e.lty[l] = mk; e.lcd[l] = 2; e.lal[l] = 1;
  }
  bool aquatic = C_COLL[rk] == 3;
  e.lr[3] = (int16_t)(aquatic ? T::H / 2 + 4 + 1 : e.nr + 3);
  e.lc[3] = (int16_t)(aquatic ? T::W / 2 - 5 + 1 : e.nc);
  e.lhp[3] = C_HP[rk]; e.lty[3] = rk; e.lcd[3] = 6; e.lal[3] = 1;
  *pending &= (uint8_t)~((1u << 0) | (1u << 1) | (1u << 3));
}

// creatures._boss_logic (creatures.py:489-520)
template <bool EXT>
GR_STEP_NI __device__ void boss_logic(Ctx& e, uint8_t* pending) {
  if (!(e.pfloor == 8 && e.boss_hp > 0.0f)) return;
  int enemies = e.lal[0] + e.lal[1] + e.lal[2] + e.lal[3] + e.lal[4];
  if (enemies != 0) return;
  bool first = e.boss_wave == 0;
  if (first) { spawn_wave<EXT>(e, 0, pending); e.boss_wave = 1; }
  bool was_vuln = e.boss_vuln;
  if (!first && !was_vuln && e.boss_wave > 0) {
    e.boss_vuln = 1;
    e.boss_timer = 20;
    sblock<EXT>(e, 8, e.nr, e.nc, B_NECROMANCER_VULN);
  }
  if (was_vuln && e.boss_wave < 8) {
    e.boss_timer -= 1;
    if (e.boss_timer == 0) {
      spawn_wave<EXT>(e, e.boss_wave, pending);
      e.boss_wave += 1;
      e.boss_vuln = 0;
      sblock<EXT>(e, 8, e.nr, e.nc, B_NECROMANCER);
    }
  }
}

template <bool EXT>
__device__ void spawn_despawn(Ctx& e, uint8_t* pending) {
  const int af = e.lf;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    if (!e.lal[s]) continue;
    int d = max(abs(e.lr[s] - e.prow), abs(e.lc[s] - e.pcol));
    if (!(d <= 12 || af == 8)) e.lal[s] = 0;
  }
  int night = (e.time % 300) >= 150;
  spawn_class<EXT>(e, 0, C_MEL_KIND[af], C_MEL_PROB[night][af], 4, pending);
  spawn_class<EXT>(e, 1, C_RAN_KIND[af], C_RAN_PROB[af], 5, pending);
  spawn_class<EXT>(e, 2, C_PAS_KIND[af], C_PAS_PROB[af], 6, pending);
  if (EXT) boss_logic<EXT>(e, pending);
}

// creatures.grow_plants (creatures.py:525-541)
template <bool EXT>
GR_STEP_NI __device__ void grow_plants(Ctx& e) {
#pragma unroll
  for (int l = 0; l < 10; ++l) {
    if (!e.plal[l]) continue;
    e.plage[l] = (uint16_t)(e.plage[l] + 1);
    uint8_t b = gblock<EXT>(e, 0, e.plr[l], e.plc[l]);
    bool is_plant = b == B_PLANT;
    bool keep = is_plant || b == B_RIPE_PLANT;
    e.plal[l] = keep;
    if (keep && is_plant && e.plage[l] >= 60) sblock<EXT>(e, 0, e.plr[l], e.plc[l], B_RIPE_PLANT);
  }
}

// the observation descriptor of this env (gr_desc.cuh) from registers
template <bool EXT>
__device__ void write_desc(const Ctx& e, uint32_t* d, const float* lut) {
  InvSrc s;
  s.wood = e.inv_wood; s.stone = e.inv_stone; s.coal = e.inv_coal; s.iron = e.inv_iron;
  s.diamond = e.inv_diamond; s.sapphire = e.inv_sapphire; s.ruby = e.inv_ruby; s.sapling = e.inv_sapling;
  s.torch = e.inv_torch; s.arrow = e.inv_arrow; s.book = e.inv_book;
#pragma unroll
  for (int k = 0; k < 6; ++k) s.potion[k] = e.inv_potion[k];
  s.pick = e.pick_tier; s.sword = e.sword_tier; s.sword_ench = e.sword_ench; s.has_bow = e.has_bow;
#pragma unroll
  for (int k = 0; k < 4; ++k) { s.armour[k] = e.armour[k]; s.armour_ench[k] = e.armour_ench[k]; }
  s.xp = e.xp; s.dex = e.dex; s.str_ = e.str_; s.intel = e.intel; s.facing = e.facing;
  s.sleeping = e.sleeping; s.resting = e.resting; s.learned_fire = e.learned_fire; s.learned_ice = e.learned_ice;
  s.pf = e.pfloor; s.cleared = EXT ? (e.cleared >> e.pfloor) & 1 : 0; s.boss_vuln = EXT ? e.boss_vuln : 0;
  s.health = e.health; s.food = e.food; s.drink = e.drink; s.energy = e.energy; s.mana = e.mana;
  s.time = e.time;
  float inv[50];
  inv_section<EXT>(s, inv, lut);
  uint32_t w[DESC_WORDS];
  constexpr int NINV = EXT ? 50 : 18;
#pragma unroll
  for (int k = 0; k < 50; ++k) w[k] = k < NINV ? __float_as_uint(inv[k]) : 0u;
  w[D_BASE] = __float_as_uint(e.pfloor == 0 ? lut_daylight(lut, e.time) : C_FLOOR_AMB[e.pfloor]);
  w[D_POS] = (uint32_t)(uint16_t)e.prow | ((uint32_t)(uint16_t)e.pcol << 16);
  w[D_FLAGS] = (uint32_t)e.pfloor | ((uint32_t)e.sleeping << 8) | ((uint32_t)((e.torch >> e.pfloor) & 1u) << 9);
  uint32_t slot[14];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int ch = EXT ? e.lty[q] + 1 : classic_channel(e.lty[q]);
    slot[q] = cre_slot<EXT>(e.lr[q], e.lc[q], e.lal[q], ch, e.prow, e.pcol);
  }
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    slot[8 + l] = cre_slot<EXT>(e.epr[l], e.epc[l], e.epal[l], EXT ? e.eptype[l] + 20 : 4, e.prow, e.pcol);
    slot[11 + l] = EXT ? cre_slot<EXT>(e.ppr[l], e.ppc[l], e.ppal[l], e.pptype[l] + 20, e.prow, e.pcol) : 0xFFFFu;
  }
#pragma unroll
  for (int q = 0; q < 7; ++q) w[D_CRE + q] = slot[2 * q] | (slot[2 * q + 1] << 16);
  w[60] = w[61] = w[62] = w[63] = 0;
  uint4* dst = reinterpret_cast<uint4*>(d);
#pragma unroll
  for (int q = 0; q < DESC_WORDS / 4; ++q) dst[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
}

// observation descriptors straight from the stored state (after an import,
// or for gr_observe); the step kernel writes them as a by-product
template <bool EXT>
__global__ void __launch_bounds__(128) k_make_desc(DS S, int64_t n) {
  using T = TD<EXT>;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (threadIdx.x == 0) {
    s_blk_base = (uint8_t*)S.f[GR_F_BLOCKS];
    s_itm_base = (uint8_t*)S.f[GR_F_ITEMS];
  }
  __syncthreads();
  if (i >= n) return;
  Ctx e;
  e.i = (uint32_t)i;
  load_env<EXT>(e, S);
  load_lanes<EXT>(e, S, e.pfloor);
  write_desc<EXT>(e, S.desc + (size_t)i * DESC_WORDS, S.lut);
}

void launch_make_desc(bool ext, const DS& S, int64_t n, cudaStream_t st) {
  const int grid = (int)((n + 127) / 128);
  if (grid <= 0) return;
  if (ext) k_make_desc<true><<<grid, 128, 0, st>>>(S, n);
  else k_make_desc<false><<<grid, 128, 0, st>>>(S, n);
}

// apply the previous step's deferred dead-lane cooldown decrements to the
// lanes currently loaded (the pending floor is the env's current floor)
__device__ __forceinline__ void apply_pending(Ctx& e, uint8_t pend, uint32_t prev_flags) {
  if (!pend) return;
  const bool mel = prev_flags & 1u, ran = prev_flags & 2u;
#pragma unroll
  for (int l = 0; l < 3; ++l)
    if (mel && ((pend >> l) & 1) && e.lcd[l] > 0) e.lcd[l] -= 1;
#pragma unroll
  for (int l = 0; l < 2; ++l)
    if (ran && ((pend >> (3 + l)) & 1) && e.lcd[3 + l] > 0) e.lcd[3 + l] -= 1;
}


#ifndef GR_STEP_SORT
#define GR_STEP_SORT 1   // game logic on action-sorted envs inside each CTA (needs GR_STEP_SMEM_CTX)
#endif
#ifndef GR_STEP_SMEM_CTX
#define GR_STEP_SMEM_CTX 1   // per-thread working copy in shared memory (0: registers + local memory)
#endif
template <bool EXT>
#ifndef GR_STEP_MINB
#define GR_STEP_MINB 4   // resident CTAs per SM the register budget is fitted to (128 regs/thread)
#endif
__global__ void __launch_bounds__(128, GR_STEP_MINB) k_step(DS S, StepArgs a) {
  using T = TD<EXT>;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < a.n && !(a.bad && a.bad[0] >= 0);
  uint32_t my_flags = 0;
  int my_done = 0;
  if (threadIdx.x == 0) {
    s_blk_base = (uint8_t*)S.f[GR_F_BLOCKS];
    s_itm_base = (uint8_t*)S.f[GR_F_ITEMS];
  }
  // a speculative worldgen pass launched behind this kernel as a programmatic
  // dependent (it reads nothing this kernel writes) may start once every CTA
  // of this grid is resident, i.e. after this kernel has its SMs
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#if GR_STEP_SMEM_CTX
  extern __shared__ __align__(16) unsigned char s_ctx_raw[];
  Ctx& e = reinterpret_cast<Ctx*>(s_ctx_raw)[threadIdx.x];
#else
  Ctx e;
#endif
  __syncthreads();
#if GR_STEP_SORT
  // Phase A (thread t = env t, coalesced): load the state into the working copy.
  const uint32_t prev_fl = a.prev_flags ? a.prev_flags[0] : 0u;
  double ep_ret0 = 0.0;
  int32_t ep_len0 = 0;
  __shared__ int s_hist[64], s_perm[128];
  if (threadIdx.x < 64) s_hist[threadIdx.x] = 0;
  int my_act = 63;   // invalid threads sort last
  if (valid) {
    e.i = (uint32_t)i;
    my_act = (int)a.actions[i];
    ep_ret0 = S.ep_return[i];
    ep_len0 = S.ep_length[i];
    e.act = (uint8_t)my_act;
    e.pend = S.cd_pending[i];
    load_env<EXT>(e, S);
    load_lanes<EXT>(e, S, e.pfloor);
  }
  __syncthreads();
  // counting sort of the CTA's envs by action: the game logic below runs
  // with each warp's lanes on few distinct actions (less branch divergence)
  const int rank_in = atomicAdd(&s_hist[my_act], 1);
  __syncthreads();
  if (threadIdx.x < 32) {   // exclusive scan of the 64 bucket counts
    const int c0 = s_hist[2 * threadIdx.x], c1 = s_hist[2 * threadIdx.x + 1];
    int x = c0 + c1;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if ((int)threadIdx.x >= o) x += y;
    }
    const int excl = x - c0 - c1;
    s_hist[2 * threadIdx.x] = excl;
    s_hist[2 * threadIdx.x + 1] = excl + c0;
  }
  __syncthreads();
  s_perm[s_hist[my_act] + rank_in] = threadIdx.x;
  __syncthreads();
  // Phase B (thread t = the env at sorted position t): the game logic.
  {
    const int slot = s_perm[threadIdx.x];
    const int64_t ii = (int64_t)blockIdx.x * blockDim.x + slot;
    const bool v2 = ii < a.n && !(a.bad && a.bad[0] >= 0);
    if (v2) {
      Ctx& g = reinterpret_cast<Ctx*>(s_ctx_raw)[slot];
      uint8_t pend = g.pend;
      apply_pending(g, pend, prev_fl);
      pend = 0;
      g.unlock[0] = g.unlock[1] = g.unlock[2] = 0;
      g.hurt = false;
      g.health0 = g.health;
      g.base = mix32(g.key_lo ^ (g.time * 0x9E3779B9u));
      const int f0 = g.pfloor;
      player_actions<EXT>(g, S, (int)g.act);
      if (EXT && g.pfloor != f0) {
#pragma unroll
        for (int s_ = 0; s_ < 5; ++s_) {
          const int cls = s_ < 3 ? 0 : 1, l = s_ < 3 ? s_ : s_ - 3;
          GR_AT(S, cls == 0 ? GR_F_MEL_CD : GR_F_RAN_CD, uint8_t, f0 * LCAP(cls) + l, ii) = g.lcd[s_];
        }
        load_lanes<EXT>(g, S, g.pfloor);
      }
      advance_projectiles<EXT>(g);
      uint8_t lf = 0;
      lf |= (g.lal[0] | g.lal[1] | g.lal[2]) ? 1u : 0u;
      lf |= (g.lal[3] | g.lal[4]) ? 2u : 0u;
      g.lflags = lf;
      creatures_act<EXT>(g, &pend);
      survival_tick<EXT>(g);
      spawn_despawn<EXT>(g, &pend);
      grow_plants<EXT>(g);
      g.time += 1;
      g.pend = pend;
    }
  }
  __syncthreads();
  // Phase C (thread t = env t again, coalesced): outcome, write-back, outputs.
  if (valid) {
    my_flags = e.lflags;
    const uint8_t pend = e.pend;
#else
  if (valid) {
    e.i = (uint32_t)i;
    // the per-env words the tail needs are loaded with the state, not after
    // the game logic (the compiler does not move loads across its stores)
    const int action = (int)a.actions[i];
    const double ep_ret0 = S.ep_return[i];
    const int32_t ep_len0 = S.ep_length[i];
    uint8_t pend = S.cd_pending[i];
    const uint32_t prev_fl = a.prev_flags ? a.prev_flags[0] : 0u;
    load_env<EXT>(e, S);
    load_lanes<EXT>(e, S, e.pfloor);
    apply_pending(e, pend, prev_fl);
    pend = 0;
    // _kern.Workspace.begin_step
    e.unlock[0] = e.unlock[1] = e.unlock[2] = 0;
    e.hurt = false;
    e.health0 = e.health;
    e.base = mix32(e.key_lo ^ (e.time * 0x9E3779B9u));
    const int f0 = e.pfloor;
    player_actions<EXT>(e, S, action);
    if (EXT && e.pfloor != f0) {   // a ladder: the creature phases act on the new floor
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        const int cls = s < 3 ? 0 : 1, l = s < 3 ? s : s - 3;
        GR_AT(S, cls == 0 ? GR_F_MEL_CD : GR_F_RAN_CD, uint8_t, f0 * LCAP(cls) + l, i) = e.lcd[s];
      }
      load_lanes<EXT>(e, S, e.pfloor);
    }
    advance_projectiles<EXT>(e);
    my_flags |= (e.lal[0] | e.lal[1] | e.lal[2]) ? 1u : 0u;
    my_flags |= (e.lal[3] | e.lal[4]) ? 2u : 0u;
    creatures_act<EXT>(e, &pend);
    survival_tick<EXT>(e);
    spawn_despawn<EXT>(e, &pend);
    grow_plants<EXT>(e);
    e.time += 1;
#endif
    // achievements, reward, done (engine.py:731-745)
    double reward = 0.0;
    uint32_t newly[3];
#pragma unroll
    for (int w = 0; w < 3; ++w) {
      newly[w] = e.unlock[w] & ~e.ach[w];
      e.ach[w] |= newly[w];
    }
#pragma unroll
    for (int w = 0; w < 3; ++w) {
      uint32_t m = newly[w];
      while (m) {
        int b = __ffs(m) - 1;
        m &= m - 1;
        reward += EXT ? (double)C_ACH_TIER[w * 32 + b] : 1.0;
      }
    }
    float delta = __fsub_rn(e.health, e.health0);
    reward = __dadd_rn(reward, __dmul_rn(0.1, (double)delta));
    const bool done = e.health <= 0.0f || (int64_t)e.time >= a.max_len;
    store_env<EXT>(e, S);
    store_lanes<EXT>(e, S);
    S.cd_pending[i] = pend;
    GR_AT(S, GR_F_DONE, uint8_t, 0, i) = done;
    // batch.batch_step bookkeeping (batch.py:206-209) and outputs
    S.ep_return[i] = __dadd_rn(ep_ret0, reward);
    S.ep_length[i] = ep_len0 + 1;
    a.reward[i] = (float)reward;
    a.done[i] = done;
    if (a.itime) a.itime[i] = e.time;
    if (a.ifloor) a.ifloor[i] = e.pfloor;
    if (a.newly) {
      uint8_t* nw = a.newly + (size_t)i * T::A;
#pragma unroll 1
      for (int k = 0; k < T::A; ++k) nw[k] = (newly[k >> 5] >> (k & 31)) & 1u;
    }
    if (a.reward64) a.reward64[i] = reward;
    if (!done) write_desc<EXT>(e, S.desc + (size_t)i * DESC_WORDS, S.lut);   // reset envs: install writes it
    my_done = done;
    if (EXT && !done && C_FLOOR_AMB[e.pfloor] < 1.0f) my_flags |= 4u;
  }
  const int cnt = __syncthreads_count(my_done);
  const int fl_mel = __syncthreads_or(my_flags & 1u);
  const int fl_ran = __syncthreads_or(my_flags & 2u);
  const int fl_dark = __syncthreads_or(my_flags & 4u);
  __shared__ int last;
  if (threadIdx.x == 0) {
    if (a.block_done) a.block_done[blockIdx.x] = cnt;
    uint32_t f = (fl_mel ? 1u : 0u) | (fl_ran ? 2u : 0u) | (fl_dark ? 4u : 0u);
    if (f) atomicOr(a.cur_flags, f);
    last = 0;
    if (a.arrive) {
      __threadfence();   // this CTA's count and flags before its arrival
      last = atomicAdd(a.arrive, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!last) return;
  // the last CTA: every other CTA's block_done / cur_flags are visible
  __threadfence();
  const int32_t total = cta_scan_blocks(a.block_done, a.block_off, a.nb);
  if (threadIdx.x == 0) {
    const uint32_t fl = *(volatile const uint32_t*)a.cur_flags;
    a.exchange[0] = total;
    a.exchange[1] = (int32_t)fl;
    a.exchange[2] = 0;
    a.exchange[3] = 0;
    if (a.info) combine_info(a.exchange, 0, 1, a.M, a.pool_key, a.dstep, a.info, a.flags_out, !a.defer_advance);
    *a.arrive = 0u;
    *a.cur_flags = 0u;   // consumed: clean for the next step (no memset node per step)
  }
}

// the observation value tables (gr_desc.cuh), evaluated by the exact expressions
__global__ void k_init_lut(float* lut) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < LUT_N) lut[k] = lut_value_exact(k);
}

void launch_init_lut(float* lut, cudaStream_t st) { k_init_lut<<<(LUT_N + 127) / 128, 128, 0, st>>>(lut); }

void launch_step(bool ext, const DS& S, const StepArgs& a, cudaStream_t st) {
  const int bs = 128;
  const int grid = (int)((a.n + bs - 1) / bs);
  if (grid == 0) return;
#if GR_STEP_SMEM_CTX
  const size_t smem = (size_t)bs * sizeof(Ctx);
  static PerDeviceOnce once;
  once([&](int) {
    cudaFuncSetAttribute(k_step<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_step<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
#else
  const size_t smem = 0;
#endif
  if (ext) k_step<true><<<grid, bs, smem, st>>>(S, a);
  else k_step<false><<<grid, bs, smem, st>>>(S, a);
}

}  // namespace gr
