// gr_state.cuh -- device memory layout of the batch state.
//
// Non-map fields are struct-of-arrays with the env index fastest:
// component c of field f for env i lives at  f_ptr[c * ns + i]  where the
// components are the row-major flattening of the reference's trailing shape
// (state._SHAPES, state.py:29-125).  One thread per env therefore loads and
// stores every field with fully coalesced 32-128 B warp transactions.
// Maps (blocks/items) stay env-major [n][F][H][W]: a step touches a small
// window around one player, contiguous per row.
// Achievements are packed to 3 x u32 bit-words per env ([3][ns]).
#pragma once
#include <cstdint>
#include "../../include/gridrogue_b200.h"

namespace gr {

enum : int8_t { K_MAP, K_PERF, K_FIX, K_ACH };
struct FieldDesc { int8_t esz, kind; int16_t k; };

// esz, kind, components (per floor for K_PERF)
constexpr FieldDesc FIELD_TABLE[GR_NFIELDS] = {
    {1, K_MAP, 0}, {1, K_MAP, 0},                                     // blocks items
    {2, K_PERF, 2}, {2, K_PERF, 2}, {2, K_FIX, 2}, {1, K_FIX, 6},     // ladders spawn0 potion_map
    {2, K_PERF, 12}, {1, K_PERF, 6}, {1, K_PERF, 6}, {1, K_PERF, 6},  // chest_*
    {2, K_FIX, 2}, {8, K_FIX, 1},                                     // necro_pos params_seed
    {1, K_FIX, 1}, {2, K_FIX, 1}, {2, K_FIX, 1}, {1, K_FIX, 1},       // pfloor prow pcol facing
    {4, K_FIX, 1}, {4, K_FIX, 1}, {4, K_FIX, 1}, {4, K_FIX, 1}, {4, K_FIX, 1},  // vitals
    {1, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1},       // xp dex str intel
    {1, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1},  // tiers bow ench
    {1, K_FIX, 4}, {1, K_FIX, 4},                                     // armour armour_ench
    {1, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1},       // learned* sleeping resting
    {1, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1},
    {1, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1},  // inv_*
    {1, K_FIX, 6},                                                    // inv_potion
    {2, K_PERF, 6}, {4, K_PERF, 3}, {1, K_PERF, 3}, {1, K_PERF, 3}, {1, K_PERF, 3},  // mel_*
    {2, K_PERF, 4}, {4, K_PERF, 2}, {1, K_PERF, 2}, {1, K_PERF, 2}, {1, K_PERF, 2},  // ran_*
    {2, K_PERF, 6}, {4, K_PERF, 3}, {1, K_PERF, 3}, {1, K_PERF, 3},                  // pas_*
    {2, K_FIX, 6}, {1, K_FIX, 3}, {1, K_FIX, 3}, {1, K_FIX, 3}, {1, K_FIX, 3}, {4, K_FIX, 9},  // pproj
    {2, K_FIX, 6}, {1, K_FIX, 3}, {1, K_FIX, 3}, {1, K_FIX, 3}, {1, K_FIX, 3}, {4, K_FIX, 9},  // eproj
    {2, K_FIX, 20}, {2, K_FIX, 10}, {1, K_FIX, 10},                   // plants
    {4, K_ACH, 3}, {4, K_FIX, 1}, {8, K_FIX, 1},                      // ach(bits) time rng_key
    {1, K_PERF, 1}, {1, K_PERF, 1},                                   // floors_visited floor_cleared
    {4, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1}, {1, K_FIX, 1},       // boss_*
    {2, K_FIX, 6}, {1, K_FIX, 1}};                                    // clocks done

struct TierDims { int F, H, W, A, NA, VR, VC; };
constexpr TierDims CLASSIC_DIMS{1, 64, 64, 22, 17, 7, 9};
constexpr TierDims EXT_DIMS{9, 48, 48, 67, 43, 9, 11};

// device components per env (ach: 3 packed words)
inline int64_t device_comps(int fid, const TierDims& d) {
  const FieldDesc& f = FIELD_TABLE[fid];
  switch (f.kind) {
    case K_MAP: return (int64_t)d.F * d.H * d.W;
    case K_PERF: return (int64_t)d.F * f.k;
    case K_ACH: return 3;
    default: return f.k;
  }
}
// reference-layout elements per env
inline int64_t ref_elems(int fid, const TierDims& d) {
  const FieldDesc& f = FIELD_TABLE[fid];
  if (f.kind == K_ACH) return d.A;
  return device_comps(fid, d);
}
inline int ref_esz(int fid) { return FIELD_TABLE[fid].kind == K_ACH ? 1 : FIELD_TABLE[fid].esz; }

// Device state handle (passed by value to kernels).
struct DS {
  int64_t ns;                 // env stride (= n local envs)
  void* f[GR_NFIELDS];
  uint8_t* cd_pending;        // deferred dead-lane cooldown decrements (bits)
  double* ep_return;          // batch.BatchState.ep_return
  int32_t* ep_length;         // batch.BatchState.ep_length
  uint32_t* desc;             // [ns][64] observation descriptors (gr_desc.cuh)
  uint16_t* torch_bits;       // bit f: a torch may lie on floor f (torches are never removed)
  const float* lut;           // exact small-argument tables of the observation values (gr_desc.cuh)
};

// one generated world (worldgen.World) in a world buffer
struct WMeta {
  int16_t spawn[2];
  int16_t ld[9][2], lu[9][2];
  int16_t chest[9][6][4];     // r, c, loot, qty
  uint8_t nch[9];
  uint8_t potion[6];
  uint8_t pad;
  uint64_t seed;              // LevelParams.seed
  uint64_t key;               // install key (state key)
  uint32_t flags;             // WG_FLAG_*
  uint32_t pad2;
};
enum : uint32_t { WG_FLAG_RETRY = 1, WG_FLAG_TEMPLATE = 2, WG_FLAG_POTION_TIE = 4,
                  WG_FLAG_TEMPLATE_F0 = 1u << 8 };   // + f: floor f is the _template_floor fallback

struct WBuf {
  uint8_t* blocks;            // [cap][F][H][W]
  uint8_t* items;
  WMeta* meta;                // [cap]
  int64_t cap;
};

#define GR_AT(S, fid, T, comp, i) (((T*)(S).f[fid])[(size_t)(comp) * (size_t)(S).ns + (size_t)(i)])

}  // namespace gr
