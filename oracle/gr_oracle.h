/*
 * gr_oracle.h -- CPU restatement of the gridrogue batched-env hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * CUDA product in paper_2402_16801_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The
 * product never links, imports or calls anything under oracle/.
 *
 * It restates, in scalar per-env C, the numpy reference at
 * /root/reference/pkg/src/gridrogue (rng.py, _kern.py, engine.py,
 * creatures.py, perlin.py, worldgen.py, state.py, obs.py, tiles.py,
 * batch.py, policies.py).  The state is held in the reference's own
 * SimState layout (state.py:29-125): one env-major array per field, so a
 * SimState built by the reference can be handed over field by field.
 *
 * Parity is pinned against golden vectors minted from the reference by
 * tests/golden/make_golden.py.
 *
 * Floating point: compiled with -ffp-contract=off so every f32 / f64 op is
 * separately rounded, matching numpy's elementwise evaluation.
 */
#ifndef GR_ORACLE_H
#define GR_ORACLE_H

#include <stdint.h>
#include <stdbool.h>

#ifdef __cplusplus
extern "C" {
#endif

/* field ids follow state.FIELD_NAMES order (state.py:29-125) */
enum {
  FO_BLOCKS, FO_ITEMS, FO_LADDER_DOWN, FO_LADDER_UP, FO_SPAWN0, FO_POTION_MAP,
  FO_CHEST_POS, FO_CHEST_LOOT, FO_CHEST_QTY, FO_CHEST_AUX, FO_NECRO_POS,
  FO_PARAMS_SEED,
  FO_PFLOOR, FO_PROW, FO_PCOL, FO_FACING, FO_HEALTH, FO_FOOD, FO_DRINK,
  FO_ENERGY, FO_MANA, FO_XP, FO_DEX, FO_STR, FO_INTEL, FO_SWORD_TIER,
  FO_PICK_TIER, FO_HAS_BOW, FO_SWORD_ENCH, FO_BOW_ENCH, FO_ARMOUR,
  FO_ARMOUR_ENCH, FO_LEARNED_FIRE, FO_LEARNED_ICE, FO_SLEEPING, FO_RESTING,
  FO_INV_WOOD, FO_INV_STONE, FO_INV_COAL, FO_INV_IRON, FO_INV_DIAMOND,
  FO_INV_SAPPHIRE, FO_INV_RUBY, FO_INV_SAPLING, FO_INV_TORCH, FO_INV_ARROW,
  FO_INV_BOOK, FO_INV_POTION,
  FO_MEL_POS, FO_MEL_HP, FO_MEL_CD, FO_MEL_ALIVE, FO_MEL_TYPE,
  FO_RAN_POS, FO_RAN_HP, FO_RAN_CD, FO_RAN_ALIVE, FO_RAN_TYPE,
  FO_PAS_POS, FO_PAS_HP, FO_PAS_ALIVE, FO_PAS_TYPE,
  FO_PPROJ_POS, FO_PPROJ_DIR, FO_PPROJ_TYPE, FO_PPROJ_TTL, FO_PPROJ_ALIVE,
  FO_PPROJ_DMG,
  FO_EPROJ_POS, FO_EPROJ_DIR, FO_EPROJ_TYPE, FO_EPROJ_TTL, FO_EPROJ_ALIVE,
  FO_EPROJ_DMG,
  FO_PLANT_POS, FO_PLANT_AGE, FO_PLANT_ALIVE,
  FO_ACH, FO_TIME, FO_RNG_KEY, FO_FLOORS_VISITED, FO_FLOOR_CLEARED,
  FO_BOSS_HP, FO_BOSS_WAVE, FO_BOSS_VULN, FO_BOSS_TIMER, FO_CLOCKS, FO_DONE,
  FO_NFIELDS
};

/* one generated world (worldgen.World), extended-sized buffers */
typedef struct {
  uint8_t blocks[9][64 * 64];
  uint8_t items[9][64 * 64];
  int16_t spawn[2];                 /* floors[0].spawn */
  int16_t ladder_down[9][2];        /* (-1,-1) when absent */
  int16_t ladder_up[9][2];
  int16_t chest[9][6][4];           /* r, c, loot, qty */
  int32_t n_chests[9];
  uint8_t potion[6];
  uint64_t seed;                    /* params.seed */
  int32_t attempts[9];              /* retries used per floor (diagnostic) */
  int32_t potion_tie;               /* 1 if the potion argsort saw a tie */
} go_world;

/* --- rng.py -------------------------------------------------------------- */
uint64_t go_mix(uint64_t z);
uint64_t go_hash2(uint64_t key, uint64_t n);
uint32_t go_vmix32(uint32_t x);
float go_vuniform32(uint32_t key, uint32_t n);
double go_vuniform(uint64_t key, uint64_t n);

/* numpy's float32 SIMD sin / cos (loops_trigonometric), restated */
float go_np_sinf(float x);
float go_np_cosf(float x);
/* numpy's AVX-512 np.argsort of 6 float32 (tie order included) */
void go_np_argsort6(const float *v, uint8_t *idx);

/* --- worldgen ------------------------------------------------------------ */
void go_level_angles(uint64_t seed, float *angles252, uint64_t *floor_seeds9);
void go_generate_world(uint64_t seed, int classic, go_world *w);
/* worldgen.MAX_GEN_RETRIES (default 16; 0 forces every floor to the template) */
void go_set_max_gen_retries(int n);
void go_overworld_fields(const float *angles252, int h, int w,
                         float *height, float *forest, float *special);
void go_perlin_cave(const float *a25, const float *a81, int h, int w,
                    double *field);

/* --- native oracle state (go_state.h) ------------------------------------ */
typedef struct go_state go_state_t;
go_state_t *go_state_new(int classic, int64_t n, int64_t max_len);
void go_state_free(go_state_t *s);
/* reference-layout (state.FIELD_NAMES order) field arrays <-> oracle state */
void go_state_import(go_state_t *s, void *const *fields);
void go_state_export(const go_state_t *s, void *const *fields);
void go_state_install_seed(go_state_t *s, int64_t env, uint64_t world_seed, uint64_t key);
/* engine.step_batch over the whole state: returns 0 or -1-env of the first
 * invalid action (nothing mutated) */
int64_t go_state_step(go_state_t *s, const int64_t *actions, double *reward,
                      uint8_t *done, uint8_t *newly, float *delta);
void go_state_encode(const go_state_t *s, float *out);            /* [n, L] */
void go_state_pixels(const go_state_t *s, int tile_px, uint8_t *out);

/* --- batch.py ------------------------------------------------------------ */
typedef struct go_batch go_batch;
go_batch *go_batch_create(int classic, int64_t n, uint64_t seed, int reset_ratio,
                          int64_t max_len, int threads);
go_batch *go_batch_create_shard(int classic, int64_t n, int64_t env_offset, int64_t n_global,
                                uint64_t seed, int reset_ratio, int64_t max_len, int threads);
int64_t go_batch_step_a(go_batch *b, const int64_t *actions, int *flags);
int64_t go_batch_step_b(go_batch *b, const int *flags, double *reward, uint8_t *done, uint8_t *newly,
                        uint32_t *info_time, uint8_t *info_floor);
void go_batch_step_c(go_batch *b, int64_t offset);
int go_state_any_dark(const go_state_t *s);
void go_state_encode_flag(const go_state_t *s, int dark, float *out);
void go_batch_destroy(go_batch *b);
go_state_t *go_batch_state(go_batch *b);
int64_t go_batch_step(go_batch *b, const int64_t *actions, double *reward,
                      uint8_t *done, uint8_t *newly, uint32_t *info_time,
                      uint8_t *info_floor);
void go_batch_stats(const go_batch *b, int64_t *episodes, double *total_return,
                    int64_t *total_steps, int64_t *ach_counts);
void go_batch_ep(const go_batch *b, double *ep_return, int64_t *ep_length);
void go_random_actions(uint32_t seed, uint64_t t, int64_t env0, int64_t n,
                       int n_actions, int64_t *out);

#ifdef __cplusplus
}
#endif
#endif
