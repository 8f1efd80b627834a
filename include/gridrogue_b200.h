/*
 * gridrogue_b200.h -- C ABI of the B200-native batched gridrogue/Craftax
 * environment (libgridrogue_b200.so).
 *
 * Drop-in boundary for the reference's batched hot path:
 *   gridrogue_gym.BatchEnv   (/root/reference/pkg/bindings/src/gridrogue_gym/__init__.py:24-95)
 *   gridrogue.batch          (/root/reference/pkg/src/gridrogue/batch.py:127-234)
 * Each entry point below names the reference interface it replaces.
 *
 * Conventions
 *   - plain pointers + sizes, no framework types; "dev" pointers are CUDA
 *     device memory on the handle's device, "host" pointers are host memory
 *     (pinned for the asynchronous *_host entry points).
 *   - one handle <=> one CUDA device <=> one owner (the reference's
 *     single-owner lock, __init__.py:47,66-68, lives in the Python wrapper).
 *   - every call returns GR_OK (0) or a negative GR_E* code; the message is
 *     available from gr_last_error().  A failing call mutates nothing.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 */
#ifndef GRIDROGUE_B200_H
#define GRIDROGUE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GR_ABI_VERSION 1

enum {
  GR_OK = 0,
  GR_E_INVALID = -1,       /* bad argument (ValueError in the reference)   */
  GR_E_CUDA = -2,          /* CUDA runtime failure                           */
  GR_E_STATE = -3,         /* call order violated (RuntimeError)            */
  GR_E_BAD_ACTION = -4,    /* action out of range: gr_bad_action() has env  */
  GR_E_OOM = -5
};

enum { GR_TIER_CLASSIC = 0, GR_TIER_EXTENDED = 1 };            /* constants.tier_by_name */
enum { GR_OBS_NONE = 0, GR_OBS_SYMBOLIC = 1, GR_OBS_PIXELS = 2 }; /* BatchEnv obs_mode (+pixels) */

/* state field ids: the order of gridrogue.state.FIELD_NAMES (state.py:29-125) */
enum {
  GR_F_BLOCKS, GR_F_ITEMS, GR_F_LADDER_DOWN, GR_F_LADDER_UP, GR_F_SPAWN0, GR_F_POTION_MAP,
  GR_F_CHEST_POS, GR_F_CHEST_LOOT, GR_F_CHEST_QTY, GR_F_CHEST_AUX, GR_F_NECRO_POS,
  GR_F_PARAMS_SEED, GR_F_PFLOOR, GR_F_PROW, GR_F_PCOL, GR_F_FACING, GR_F_HEALTH, GR_F_FOOD,
  GR_F_DRINK, GR_F_ENERGY, GR_F_MANA, GR_F_XP, GR_F_DEX, GR_F_STR, GR_F_INTEL,
  GR_F_SWORD_TIER, GR_F_PICK_TIER, GR_F_HAS_BOW, GR_F_SWORD_ENCH, GR_F_BOW_ENCH, GR_F_ARMOUR,
  GR_F_ARMOUR_ENCH, GR_F_LEARNED_FIRE, GR_F_LEARNED_ICE, GR_F_SLEEPING, GR_F_RESTING,
  GR_F_INV_WOOD, GR_F_INV_STONE, GR_F_INV_COAL, GR_F_INV_IRON, GR_F_INV_DIAMOND,
  GR_F_INV_SAPPHIRE, GR_F_INV_RUBY, GR_F_INV_SAPLING, GR_F_INV_TORCH, GR_F_INV_ARROW,
  GR_F_INV_BOOK, GR_F_INV_POTION, GR_F_MEL_POS, GR_F_MEL_HP, GR_F_MEL_CD, GR_F_MEL_ALIVE,
  GR_F_MEL_TYPE, GR_F_RAN_POS, GR_F_RAN_HP, GR_F_RAN_CD, GR_F_RAN_ALIVE, GR_F_RAN_TYPE,
  GR_F_PAS_POS, GR_F_PAS_HP, GR_F_PAS_ALIVE, GR_F_PAS_TYPE, GR_F_PPROJ_POS, GR_F_PPROJ_DIR,
  GR_F_PPROJ_TYPE, GR_F_PPROJ_TTL, GR_F_PPROJ_ALIVE, GR_F_PPROJ_DMG, GR_F_EPROJ_POS,
  GR_F_EPROJ_DIR, GR_F_EPROJ_TYPE, GR_F_EPROJ_TTL, GR_F_EPROJ_ALIVE, GR_F_EPROJ_DMG,
  GR_F_PLANT_POS, GR_F_PLANT_AGE, GR_F_PLANT_ALIVE, GR_F_ACH, GR_F_TIME, GR_F_RNG_KEY,
  GR_F_FLOORS_VISITED, GR_F_FLOOR_CLEARED, GR_F_BOSS_HP, GR_F_BOSS_WAVE, GR_F_BOSS_VULN,
  GR_F_BOSS_TIMER, GR_F_CLOCKS, GR_F_DONE,
  GR_NFIELDS
};

typedef struct gr_env gr_env;

/* batch.BatchConfig (batch.py:34-55) + BatchEnv(...) (__init__.py:35-47),
 * extended with the shard description for multi-GPU runs. */
typedef struct {
  int32_t tier;                /* GR_TIER_*                                       */
  int32_t obs_mode;            /* GR_OBS_*                                        */
  int32_t tile_px;             /* pixels: 7, 10 or 16 (tiles.SUPPORTED_TILE_PX)   */
  int32_t reset_ratio;         /* BatchConfig.reset_ratio (default 16)            */
  int64_t n_envs;              /* envs owned by this handle                        */
  int64_t env_offset;          /* global index of this handle's env 0              */
  int64_t n_envs_global;       /* BatchConfig.n_envs of the whole batch            */
  int64_t max_episode_length;  /* 0 = tier default (100000)                        */
  uint64_t seed;               /* batch_reset(cfg, seed)                           */
  int32_t device;              /* CUDA ordinal                                     */
  int32_t reserved;
} gr_config;

/* batch.EpisodeStats (batch.py:109-124), summed over completed episodes */
typedef struct {
  int64_t episodes;
  int64_t total_steps;
  double total_return;         /* summed in device order (not numpy pairwise)     */
  int64_t ach_episodes[67];    /* per achievement: episodes that unlocked it      */
} gr_stats;

/* ---- lifecycle --------------------------------------------------------- */
/* BatchEnv.__init__ (__init__.py:35-47): allocates all device state. */
int gr_create(const gr_config *cfg, gr_env **out);
void gr_destroy(gr_env *env);
const char *gr_last_error(void);
int gr_version(void);

/* ---- shapes -------------------------------------------------------------- */
/* obs.obs_length / tiles frame size: floats (symbolic) or bytes (pixels) per env */
int64_t gr_obs_elems(const gr_env *env);
int32_t gr_n_actions(const gr_env *env);        /* TierConf.n_actions        */
int32_t gr_n_achievements(const gr_env *env);   /* TierConf.n_achievements   */
/* per-env element count and element size of state field `field` in the
 * reference layout (state._SHAPES); returns GR_E_INVALID for a bad id */
int gr_field_info(int32_t tier, int32_t field, int64_t *elems_per_env, int32_t *elem_size);

/* ---- hot path (device buffers) ------------------------------------------ */
/* batch_reset (batch.py:167-169) + BatchEnv._observe (__init__.py:92-95):
 * generates every env's world on device and writes the post-reset obs. */
int gr_reset(gr_env *env, void *obs_dev, void *stream);

/* BatchEnv.step (__init__.py:63-84) == batch_step(bs, actions)
 * (batch.py:193-234) + post-reset encode_symbolic_batch.
 *   actions_dev  int64[n]                 (validate: see gr_set_validate)
 *   obs_dev      float32[n, L] or uint8[n, H, W, 3], post-reset; may be NULL;
 *                any alignment of its element type (16-byte-aligned buffers
 *                take the TMA row stores, others plain stores)
 *   reward_dev   float32[n]               (reward.astype(float32))
 *   done_dev     uint8[n]
 *   newly_dev    uint8[n, A] or NULL      (info["newly_unlocked"])
 *   time_dev     uint32[n] or NULL        (info["time"], pre-reset)
 *   floor_dev    uint8[n] or NULL         (info["floor"], pre-reset)   */
int gr_step(gr_env *env, const int64_t *actions_dev, void *obs_dev, float *reward_dev,
            uint8_t *done_dev, uint8_t *newly_dev, uint32_t *time_dev, uint8_t *floor_dev,
            void *stream);

/* policies.RandomPolicy(seed, n_actions).actions at step t, for this shard's
 * global env indices (policies.py:31-37) */
int gr_random_actions(gr_env *env, uint32_t seed, uint64_t t, int64_t *actions_dev, void *stream);

/* When enabled (default), gr_step checks actions on device first; on a bad
 * action nothing is mutated, GR_E_BAD_ACTION is returned (this synchronises
 * the stream) and gr_bad_action() reports the first offending env/action
 * (engine.py:713-717, __init__.py:74-77). */
int gr_set_validate(gr_env *env, int32_t on);
int gr_bad_action(const gr_env *env, int64_t *env_index, int64_t *action);

/* ---- sharded (multi-GPU) step ------------------------------------------ *
 * The optimistic-reset pool assigns slot = global rank of each done env mod
 * M (batch.py:217-229), and two batch-wide `any()` flags of the reference
 * (creatures.py:290,329 and obs.py:236) couple envs across shards.  A step
 * is therefore split around one small all-gather:
 *   gr_step_local  -> writes this shard's 4 x int32 exchange record
 *   (caller all-gathers the records of all ranks, rank order)
 *   gr_step_finish -> pool worldgen, install, observation.
 * gr_step == gr_step_local + gr_step_finish with world size 1. */
int gr_step_local(gr_env *env, const int64_t *actions_dev, float *reward_dev, uint8_t *done_dev,
                  uint8_t *newly_dev, uint32_t *time_dev, uint8_t *floor_dev,
                  int32_t *exchange_dev /* int32[4] */, void *stream);
int gr_step_finish(gr_env *env, const int32_t *exchange_all_dev /* int32[world*4] */,
                   int32_t rank, int32_t world, void *obs_dev, void *stream);
/* Both halves and the caller's collective between them are capturable
 * (validation off): a caller that captured local + all-gather + finish in one
 * CUDA graph and replayed it `steps` times reports it here, so the host-side
 * step index and launch counter stay exact (launches_per_step = the kernels
 * the captured step contains). */
int gr_account_replay(gr_env *env, int64_t steps, int64_t launches_per_step);

/* ---- end-to-end (host buffers) ------------------------------------------ *
 * Same contract as gr_step with host arrays: H2D of actions, the step,
 * D2H of obs/reward/done/newly/info; synchronous on return. */
int gr_step_host(gr_env *env, const int64_t *actions_host, void *obs_host, float *reward_host,
                 uint8_t *done_host, uint8_t *newly_host, uint32_t *time_host,
                 uint8_t *floor_host);
int gr_reset_host(gr_env *env, void *obs_host);

/* Delta observation transfer (symbolic observations only).  Attaching a host
 * buffer of n_envs x obs_width float32 hands its contents to the handle: it
 * is zero-filled now, the handle keeps a device copy of it, and every later
 * gr_step_host / gr_reset_host into it moves only the words that changed
 * since the observation last written into that buffer ((word index, value
 * bits), 8 B each; ~1.3 % of the words two steps apart) and rewrites only
 * those on the host, instead of copying 4 B x n x width.  The buffer then
 * equals a dense copy bit for bit, as long as the caller never writes into
 * it.  Needs n x width < 2^32.  The transfer behind BatchEnv.step's obs
 * (bindings/src/gridrogue_gym/__init__.py:63-84), BatchEnv(obs_transfer=
 * "delta") in the Python mirror. */
int gr_host_obs_attach(gr_env *env, void *obs_host);
int gr_host_obs_detach(gr_env *env, void *obs_host);
/* Host-measured phases of gr_step_host / gr_reset_host since the last read
 * (then reset), milliseconds summed over calls: [0] enqueue (H2D of actions,
 * step launch, delta kernels), [1] waiting on the device (step + change
 * detection; with a dense copy, included in [3]), [2] host scatter of the
 * changed words, [3] final synchronisation (small outputs, dense obs copy);
 * calls / words: host-path calls and changed words delivered. */
int gr_host_phase_times(gr_env *env, double out[4], int64_t *calls, int64_t *words);
/* Copy a device observation buffer of this handle's shape (e.g. what
 * gr_step_finish wrote on a shard) into a plain host array, every word
 * written, ordered after the caller's work on `stream`; synchronous.
 * Symbolic observations travel packed (per-row non-zero bitmap + values,
 * expanded by host threads) unless GR_HOST_COMPACT=0 -- the transfer behind
 * gr_step_host's dense path. */
int gr_obs_to_host(gr_env *env, const void *obs_dev, void *obs_host, void *stream);


/* ---- state channel (parity / checkpoint) -------------------------------- *
 * Copy one SimState field to / from host memory in the reference layout
 * (env-major, state._SHAPES).  Synchronous.  Importing clears any deferred
 * bookkeeping so the device state equals the imported SimState exactly. */
int gr_export_field(gr_env *env, int32_t field, void *host_dst);
int gr_import_field(gr_env *env, int32_t field, const void *host_src);
/* BatchState bookkeeping outside SimState (batch.py:144-153): the running
 * episode return (f64[N]) / length (i64[N]) and the step counter that keys
 * the reset pool (WorldPool(pool_key, step_index + 1)).  Checkpoint/resume
 * and the rollout report (bench.run_rollout_report, bench.py:67-107). */
int gr_export_episode(gr_env *env, double *ep_return_host, int64_t *ep_length_host);
int gr_import_episode(gr_env *env, const double *ep_return_host, const int64_t *ep_length_host);
int gr_get_step_index(gr_env *env, int64_t *out);
int gr_set_step_index(gr_env *env, int64_t step_index);
/* encode the current state (no step): symbolic or pixels per obs_mode */
int gr_observe(gr_env *env, void *obs_dev, void *stream);

/* ---- level buffers (UED curricula; mutate.py, worldgen.py, state.py) ------ *
 * A device buffer of `capacity` levels: LevelParams (seed, 252 overworld
 * angles, 9 floor seeds) and the World generated from them.  All calls are
 * synchronous; index / key arrays are host memory. */
typedef struct gr_levels gr_levels;
enum { GR_MUT_NOISE = 0, GR_MUT_SWAP = 1, GR_MUT_RSWAP = 2 };
int gr_levels_create(gr_env *env, int64_t capacity, gr_levels **out);
void gr_levels_destroy(gr_levels *lv);
/* params of levels [first, first+count): angles / floor_seeds NULL =
 * worldgen.make_level_params(seed) (worldgen.py:75-87) */
int gr_levels_set_params(gr_levels *lv, int64_t first, int64_t count, const uint64_t *seeds,
                         const float *angles, const uint64_t *floor_seeds);
int gr_levels_get_params(gr_levels *lv, int64_t first, int64_t count, uint64_t *seeds, float *angles,
                         uint64_t *floor_seeds);
/* worldgen.generate_world(params) for levels [first, first+count) (worldgen.py:636-651) */
int gr_levels_generate(gr_levels *lv, int64_t first, int64_t count);
/* mutate.mutate_noise (params; regenerate after) / mutate_swap / mutate_rswap
 * (worlds, in place) of level_idx[k] with the RngStream (stream_key[k],
 * stream_counter[k]); scale: mutate_noise's range (mutate.NOISE_RANGE = 0.5) */
int gr_levels_mutate(gr_levels *lv, int32_t op, int64_t count, const int64_t *level_idx,
                     const uint64_t *stream_key, const uint64_t *stream_counter, double scale);
/* state.install_world(sim, env_idx[k], level level_idx[k], keys[k]) (state.py:169-249);
 * also clears the env's running episode return / length */
int gr_levels_install(gr_levels *lv, int64_t count, const int64_t *env_idx, const int64_t *level_idx,
                      const uint64_t *keys);
/* one World in the reference's layout: blocks / items [F][H][W], spawn[2],
 * ladders [F][4] (down r, c, up r, c; -1 none), chests [F][6][4] (r, c,
 * loot, qty; -1 rows pad), potion permutation [6] */
int gr_levels_export_world(gr_levels *lv, int64_t level, uint8_t *blocks, uint8_t *items, int16_t *spawn,
                           int16_t *ladders, int64_t *chests, uint8_t *potion);
/* the level's LevelParams seed and which floors are the _template_floor
 * fallback (bit f; their FloorMap.spawn is the map centre, worldgen.py:549-575,
 * while every generated lower floor spawns on its up ladder) */
int gr_levels_world_info(gr_levels *lv, int64_t level, uint64_t *seed, uint32_t *template_floors);
/* write a World (worldgen.World, e.g. read with serialize.world_from_bytes,
 * serialize.py:97-118) into level slot `level`, in the layout
 * gr_levels_export_world produces; seed = its LevelParams.seed.  The slot can
 * then be installed like a generated one. */
int gr_levels_import_world(gr_levels *lv, int64_t level, uint64_t seed, const uint8_t *blocks,
                           const uint8_t *items, const int16_t *spawn, const int16_t *ladders,
                           const int64_t *chests, const uint8_t *potion, uint32_t template_floors);

/* ---- metrics ------------------------------------------------------------- */
int gr_stats_get(gr_env *env, gr_stats *out);                 /* EpisodeStats */
int gr_stats_set(gr_env *env, const gr_stats *in);            /* restore (checkpoint / resume) */
int gr_level_seeds(gr_env *env, uint64_t *host_dst);          /* BatchState.level_seeds */
int gr_episodes_completed(gr_env *env, int64_t *out);         /* info["episodes_completed"] */
/* count of kernels this library launched since creation (bench evidence) */
int64_t gr_kernel_launches(const gr_env *env);
/* per-kernel device timing with CUDA events on the launching stream:
 * classes 0..9 = step, scan, info, worldgen, install, obs (writer, envs not
 * reset), policy, other, obs_reset (envs reset this step), obs_prep (the
 * per-env pass before the writer) */
int gr_set_profiling(gr_env *env, int32_t on);
int gr_kernel_times(gr_env *env, double *ms, int64_t *counts, int32_t n_classes);
/* worldgen diagnostics: [worlds generated, floors retried, template floors,
 * potion draws with ties (reproduced in numpy's order), 0 (reserved)] */
int gr_worldgen_counters(gr_env *env, int64_t out[5]);
/* worldgen.MAX_GEN_RETRIES (worldgen.py:36, default 16) for every later
 * world this handle generates (pool, reset, level buffers); 0 sends every
 * floor to the _template_floor fallback (worldgen.py:549-595) -- the hook the
 * parity tests use to reach that branch */
int gr_set_worldgen_attempts(gr_env *env, int32_t max_attempts);

/* ---- numerics self-test -------------------------------------------------- *
 * The exact device routines the kernels use where the reference's results
 * depend on its host libraries, exposed so tests can compare them with
 * numpy directly over large input sets (device pointers, async on stream):
 * float64 sin / cos of float32 angles as glibc computes them (the cave noise,
 * perlin.py:71-72 + worldgen.py:424), and np.argsort of six float32 keys in
 * numpy's AVX-512 tie order (the potion permutation, worldgen.py:647-649). */
int gr_selftest_sincos64(const float *x_dev, double *sin_dev, double *cos_dev, int64_t n, void *stream);
int gr_selftest_argsort6(const float *keys_dev, uint8_t *idx_dev, int64_t n, void *stream);

#ifdef __cplusplus
}
#endif
#endif
