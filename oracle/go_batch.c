/*
 * go_batch.c -- oracle state lifecycle, reference-layout import/export, and
 * batch.py's auto-resetting batch_step with the optimistic world pool.
 * TEST INFRASTRUCTURE ONLY (see gr_oracle.h).
 */
#include "go_state.h"
#include "go_tables.h"

#include <stddef.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

void gs_init(go_state *s, int classic, int64_t n, int64_t max_len) {
  memset(s, 0, sizeof(*s));
  s->n = n;
  s->classic = classic;
  s->F = classic ? 1 : 9;
  s->H = s->W = classic ? 64 : 48;
  s->A = classic ? 22 : 67;
  s->NA = classic ? 17 : 43;
  s->VR = classic ? 7 : 9;
  s->VC = classic ? 9 : 11;
  s->max_len = max_len > 0 ? max_len : 100000;
  s->env = (Env *)calloc((size_t)n, sizeof(Env));
  size_t m = (size_t)n * s->F * s->H * s->W;
  s->blocks = (uint8_t *)calloc(m, 1);
  s->items = (uint8_t *)calloc(m, 1);
}

void gs_free(go_state *s) {
  free(s->env); free(s->blocks); free(s->items);
  memset(s, 0, sizeof(*s));
}

/* state._SHAPES (state.py:29-125): where each field lives in Env */
enum { K_MAP, K_F, K_FIX, K_A };
typedef struct { size_t off; int esz, kind, k; } fdesc;
#define FD(name, esz, kind, k) {offsetof(Env, name), esz, kind, k}
static const fdesc FIELDS[FO_NFIELDS] = {
  {0, 1, K_MAP, 0}, {0, 1, K_MAP, 0},
  FD(ladder_down, 2, K_F, 2), FD(ladder_up, 2, K_F, 2), FD(spawn0, 2, K_FIX, 2),
  FD(potion_map, 1, K_FIX, 6), FD(chest_pos, 2, K_F, 12), FD(chest_loot, 1, K_F, 6),
  FD(chest_qty, 1, K_F, 6), FD(chest_aux, 1, K_F, 6), FD(necro_pos, 2, K_FIX, 2),
  FD(params_seed, 8, K_FIX, 1),
  FD(pfloor, 1, K_FIX, 1), FD(prow, 2, K_FIX, 1), FD(pcol, 2, K_FIX, 1), FD(facing, 1, K_FIX, 1),
  FD(health, 4, K_FIX, 1), FD(food, 4, K_FIX, 1), FD(drink, 4, K_FIX, 1), FD(energy, 4, K_FIX, 1),
  FD(mana, 4, K_FIX, 1), FD(xp, 1, K_FIX, 1), FD(dex, 1, K_FIX, 1), FD(str_, 1, K_FIX, 1),
  FD(intel, 1, K_FIX, 1), FD(sword_tier, 1, K_FIX, 1), FD(pick_tier, 1, K_FIX, 1),
  FD(has_bow, 1, K_FIX, 1), FD(sword_ench, 1, K_FIX, 1), FD(bow_ench, 1, K_FIX, 1),
  FD(armour, 1, K_FIX, 4), FD(armour_ench, 1, K_FIX, 4), FD(learned_fire, 1, K_FIX, 1),
  FD(learned_ice, 1, K_FIX, 1), FD(sleeping, 1, K_FIX, 1), FD(resting, 1, K_FIX, 1),
  FD(inv_wood, 1, K_FIX, 1), FD(inv_stone, 1, K_FIX, 1), FD(inv_coal, 1, K_FIX, 1),
  FD(inv_iron, 1, K_FIX, 1), FD(inv_diamond, 1, K_FIX, 1), FD(inv_sapphire, 1, K_FIX, 1),
  FD(inv_ruby, 1, K_FIX, 1), FD(inv_sapling, 1, K_FIX, 1), FD(inv_torch, 1, K_FIX, 1),
  FD(inv_arrow, 1, K_FIX, 1), FD(inv_book, 1, K_FIX, 1), FD(inv_potion, 1, K_FIX, 6),
  FD(mel_pos, 2, K_F, 6), FD(mel_hp, 4, K_F, 3), FD(mel_cd, 1, K_F, 3), FD(mel_alive, 1, K_F, 3),
  FD(mel_type, 1, K_F, 3),
  FD(ran_pos, 2, K_F, 4), FD(ran_hp, 4, K_F, 2), FD(ran_cd, 1, K_F, 2), FD(ran_alive, 1, K_F, 2),
  FD(ran_type, 1, K_F, 2),
  FD(pas_pos, 2, K_F, 6), FD(pas_hp, 4, K_F, 3), FD(pas_alive, 1, K_F, 3), FD(pas_type, 1, K_F, 3),
  FD(pproj_pos, 2, K_FIX, 6), FD(pproj_dir, 1, K_FIX, 3), FD(pproj_type, 1, K_FIX, 3),
  FD(pproj_ttl, 1, K_FIX, 3), FD(pproj_alive, 1, K_FIX, 3), FD(pproj_dmg, 4, K_FIX, 9),
  FD(eproj_pos, 2, K_FIX, 6), FD(eproj_dir, 1, K_FIX, 3), FD(eproj_type, 1, K_FIX, 3),
  FD(eproj_ttl, 1, K_FIX, 3), FD(eproj_alive, 1, K_FIX, 3), FD(eproj_dmg, 4, K_FIX, 9),
  FD(plant_pos, 2, K_FIX, 20), FD(plant_age, 2, K_FIX, 10), FD(plant_alive, 1, K_FIX, 10),
  FD(ach, 1, K_A, 1), FD(time, 4, K_FIX, 1), FD(rng_key, 8, K_FIX, 1),
  FD(floors_visited, 1, K_F, 1), FD(floor_cleared, 1, K_F, 1),
  FD(boss_hp, 4, K_FIX, 1), FD(boss_wave, 1, K_FIX, 1), FD(boss_vuln, 1, K_FIX, 1),
  FD(boss_timer, 1, K_FIX, 1), FD(clocks, 2, K_FIX, 6), FD(done, 1, K_FIX, 1)};

static size_t per_env_bytes(const go_state *s, int fid) {
  const fdesc *d = &FIELDS[fid];
  if (d->kind == K_MAP) return (size_t)s->F * s->H * s->W;
  if (d->kind == K_F) return (size_t)s->F * d->k * d->esz;
  if (d->kind == K_A) return (size_t)s->A;
  return (size_t)d->k * d->esz;
}

static void xfer(go_state *s, void *const *fields, int to_state) {
  for (int fid = 0; fid < FO_NFIELDS; ++fid) {
    size_t b = per_env_bytes(s, fid);
    uint8_t *arr = (uint8_t *)fields[fid];
    if (!arr) continue;
    if (FIELDS[fid].kind == K_MAP) {
      uint8_t *m = fid == FO_BLOCKS ? s->blocks : s->items;
      if (to_state) memcpy(m, arr, b * s->n); else memcpy(arr, m, b * s->n);
      continue;
    }
    for (int64_t i = 0; i < s->n; ++i) {
      uint8_t *e = (uint8_t *)&s->env[i] + FIELDS[fid].off;
      if (to_state) memcpy(e, arr + i * b, b); else memcpy(arr + i * b, e, b);
    }
  }
}

go_state_t *go_state_new(int classic, int64_t n, int64_t max_len) {
  go_state *s = (go_state *)malloc(sizeof(go_state));
  gs_init(s, classic, n, max_len);
  return s;
}
void go_state_free(go_state_t *s) { gs_free(s); free(s); }
void go_state_import(go_state_t *s, void *const *fields) { xfer(s, fields, 1); }
void go_state_export(const go_state_t *s, void *const *fields) { xfer((go_state *)s, fields, 0); }

void go_state_install_seed(go_state_t *s, int64_t env, uint64_t world_seed, uint64_t key) {
  go_world *w = (go_world *)malloc(sizeof(go_world));
  go_generate_world(world_seed, s->classic, w);
  gs_install(s, env, w, key);
  free(w);
}

int64_t go_state_step(go_state_t *s, const int64_t *actions, double *reward, uint8_t *done,
                      uint8_t *newly, float *delta) {
  for (int64_t i = 0; i < s->n; ++i)
    if (actions[i] < 0 || actions[i] >= s->NA) return -1 - i;
  WS *ws = (WS *)malloc(sizeof(WS) * (size_t)(s->n ? s->n : 1));
  int fl[2] = {0, 0};
  gs_step_pass1(s, actions, ws, 0, s->n, fl);
  gs_step_pass2(s, ws, 0, s->n, fl, reward, done, newly, delta);
  free(ws);
  return 0;
}

void go_state_encode(const go_state_t *s, float *out) {
  int L = s->classic ? 1345 : 8268;
  int dark = gs_any_dark(s);
#pragma omp parallel for schedule(static) if (s->n >= 512)
  for (int64_t i = 0; i < s->n; ++i) gs_encode_symbolic(s, i, dark, out + (size_t)i * L);
}

void go_state_pixels(const go_state_t *s, int px, uint8_t *out) {
  size_t fr = (size_t)(s->VR + 2) * px * (s->VC + (s->classic ? 0 : 2)) * px * 3;
#pragma omp parallel for schedule(static) if (s->n >= 128)
  for (int64_t i = 0; i < s->n; ++i) gs_render_pixels(s, i, px, out + i * fr);
}

/* ------------------------------------------------------------- batch.py */

struct go_batch {
  go_state st;
  int threads, M;
  uint64_t pool_key;
  int64_t step_index;
  double *ep_return;
  int64_t *ep_length;
  WS *ws;
  int64_t episodes, total_steps;
  double total_return;
  int64_t ach_counts[67];
  int64_t *done_idx;
  int64_t k_local;
  go_world *worlds;
  int n_worlds_cap;
  int64_t env_offset, n_global;   /* shard of a larger batch (multi-rank) */
};

go_batch *go_batch_create(int classic, int64_t n, uint64_t seed, int reset_ratio, int64_t max_len,
                          int threads) {
  return go_batch_create_shard(classic, n, 0, n, seed, reset_ratio, max_len, threads);
}

/* one contiguous shard [env_offset, env_offset + n) of an n_global batch:
 * every key uses the global env index, the pool size is global */
go_batch *go_batch_create_shard(int classic, int64_t n, int64_t env_offset, int64_t n_global,
                                uint64_t seed, int reset_ratio, int64_t max_len, int threads) {
  go_batch *b = (go_batch *)calloc(1, sizeof(go_batch));
  gs_init(&b->st, classic, n, max_len);
  b->threads = threads > 0 ? threads : 1;
  b->env_offset = env_offset;
  b->n_global = n_global;
  b->M = (int)((n_global + reset_ratio - 1) / reset_ratio);
  if (b->M < 1) b->M = 1;
  /* batch.py:139-160 */
  uint64_t base = go_mix(seed);
  b->pool_key = go_hash2(base, go_hash2(1, 0));
  uint64_t env_key = go_hash2(base, go_hash2(0, 0));
  b->ep_return = (double *)calloc((size_t)n, sizeof(double));
  b->ep_length = (int64_t *)calloc((size_t)n, sizeof(int64_t));
  b->ws = (WS *)malloc(sizeof(WS) * (size_t)n);
  b->done_idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
#pragma omp parallel num_threads(b->threads)
  {
    go_world *w = (go_world *)malloc(sizeof(go_world));
#pragma omp for schedule(dynamic, 4)
    for (int64_t i = 0; i < n; ++i) {
      uint64_t ps = go_hash2(env_key, go_hash2((uint64_t)(env_offset + i), 0));
      uint64_t key = go_hash2(ps, go_hash2(1, 0));
      go_generate_world(ps, classic, w);
      gs_install(&b->st, i, w, key);
    }
    free(w);
  }
  return b;
}

void go_batch_destroy(go_batch *b) {
  gs_free(&b->st);
  free(b->ep_return); free(b->ep_length); free(b->ws); free(b->done_idx); free(b->worlds);
  free(b);
}

go_state_t *go_batch_state(go_batch *b) { return &b->st; }

/* batch.py:193-234 in three phases so that a sharded batch can exchange
 * the batch-wide quantities between them (the reference batch is global):
 *   a: validation + player actions/projectiles -> local `alive.any()` flags
 *   b: (global flags) creatures .. reward/done  -> local done count
 *   c: (global rank offset of this shard's first done env) pool + install */
int64_t go_batch_step_a(go_batch *b, const int64_t *actions, int *flags) {
  go_state *s = &b->st;
  int64_t n = s->n;
  for (int64_t i = 0; i < n; ++i)
    if (actions[i] < 0 || actions[i] >= s->NA) return -1 - i;
  int mel = 0, ran = 0;
  int T = b->threads;
  int64_t chunk = (n + T - 1) / T;
#pragma omp parallel for num_threads(T) reduction(| : mel, ran)
  for (int t = 0; t < T; ++t) {
    int64_t lo = t * chunk, hi = lo + chunk < n ? lo + chunk : n;
    int fl[2] = {0, 0};
    if (lo < hi) gs_step_pass1(s, actions, b->ws, lo, hi, fl);
    mel |= fl[0]; ran |= fl[1];
  }
  flags[0] = mel;
  flags[1] = ran;
  return 0;
}

int64_t go_batch_step_b(go_batch *b, const int *flags, double *reward, uint8_t *done, uint8_t *newly,
                        uint32_t *info_time, uint8_t *info_floor) {
  go_state *s = &b->st;
  int64_t n = s->n;
  int T = b->threads;
  int64_t chunk = (n + T - 1) / T;
  int fl[2] = {flags[0], flags[1]};
#pragma omp parallel for num_threads(T)
  for (int t = 0; t < T; ++t) {
    int64_t lo = t * chunk, hi = lo + chunk < n ? lo + chunk : n;
    if (lo < hi) gs_step_pass2(s, b->ws, lo, hi, fl, reward, done, newly, NULL);
  }
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i) {
    b->ep_return[i] += reward[i];
    b->ep_length[i] += 1;
    if (info_time) info_time[i] = s->env[i].time;
    if (info_floor) info_floor[i] = s->env[i].pfloor;
    if (done[i]) b->done_idx[k++] = i;
  }
  b->k_local = k;
  return k;
}

void go_batch_step_c(go_batch *b, int64_t offset) {
  go_state *s = &b->st;
  int T = b->threads;
  int64_t k = b->k_local;
  uint64_t step_key = go_hash2(b->pool_key, (uint64_t)(b->step_index + 1));
  if (k) {
    /* pool entry p holds slot (offset + p) % M; local done rank r uses entry r % M */
    int m = (int)(k < b->M ? k : b->M);
    if (m > b->n_worlds_cap) {
      free(b->worlds);
      b->worlds = (go_world *)malloc(sizeof(go_world) * (size_t)m);
      b->n_worlds_cap = m;
    }
#pragma omp parallel for num_threads(T) schedule(dynamic, 1)
    for (int j = 0; j < m; ++j)
      go_generate_world(go_hash2(step_key, (uint64_t)((offset + j) % b->M)), s->classic, &b->worlds[j]);
    for (int64_t r = 0; r < k; ++r) {
      int64_t i = b->done_idx[r];
      b->episodes += 1;
      b->total_return += b->ep_return[i];
      b->total_steps += b->ep_length[i];
      for (int a = 0; a < s->A; ++a) b->ach_counts[a] += s->env[i].ach[a];
    }
#pragma omp parallel for num_threads(T)
    for (int64_t r = 0; r < k; ++r) {
      int64_t i = b->done_idx[r];
      int p = (int)(r % b->M);
      uint64_t slot = (uint64_t)((offset + r) % b->M);
      gs_install(s, i, &b->worlds[p], go_hash2(step_key, (1ULL << 32) + slot));
      b->ep_return[i] = 0.0;
      b->ep_length[i] = 0;
    }
  }
  b->step_index += 1;
}

int64_t go_batch_step(go_batch *b, const int64_t *actions, double *reward, uint8_t *done,
                      uint8_t *newly, uint32_t *info_time, uint8_t *info_floor) {
  int fl[2];
  int64_t rc = go_batch_step_a(b, actions, fl);
  if (rc < 0) return rc;
  int64_t k = go_batch_step_b(b, fl, reward, done, newly, info_time, info_floor);
  go_batch_step_c(b, 0);
  return k;
}

/* the torch-glow flag of obs.py:236 for this shard (OR over shards = batch) */
int go_state_any_dark(const go_state_t *s) { return gs_any_dark(s); }

void go_state_encode_flag(const go_state_t *s, int dark, float *out) {
  int L = s->classic ? 1345 : 8268;
#pragma omp parallel for schedule(static) if (s->n >= 512)
  for (int64_t i = 0; i < s->n; ++i) gs_encode_symbolic(s, i, dark, out + (size_t)i * L);
}

void go_batch_stats(const go_batch *b, int64_t *episodes, double *total_return,
                    int64_t *total_steps, int64_t *ach_counts) {
  *episodes = b->episodes;
  *total_return = b->total_return;
  *total_steps = b->total_steps;
  if (ach_counts) memcpy(ach_counts, b->ach_counts, sizeof(int64_t) * b->st.A);
}

void go_batch_ep(const go_batch *b, double *ep_return, int64_t *ep_length) {
  memcpy(ep_return, b->ep_return, sizeof(double) * b->st.n);
  memcpy(ep_length, b->ep_length, sizeof(int64_t) * b->st.n);
}

/* policies.py:22-37 */
void go_random_actions(uint32_t seed, uint64_t t, int64_t env0, int64_t n, int n_actions,
                       int64_t *out) {
  uint32_t k = (uint32_t)((uint64_t)seed + t * 2654435761ULL);
  for (int64_t i = 0; i < n; ++i) {
    float u = go_vuniform32(k, (uint32_t)(env0 + i));
    out[i] = (int64_t)(u * (float)n_actions) % n_actions;
  }
}
