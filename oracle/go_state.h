/*
 * go_state.h -- the oracle's native per-env state (TEST INFRASTRUCTURE).
 * One Env struct holds every non-map SimState field of one environment
 * (state.py:29-125) at extended-tier capacity; maps live in flat arrays.
 */
#ifndef GO_STATE_H
#define GO_STATE_H
#include "gr_oracle.h"
#include <stddef.h>

typedef struct {
  int16_t ladder_down[9][2], ladder_up[9][2], spawn0[2];
  uint8_t potion_map[6];
  int16_t chest_pos[9][6][2];
  uint8_t chest_loot[9][6], chest_qty[9][6], chest_aux[9][6];
  int16_t necro_pos[2];
  uint64_t params_seed;
  uint8_t pfloor;
  int16_t prow, pcol;
  uint8_t facing;
  float health, food, drink, energy, mana;
  uint8_t xp, dex, str_, intel, sword_tier, pick_tier, has_bow, sword_ench, bow_ench;
  uint8_t armour[4], armour_ench[4];
  uint8_t learned_fire, learned_ice, sleeping, resting;
  uint8_t inv_wood, inv_stone, inv_coal, inv_iron, inv_diamond, inv_sapphire, inv_ruby,
      inv_sapling, inv_torch, inv_arrow, inv_book, inv_potion[6];
  int16_t mel_pos[9][3][2];
  float mel_hp[9][3];
  uint8_t mel_cd[9][3], mel_alive[9][3], mel_type[9][3];
  int16_t ran_pos[9][2][2];
  float ran_hp[9][2];
  uint8_t ran_cd[9][2], ran_alive[9][2], ran_type[9][2];
  int16_t pas_pos[9][3][2];
  float pas_hp[9][3];
  uint8_t pas_alive[9][3], pas_type[9][3];
  int16_t pproj_pos[3][2];
  uint8_t pproj_dir[3], pproj_type[3], pproj_ttl[3], pproj_alive[3];
  float pproj_dmg[3][3];
  int16_t eproj_pos[3][2];
  uint8_t eproj_dir[3], eproj_type[3], eproj_ttl[3], eproj_alive[3];
  float eproj_dmg[3][3];
  int16_t plant_pos[10][2];
  uint16_t plant_age[10];
  uint8_t plant_alive[10];
  uint8_t ach[67];
  uint32_t time;
  uint64_t rng_key;
  uint8_t floors_visited[9], floor_cleared[9];
  float boss_hp;
  uint8_t boss_wave, boss_vuln, boss_timer;
  uint16_t clocks[6];
  uint8_t done;
} Env;

struct go_state {
  int64_t n;
  int classic, F, H, W, A, NA, VR, VC;
  int64_t max_len;
  Env *env;
  uint8_t *blocks, *items;   /* [n][F][H][W] */
};
typedef struct go_state go_state;

void gs_init(go_state *s, int classic, int64_t n, int64_t max_len);
void gs_free(go_state *s);
void gs_install(go_state *s, int64_t i, const go_world *w, uint64_t key);
typedef struct { uint8_t unlock[67]; uint8_t hurt; float health0; uint32_t base; } WS;
void gs_step_pass1(go_state *s, const int64_t *actions, WS *ws, int64_t lo, int64_t hi, int *flags);
void gs_step_pass2(go_state *s, WS *ws, int64_t lo, int64_t hi, const int *flags,
                   double *reward, uint8_t *done, uint8_t *newly, float *delta);
void gs_encode_symbolic(const go_state *s, int64_t i, int batch_dark, float *out);
void gs_render_pixels(const go_state *s, int64_t i, int px, uint8_t *out);
int gs_any_dark(const go_state *s);

#endif
