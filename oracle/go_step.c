/*
 * go_step.c -- oracle restatement of engine.py, creatures.py, _kern.py and
 * state.install_worlds.  TEST INFRASTRUCTURE ONLY (see gr_oracle.h).
 *
 * The reference evaluates each phase over the whole batch (numpy masks); a
 * per-env scalar restatement is equivalent because every effect is masked
 * per env, with one exception that this file reproduces explicitly: the
 * creature-cooldown decrement of creatures.py:312,345 runs over *all* lanes
 * (dead ones included) but only when some env of the batch has a live lane
 * of that class (`if alive.any()`, creatures.py:290,329).  gs_step therefore
 * runs in two passes: player actions + projectiles for every env, then the
 * batch-wide flags, then creatures onwards.
 */
#include "go_state.h"
#include "go_tables.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ helpers */

/* _kern.py:57-60 */
static float q1(float x) { return floorf(x * 10.0f + 0.5f) * 0.1f; }

/* _kern.py:63-66 */
static float resolve(const float d[3], const float df[3]) {
  float t0 = d[0] * (1.0f - df[0] / 100.0f);
  float t1 = d[1] * (1.0f - df[1] / 100.0f);
  float t2 = d[2] * (1.0f - df[2] / 100.0f);
  float s = (t0 + t1) + t2;
  if (s < 0.0f) s = 0.0f;
  return q1(s);
}

static float f32min(float a, float b) { return a < b ? a : b; }
static float f32max(float a, float b) { return a > b ? a : b; }


/* _kern.py:48-54 */
static float draw(const WS *ws, int sub, int lane) {
  return go_vuniform32(ws->base, (uint32_t)(sub * 64 + lane));
}

static void award(const go_state *s, WS *ws, int a) {
  if (a < s->A) ws->unlock[a] = 1;
}

#define MAPI(s, i, f, r, c) ((((i) * (s)->F + (f)) * (s)->H + (r)) * (s)->W + (c))

/* _kern.py:82-104 */
static uint8_t gblock(const go_state *s, int64_t i, int f, int r, int c) {
  if (r < 0 || r >= s->H || c < 0 || c >= s->W) return B_OOB;
  return s->blocks[MAPI(s, i, f, r, c)];
}
static uint8_t gitem(const go_state *s, int64_t i, int f, int r, int c) {
  if (r < 0 || r >= s->H || c < 0 || c >= s->W) return 0;
  return s->items[MAPI(s, i, f, r, c)];
}
static void sblock(go_state *s, int64_t i, int f, int r, int c, uint8_t v) {
  s->blocks[MAPI(s, i, f, r, c)] = v;
}

/* _kern.py:153-160 */
static void player_defense(const Env *e, float out[3]) {
  float phys = (float)(e->armour[0] + e->armour[1] + e->armour[2] + e->armour[3]) * 10.0f;
  int nf = 0, ni = 0;
  for (int k = 0; k < 4; ++k) {
    if (e->armour[k] > 0 && e->armour_ench[k] == 1) nf++;
    if (e->armour[k] > 0 && e->armour_ench[k] == 2) ni++;
  }
  out[0] = f32min(phys, 80.0f);
  out[1] = f32min((float)nf * 20.0f, 80.0f);
  out[2] = f32min((float)ni * 20.0f, 80.0f);
}

/* _kern.py:163-170 */
static void hurt_player(Env *e, WS *ws, float amount) {
  if (!(amount > 0.0f)) return;
  e->health = e->health - amount;
  e->health = q1(f32max(e->health, 0.0f));
  ws->hurt = 1;
}

static float food_max(const Env *e) { return 12.0f + (float)e->dex; }
static float health_max(const Env *e) { return 9.0f + (float)e->str_; }
static float mana_max(const Env *e) { return 16.0f + (float)e->intel; }
static uint8_t inv_add1(uint8_t v) { int x = v + 1; return (uint8_t)(x < 99 ? x : 99); }

/* lane views of one floor */
typedef struct {
  int16_t (*pos)[2];
  float *hp;
  uint8_t *cd, *alive, *type;
  int cap;
} Lanes;

static Lanes lanes_of(Env *e, int cls, int f) {
  Lanes L;
  if (cls == 0) { L.pos = e->mel_pos[f]; L.hp = e->mel_hp[f]; L.cd = e->mel_cd[f]; L.alive = e->mel_alive[f]; L.type = e->mel_type[f]; L.cap = 3; }
  else if (cls == 1) { L.pos = e->ran_pos[f]; L.hp = e->ran_hp[f]; L.cd = e->ran_cd[f]; L.alive = e->ran_alive[f]; L.type = e->ran_type[f]; L.cap = 2; }
  else { L.pos = e->pas_pos[f]; L.hp = e->pas_hp[f]; L.cd = NULL; L.alive = e->pas_alive[f]; L.type = e->pas_type[f]; L.cap = 3; }
  return L;
}

/* creatures.py:127-152 (the hp/alive writes land in L, which for the
 * extended tier's player melee is a discarded copy: H8) */
static void damage_creature(const go_state *s, Env *e, WS *ws, Lanes *L, int lane, const float dmg[3]) {
  int kind = L->type[lane];
  float dealt = resolve(dmg, CR_DEF[kind]);
  L->hp[lane] = q1(L->hp[lane] - dealt);
  int died = L->hp[lane] <= 0.0f && L->alive[lane] && dealt > 0.0f;
  if (!died) return;
  L->alive[lane] = 0;
  award(s, ws, DEFEAT_ACH[kind]);
  float meat = EAT_FOOD_T[kind];
  if (meat > 0.0f) {
    float fm = food_max(e);
    e->food = e->food + meat;
    e->food = q1(f32min(e->food, fm));
  }
}

/* creatures.py:166-179 */
static void check_boss_death(const go_state *s, int64_t i, Env *e, WS *ws) {
  if (!(e->boss_vuln && e->boss_hp <= 0.0f)) return;
  award(s, ws, 49);
  e->floor_cleared[8] = 1;
  e->boss_vuln = 0;
  sblock((go_state *)s, i, 8, e->necro_pos[0], e->necro_pos[1], B_PATH);
}

/* engine.py:91-100 */
static void melee_damage(const Env *e, float out[3]) {
  float phys = q1(SWORD_BASE[e->sword_tier] * (0.5f + (float)e->str_ * 0.5f));
  float elem = q1(phys * 0.5f);
  out[0] = phys;
  out[1] = e->sword_ench == 1 ? elem : 0.0f;
  out[2] = e->sword_ench == 2 ? elem : 0.0f;
}

static int occupied(Env *e, int f, int r, int c) {
  for (int cls = 0; cls < 3; ++cls) {
    Lanes L = lanes_of(e, cls, f);
    for (int l = 0; l < L.cap; ++l)
      if (L.alive[l] && L.pos[l][0] == r && L.pos[l][1] == c) return 1;
  }
  return 0;
}

/* engine.py:240-272 */
static void open_chest(go_state *s, int64_t i, Env *e, WS *ws, int af, int tr, int tc) {
  int lane = -1;
  for (int j = 0; j < 6; ++j)
    if (e->chest_loot[af][j] != LOOT_NOTHING && e->chest_pos[af][j][0] == tr && e->chest_pos[af][j][1] == tc) { lane = j; break; }
  if (lane < 0) return;
  int loot = e->chest_loot[af][lane], qty = e->chest_qty[af][lane], aux = e->chest_aux[af][lane];
  if (loot == LOOT_BOW) { e->has_bow = 1; award(s, ws, 52); }
  if (loot == LOOT_BOOK) e->inv_book = (uint8_t)(e->inv_book + qty);
  if (loot == LOOT_POTION) e->inv_potion[aux] = (uint8_t)(e->inv_potion[aux] + qty);
  if (loot == LOOT_ARROWS) e->inv_arrow = (uint8_t)(e->inv_arrow + qty);
  if (loot == LOOT_TORCHES) e->inv_torch = (uint8_t)(e->inv_torch + qty);
  if (e->inv_book > 99) e->inv_book = 99;
  for (int k = 0; k < 6; ++k) if (e->inv_potion[k] > 99) e->inv_potion[k] = 99;
  if (e->inv_arrow > 99) e->inv_arrow = 99;
  if (e->inv_torch > 99) e->inv_torch = 99;
  e->chest_loot[af][lane] = LOOT_NOTHING;
  sblock(s, i, af, tr, tc, B_PATH);
  award(s, ws, 61);
}

/* engine.py:143-237 */
static void do_interact(go_state *s, int64_t i, Env *e, WS *ws, int af) {
  int tr = e->prow + DIR_OFF[e->facing][0], tc = e->pcol + DIR_OFF[e->facing][1];
  /* act0: classic aliases the state; extended works on a throwaway copy */
  Env copy;
  Env *tgt = e;
  if (!s->classic) { memcpy(&copy, e, sizeof(Env)); tgt = &copy; }
  for (int cls = 0; cls < 3; ++cls) {
    Lanes L = lanes_of(tgt, cls, af);
    int lane = -1;
    for (int l = 0; l < L.cap; ++l)
      if (L.alive[l] && L.pos[l][0] == tr && L.pos[l][1] == tc) { lane = l; break; }
    if (lane >= 0) {
      float dmg[3];
      melee_damage(e, dmg);
      /* the food/award side effects apply to the real env */
      int kind = L.type[lane];
      float dealt = resolve(dmg, CR_DEF[kind]);
      L.hp[lane] = q1(L.hp[lane] - dealt);
      int died = L.hp[lane] <= 0.0f && L.alive[lane] && dealt > 0.0f;
      if (died) {
        L.alive[lane] = 0;
        award(s, ws, DEFEAT_ACH[kind]);
        float meat = EAT_FOOD_T[kind];
        if (meat > 0.0f) {
          float fm = food_max(e);
          e->food = e->food + meat;
          e->food = q1(f32min(e->food, fm));
        }
      }
      return;
    }
  }
  uint8_t tb = gblock(s, i, af, tr, tc);
  if (tb == B_TREE || tb == B_FIRE_TREE || tb == B_ICE_SHRUB) {
    e->inv_wood = inv_add1(e->inv_wood);
    award(s, ws, 0);
  }
  if (tb == B_GRASS) {
    if (draw(ws, 1, 0) < 0.1f) {
      e->inv_sapling = inv_add1(e->inv_sapling);
      award(s, ws, 3);
    }
  }
  if (tb == B_WATER || tb == B_FOUNTAIN) {
    e->drink = q1(f32min(e->drink + 1.0f, food_max(e)));
    award(s, ws, 4);
    if (tb == B_FOUNTAIN) e->mana = q1(f32min(e->mana + 1.0f, mana_max(e)));
  }
  /* MINEABLE dict order (constants.py:450-458) */
  {
    int req = -1, ach = -1;
    uint8_t *inv = NULL;
    switch (tb) {
      case B_STONE: req = 1; ach = 9; inv = &e->inv_stone; break;
      case B_COAL: req = 1; ach = 17; inv = &e->inv_coal; break;
      case B_STALAGMITE: req = 1; ach = -1; inv = &e->inv_stone; break;
      case B_IRON: req = 2; ach = 18; inv = &e->inv_iron; break;
      case B_DIAMOND: req = 3; ach = 19; inv = &e->inv_diamond; break;
      case B_SAPPHIRE: req = 3; ach = 54; inv = &e->inv_sapphire; break;
      case B_RUBY: req = 4; ach = 59; inv = &e->inv_ruby; break;
      default: break;
    }
    if (req >= 0 && e->pick_tier >= req) {
      *inv = inv_add1(*inv);
      sblock(s, i, af, tr, tc, B_PATH);
      if (ach >= 0) award(s, ws, ach);
    }
  }
  if (tb == B_RIPE_PLANT) {
    e->food = q1(f32min(e->food + 4.0f, food_max(e)));
    award(s, ws, 11);
    sblock(s, i, af, tr, tc, B_PLANT);
    for (int l = 0; l < 10; ++l)
      if (e->plant_alive[l] && e->plant_pos[l][0] == tr && e->plant_pos[l][1] == tc) e->plant_age[l] = 0;
  }
  if (!s->classic) {
    if (tb == B_CHEST) open_chest(s, i, e, ws, af, tr, tc);
    if (tb == B_NECROMANCER_VULN && e->boss_vuln) {
      float dmg[3], zero[3] = {0, 0, 0};
      melee_damage(e, dmg);
      float dealt = resolve(dmg, zero);
      e->boss_hp -= dealt;
      award(s, ws, 48);
      check_boss_death(s, i, e, ws);
    }
  }
}

/* engine.py:275-336 */
static void place_action(go_state *s, int64_t i, Env *e, WS *ws, int a, int af) {
  int tr = e->prow + DIR_OFF[e->facing][0], tc = e->pcol + DIR_OFF[e->facing][1];
  uint8_t tb = gblock(s, i, af, tr, tc);
  uint8_t ti = gitem(s, i, af, tr, tc);
  int open = ti == I_EMPTY && !occupied(e, af, tr, tc);
  if (a == 7 && e->inv_stone > 0 && PLACE_STONE_OK[tb] && open) {
    sblock(s, i, af, tr, tc, B_STONE); award(s, ws, 10); e->inv_stone -= 1;
  }
  if (a == 8 && e->inv_wood > 0 && PLACE_SOLID_OK[tb] && open) {
    sblock(s, i, af, tr, tc, B_TABLE); award(s, ws, 1); e->inv_wood -= 1;
  }
  if (a == 9 && e->inv_stone > 0 && PLACE_SOLID_OK[tb] && open) {
    sblock(s, i, af, tr, tc, B_FURNACE); award(s, ws, 16); e->inv_stone -= 1;
  }
  if (a == 10 && e->inv_sapling > 0 && tb == B_GRASS && open && af == 0) {
    int slot = -1;
    for (int l = 0; l < 10; ++l) if (!e->plant_alive[l]) { slot = l; break; }
    if (slot >= 0) {
      sblock(s, i, af, tr, tc, B_PLANT); award(s, ws, 7);
      e->plant_pos[slot][0] = (int16_t)tr; e->plant_pos[slot][1] = (int16_t)tc;
      e->plant_age[slot] = 0; e->plant_alive[slot] = 1;
      e->inv_sapling -= 1;
    }
  }
  if (!s->classic && a == 28 && e->inv_torch > 0 && WALKABLE_T[tb] && open) {
    s->items[MAPI(s, i, af, tr, tc)] = I_TORCH;
    e->inv_torch -= 1;
    award(s, ws, 24);
  }
}

/* engine.py:346-457 */
static void craft_action(go_state *s, int64_t i, Env *e, WS *ws, int a, int af) {
  int near_table = 0, near_furnace = 0, near_fire = 0, near_ice = 0;
  for (int dr = -1; dr <= 1; ++dr)
    for (int dc = -1; dc <= 1; ++dc) {
      uint8_t b = gblock(s, i, af, e->prow + dr, e->pcol + dc);
      near_table |= b == B_TABLE; near_furnace |= b == B_FURNACE;
      near_fire |= b == B_ENCHANT_TABLE_FIRE; near_ice |= b == B_ENCHANT_TABLE_ICE;
    }
  /* the eight tool recipes (engine.py:54-77) */
  static const struct { int action, pick, level, wood, stone, coal, iron, diamond, furnace, ach; } R[8] = {
      {11, 1, 1, 1, 0, 0, 0, 0, 0, 5},  {12, 1, 2, 1, 1, 0, 0, 0, 0, 13},
      {13, 1, 3, 1, 0, 1, 1, 0, 1, 20}, {20, 1, 4, 1, 0, 0, 0, 2, 0, 60},
      {14, 0, 1, 1, 0, 0, 0, 0, 0, 6},  {15, 0, 2, 1, 1, 0, 0, 0, 0, 14},
      {16, 0, 3, 1, 0, 1, 1, 0, 1, 21}, {21, 0, 4, 1, 0, 0, 0, 2, 0, 25}};
  for (int k = 0; k < 8; ++k) {
    if (R[k].action >= s->NA || a != R[k].action) continue;
    uint8_t *tool = R[k].pick ? &e->pick_tier : &e->sword_tier;
    if (!(*tool < R[k].level) || !near_table) continue;
    if (R[k].furnace && !near_furnace) continue;
    if (e->inv_wood < R[k].wood || e->inv_stone < R[k].stone || e->inv_coal < R[k].coal ||
        e->inv_iron < R[k].iron || e->inv_diamond < R[k].diamond) continue;
    e->inv_wood -= R[k].wood; e->inv_stone -= R[k].stone; e->inv_coal -= R[k].coal;
    e->inv_iron -= R[k].iron; e->inv_diamond -= R[k].diamond;
    *tool = (uint8_t)R[k].level;
    award(s, ws, R[k].ach);
  }
  if (s->classic) return;
  if (a == 25 && near_table && e->inv_wood >= 1 && e->inv_stone >= 1) {
    e->inv_wood -= 1; e->inv_stone -= 1;
    int x = e->inv_arrow + 2; e->inv_arrow = (uint8_t)(x < 99 ? x : 99);
    award(s, ws, 22);
  }
  if (a == 38 && e->inv_wood >= 1 && e->inv_coal >= 1) {
    e->inv_wood -= 1; e->inv_coal -= 1;
    int x = e->inv_torch + 4; e->inv_torch = (uint8_t)(x < 99 ? x : 99);
    award(s, ws, 23);
  }
  if (a == 22 && near_table && near_furnace && e->inv_iron >= 2 && e->inv_coal >= 1) {
    int slot = 0;
    for (int k = 1; k < 4; ++k) if (e->armour[k] < e->armour[slot]) slot = k;
    if (e->armour[slot] < 1) {
      e->armour[slot] = 1; e->inv_iron -= 2; e->inv_coal -= 1; award(s, ws, 26);
    }
  }
  if (a == 23 && near_table && e->inv_diamond >= 2) {
    int slot = 0;
    for (int k = 1; k < 4; ++k) if (e->armour[k] < e->armour[slot]) slot = k;
    if (e->armour[slot] < 2) {
      e->armour[slot] = 2; e->inv_diamond -= 2; award(s, ws, 27);
    }
  }
  if (a == 36 || a == 37 || a == 42) {
    int can_fire = near_fire && e->inv_ruby >= 1 && e->mana >= 2.0f;
    int can_ice = near_ice && e->inv_sapphire >= 1 && e->mana >= 2.0f;
    if ((a == 36 && e->sword_tier > 0) || (a == 42 && e->has_bow)) {
      uint8_t *slot = a == 36 ? &e->sword_ench : &e->bow_ench;
      if (can_fire) {
        *slot = 1; e->inv_ruby -= 1; e->mana -= 2.0f;
        if (a == 36) award(s, ws, 63);
      } else if (can_ice) {
        *slot = 2; e->inv_sapphire -= 1; e->mana -= 2.0f;
        if (a == 36) award(s, ws, 63);
      }
    }
    if (a == 37) {
      int slot = -1;
      for (int k = 0; k < 4; ++k) if (e->armour[k] > 0 && e->armour_ench[k] == 0) { slot = k; break; }
      if (slot >= 0) {
        if (can_fire) { e->armour_ench[slot] = 1; e->inv_ruby -= 1; e->mana -= 2.0f; award(s, ws, 64); }
        else if (can_ice) { e->armour_ench[slot] = 2; e->inv_sapphire -= 1; e->mana -= 2.0f; award(s, ws, 64); }
      }
    }
  }
}

/* engine.py:111-125 */
static int spawn_pproj(Env *e, int kind, const float dmg[3]) {
  int slot = -1;
  for (int l = 0; l < 3; ++l) if (!e->pproj_alive[l]) { slot = l; break; }
  if (slot < 0) return 0;
  e->pproj_pos[slot][0] = e->prow; e->pproj_pos[slot][1] = e->pcol;
  e->pproj_dir[slot] = e->facing; e->pproj_type[slot] = (uint8_t)kind;
  e->pproj_ttl[slot] = 6;
  for (int k = 0; k < 3; ++k) e->pproj_dmg[slot][k] = dmg[k];
  e->pproj_alive[slot] = 1;
  return 1;
}

/* engine.py:533-565 */
static void ladder_move(go_state *s, int64_t i, Env *e, WS *ws, int a) {
  uint8_t here = gitem(s, i, e->pfloor, e->prow, e->pcol);
  int down = a == 18 && here == I_LADDER_DOWN && e->pfloor + 1 < s->F;
  int up = a == 19 && here == I_LADDER_UP && e->pfloor > 0;
  if (!down && !up) return;
  int nf = e->pfloor + (down ? 1 : -1);
  e->pfloor = (uint8_t)nf;
  if (down) { e->prow = e->ladder_up[nf][0]; e->pcol = e->ladder_up[nf][1]; }
  else { e->prow = e->ladder_down[nf][0]; e->pcol = e->ladder_down[nf][1]; }
  for (int l = 0; l < 3; ++l) { e->pproj_alive[l] = 0; e->eproj_alive[l] = 0; }
  if (!e->floors_visited[nf]) {
    e->floors_visited[nf] = 1;
    uint8_t x = (uint8_t)(e->xp + 1);
    e->xp = x < 255 ? x : 255;
    if (ENTER_ACH[nf] != 255) award(s, ws, ENTER_ACH[nf]);
  }
}

/* engine.py:568-633 */
static void player_actions(go_state *s, int64_t i, Env *e, WS *ws, int action) {
  int eff = (e->sleeping || e->resting) ? 0 : action;
  int af = e->pfloor;
  if (eff >= 1 && eff <= 4) {
    e->facing = (uint8_t)(eff - 1);
    int tr = e->prow + DIR_OFF[e->facing][0], tc = e->pcol + DIR_OFF[e->facing][1];
    uint8_t tb = gblock(s, i, af, tr, tc);
    if (WALKABLE_T[tb] && !occupied(e, af, tr, tc)) { e->prow = (int16_t)tr; e->pcol = (int16_t)tc; }
  }
  if (eff == 5) do_interact(s, i, e, ws, af);
  if (eff == 6 && !e->sleeping && e->energy < food_max(e)) e->sleeping = 1;
  if ((eff >= 7 && eff <= 10) || (!s->classic && eff == 28)) place_action(s, i, e, ws, eff, af);
  if ((eff >= 11 && eff <= 16) ||
      (!s->classic && (eff == 20 || eff == 21 || eff == 22 || eff == 23 || eff == 25 || eff == 38 ||
                       eff == 36 || eff == 37 || eff == 42)))
    craft_action(s, i, e, ws, eff, af);
  if (s->classic) return;
  if (eff == 17) e->resting = 1;
  if (eff == 18 || eff == 19) ladder_move(s, i, e, ws, eff);
  if (eff == 24 && e->has_bow && e->inv_arrow > 0) {
    float phys = q1(3.0f + (float)e->dex);
    float elem = q1(phys * 0.5f);
    float dmg[3] = {phys, e->bow_ench == 1 ? elem : 0.0f, e->bow_ench == 2 ? elem : 0.0f};
    if (spawn_pproj(e, 0, dmg)) { e->inv_arrow -= 1; award(s, ws, 53); }
  }
  if (eff == 26 && e->learned_fire && e->mana >= 2.0f) {
    float dmg[3] = {0.0f, 6.0f + (float)e->intel, 0.0f};
    if (spawn_pproj(e, 1, dmg)) { e->mana = q1(e->mana - 2.0f); award(s, ws, 56); }
  }
  if (eff == 27 && e->learned_ice && e->mana >= 2.0f) {
    float dmg[3] = {0.0f, 0.0f, 6.0f + (float)e->intel};
    if (spawn_pproj(e, 2, dmg)) { e->mana = q1(e->mana - 2.0f); award(s, ws, 58); }
  }
  /* engine.py:473-517 */
  if (eff >= 29 && eff <= 34) {
    int color = eff - 29;
    if (e->inv_potion[color] > 0) {
      e->inv_potion[color] -= 1;
      int effect = e->potion_map[color];
      if (effect == 0) e->health = q1(f32min(e->health + 8.0f, health_max(e)));
      if (effect == 1) e->mana = q1(f32min(e->mana + 8.0f, mana_max(e)));
      if (effect == 2) e->energy = q1(f32min(e->energy + 8.0f, food_max(e)));
      if (effect == 3) hurt_player(e, ws, 3.0f);
      if (effect == 4) e->mana = q1(f32max(e->mana - 3.0f, 0.0f));
      if (effect == 5) {
        e->food = q1(f32min(e->food + 4.0f, food_max(e)));
        e->drink = q1(f32min(e->drink + 4.0f, food_max(e)));
      }
      award(s, ws, 62);
    }
  }
  if (eff == 35 && e->inv_book > 0) {
    int lf = !e->learned_fire, li = e->learned_fire && !e->learned_ice;
    if (lf || li) e->inv_book -= 1;
    if (lf) { e->learned_fire = 1; award(s, ws, 55); }
    if (li) { e->learned_ice = 1; award(s, ws, 57); }
  }
  /* engine.py:520-530 */
  if (e->xp >= 1) {
    if (eff == 39 && e->dex < 5) { e->dex += 1; e->xp -= 1; }
    if (eff == 40 && e->str_ < 5) { e->str_ += 1; e->xp -= 1; }
    if (eff == 41 && e->intel < 5) { e->intel += 1; e->xp -= 1; }
  }
}

/* creatures.py:182-231 */
static void advance_projectiles(go_state *s, int64_t i, Env *e, WS *ws) {
  int af = e->pfloor;
  if (!s->classic) {
    for (int l = 0; l < 3; ++l)
      if (e->pproj_alive[l]) {
        e->pproj_pos[l][0] += DIR_OFF[e->pproj_dir[l]][0];
        e->pproj_pos[l][1] += DIR_OFF[e->pproj_dir[l]][1];
      }
    for (int l = 0; l < 3; ++l) {
      if (!e->pproj_alive[l]) continue;
      int r = e->pproj_pos[l][0], c = e->pproj_pos[l][1];
      int live = 1;
      for (int cls = 0; cls < 3 && live; ++cls) {
        Lanes L = lanes_of(e, cls, af);
        for (int k = 0; k < L.cap; ++k)
          if (L.alive[k] && L.pos[k][0] == r && L.pos[k][1] == c) {
            damage_creature(s, e, ws, &L, k, e->pproj_dmg[l]);
            live = 0;
            break;
          }
      }
      if (live && e->boss_vuln && r == e->necro_pos[0] && c == e->necro_pos[1]) {
        float zero[3] = {0, 0, 0};
        e->boss_hp -= resolve(e->pproj_dmg[l], zero);
        award(s, ws, 48);
        check_boss_death(s, i, e, ws);
      }
      uint8_t blk = gblock(s, i, af, r, c);
      int stopped = !live || BLOCKS_PROJ[blk] || e->pproj_ttl[l] <= 1;
      e->pproj_ttl[l] -= 1;
      if (stopped) e->pproj_alive[l] = 0;
    }
  }
  int any = e->eproj_alive[0] | e->eproj_alive[1] | e->eproj_alive[2];
  if (!any) return;
  int at[3];
  for (int l = 0; l < 3; ++l) {
    if (e->eproj_alive[l]) {
      e->eproj_pos[l][0] += DIR_OFF[e->eproj_dir[l]][0];
      e->eproj_pos[l][1] += DIR_OFF[e->eproj_dir[l]][1];
    }
    at[l] = e->eproj_alive[l] && e->eproj_pos[l][0] == e->prow && e->eproj_pos[l][1] == e->pcol;
  }
  if (at[0] || at[1] || at[2]) {
    float pdef[3], d[3];
    player_defense(e, pdef);
    for (int l = 0; l < 3; ++l) d[l] = at[l] ? resolve(e->eproj_dmg[l], pdef) : 0.0f;
    float total = (d[0] + d[1]) + d[2];
    hurt_player(e, ws, total);
    for (int l = 0; l < 3; ++l) if (at[l]) e->eproj_alive[l] = 0;
  }
  for (int l = 0; l < 3; ++l) {
    if (!e->eproj_alive[l]) continue;
    if (BLOCKS_PROJ[gblock(s, i, af, e->eproj_pos[l][0], e->eproj_pos[l][1])]) { e->eproj_alive[l] = 0; continue; }
    e->eproj_ttl[l] -= 1;
    if (!(e->eproj_ttl[l] > 0)) e->eproj_alive[l] = 0;
  }
}

static int sgn(int x) { return (x > 0) - (x < 0); }

/* creatures.py:243-256: move one lane if the target is walkable for it */
static void move_lane(go_state *s, int64_t i, Env *e, int af, Lanes *L, int l, int sr, int sc) {
  int tr = L->pos[l][0] + sr, tc = L->pos[l][1] + sc;
  uint8_t b = gblock(s, i, af, tr, tc);
  int coll = s->classic ? 0 : CR_COLL[L->type[l]];
  if (COLL_WALK[coll][b] && !(tr == e->prow && tc == e->pcol)) {
    L->pos[l][0] = (int16_t)tr; L->pos[l][1] = (int16_t)tc;
  }
}

/* creatures.py:259-284 */
static void chase_move(go_state *s, int64_t i, Env *e, int af, Lanes *L, int l, int dr, int dc) {
  int sr = sgn(dr), sc = sgn(dc);
  int row_first = abs(dr) >= abs(dc);
  int pr = row_first ? sr : 0, pc = row_first ? 0 : sc;
  int qr = sr - pr, qc = sc - pc;
  int coll = s->classic ? 0 : CR_COLL[L->type[l]];
  int t1r = L->pos[l][0] + pr, t1c = L->pos[l][1] + pc;
  int t2r = L->pos[l][0] + qr, t2c = L->pos[l][1] + qc;
  int ok1 = COLL_WALK[coll][gblock(s, i, af, t1r, t1c)] && !(t1r == e->prow && t1c == e->pcol);
  int ok2 = COLL_WALK[coll][gblock(s, i, af, t2r, t2c)] && !(t2r == e->prow && t2c == e->pcol);
  if (ok1) { L->pos[l][0] = (int16_t)t1r; L->pos[l][1] = (int16_t)t1c; }
  else if (ok2) { L->pos[l][0] = (int16_t)t2r; L->pos[l][1] = (int16_t)t2c; }
}

/* creatures.py:287-382; mel_any/ran_any are the batch-wide `alive.any()` */
static void creatures_act(go_state *s, int64_t i, Env *e, WS *ws, int mel_any, int ran_any) {
  int af = e->pfloor;
  if (mel_any) {
    Lanes L = lanes_of(e, 0, af);
    int dr[3], dc[3], cheb_[3], adj[3], attack[3];
    for (int l = 0; l < 3; ++l) {
      dr[l] = e->prow - L.pos[l][0]; dc[l] = e->pcol - L.pos[l][1];
      cheb_[l] = abs(dr[l]) > abs(dc[l]) ? abs(dr[l]) : abs(dc[l]);
      adj[l] = abs(dr[l]) + abs(dc[l]) == 1;
      attack[l] = L.alive[l] && adj[l] && L.cd[l] == 0;
    }
    if (attack[0] || attack[1] || attack[2]) {
      float d[3];
      if (s->classic) {
        for (int l = 0; l < 3; ++l) d[l] = attack[l] ? DEALT_BARE[L.type[l]] : 0.0f;
      } else {
        float pdef[3];
        player_defense(e, pdef);
        for (int l = 0; l < 3; ++l) d[l] = attack[l] ? resolve(CR_DMG[L.type[l]], pdef) : 0.0f;
      }
      hurt_player(e, ws, (d[0] + d[1]) + d[2]);
    }
    for (int l = 0; l < 3; ++l) {
      if (L.cd[l] > 0) L.cd[l] -= 1;
      if (attack[l]) L.cd[l] = 2;
    }
    for (int l = 0; l < 3; ++l) {
      if (!L.alive[l] || adj[l]) continue;
      if (cheb_[l] <= 6) chase_move(s, i, e, af, &L, l, dr[l], dc[l]);
      else {
        float u = draw(ws, 2, l);
        if (u < 0.25f) {
          int d = (int)(u * 16.0f) % 4;
          if (d > 3) d = 3;
          move_lane(s, i, e, af, &L, l, DIR_OFF[d][0], DIR_OFF[d][1]);
        }
      }
    }
  }
  if (ran_any) {
    Lanes L = lanes_of(e, 1, af);
    int dr[2], dc[2], cheb_[2], shoot[2];
    for (int l = 0; l < 2; ++l) {
      dr[l] = e->prow - L.pos[l][0]; dc[l] = e->pcol - L.pos[l][1];
      cheb_[l] = abs(dr[l]) > abs(dc[l]) ? abs(dr[l]) : abs(dc[l]);
      int aligned = (dr[l] == 0 || dc[l] == 0) && cheb_[l] >= 1;
      int in_range = L.alive[l] && aligned && cheb_[l] <= 5;
      shoot[l] = in_range && L.cd[l] == 0;
      if (shoot[l]) {
        int sr = sgn(dr[l]), sc = sgn(dc[l]);
        for (int k = 1; k < 5; ++k) {
          if (!(k < cheb_[l])) continue;
          if (BLOCKS_PROJ[gblock(s, i, af, L.pos[l][0] + sr * k, L.pos[l][1] + sc * k)]) { shoot[l] = 0; break; }
        }
      }
    }
    for (int l = 0; l < 2; ++l) {
      if (L.cd[l] > 0) L.cd[l] -= 1;
      if (shoot[l]) L.cd[l] = 6;
    }
    for (int l = 0; l < 2; ++l) {
      if (!shoot[l]) continue;
      int slot = -1;
      for (int k = 0; k < 3; ++k) if (!e->eproj_alive[k]) { slot = k; break; }
      if (slot < 0) continue;
      int kind = L.type[l];
      uint8_t dir = dr[l] == 0 ? (dc[l] > 0 ? 1 : 0) : (dr[l] > 0 ? 3 : 2);
      e->eproj_pos[slot][0] = L.pos[l][0]; e->eproj_pos[slot][1] = L.pos[l][1];
      e->eproj_dir[slot] = dir;
      e->eproj_type[slot] = RANGED_PROJ[kind];
      e->eproj_ttl[slot] = 6;
      for (int k = 0; k < 3; ++k) e->eproj_dmg[slot][k] = CR_DMG[kind][k];
      e->eproj_alive[slot] = 1;
    }
    for (int l = 0; l < 2; ++l)
      if (L.alive[l] && !shoot[l] && cheb_[l] <= 6 && cheb_[l] > 2)
        chase_move(s, i, e, af, &L, l, dr[l], dc[l]);
  }
  {
    Lanes L = lanes_of(e, 2, af);
    for (int l = 0; l < 3; ++l) {
      if (!L.alive[l]) continue;
      float u = draw(ws, 3, l);
      if (!(u < 0.5f)) continue;
      int d = (int)(u * 16.0f) % 4;
      if (d > 3) d = 3;
      move_lane(s, i, e, af, &L, l, DIR_OFF[d][0], DIR_OFF[d][1]);
    }
  }
}

/* engine.py:640-700 */
static void survival_tick(go_state *s, Env *e, WS *ws) {
  uint16_t dex = e->dex;
  float hmax = health_max(e), fmax = food_max(e);
  for (int k = 0; k < 4; ++k) e->clocks[k] = (uint16_t)(e->clocks[k] + 1);
  static const uint16_t base[3] = {30, 20, 40};
  int due[3];
  for (int k = 0; k < 3; ++k) due[k] = e->clocks[k] >= (uint16_t)(base[k] * dex);
  int starve = due[0], parch = due[1], tire = due[2];
  if (e->sleeping) {
    int recover = e->clocks[2] >= 2;
    tire = 0;
    if (recover) { e->energy = f32min(e->energy + 1.0f, fmax); e->clocks[2] = 0; }
  }
  if (starve) e->food = e->food - 1.0f;
  if (parch) e->drink = e->drink - 1.0f;
  if (tire) e->energy = e->energy - 1.0f;
  for (int k = 0; k < 3; ++k) if (due[k]) e->clocks[k] = 0;
  if (due[0] || due[1] || due[2]) {
    e->food = f32max(e->food, 0.0f);
    e->drink = f32max(e->drink, 0.0f);
    e->energy = f32max(e->energy, 0.0f);
  }
  if (e->clocks[3] >= 10) { e->mana = f32min(e->mana + 1.0f, mana_max(e)); e->clocks[3] = 0; }
  float depleted = (float)(e->food <= 0.0f) + (float)(e->drink <= 0.0f);
  depleted = depleted + (float)(e->energy <= 0.0f);
  int starving = depleted > 0.0f;
  e->clocks[4] = starving ? (uint16_t)(e->clocks[4] + 1) : 0;
  if (e->clocks[4] >= 10) { hurt_player(e, ws, depleted); e->clocks[4] = 0; }
  int healthy = !starving && e->health < hmax && e->health > 0.0f;
  e->clocks[5] = healthy ? (uint16_t)(e->clocks[5] + 1) : 0;
  if (e->clocks[5] >= 30) { e->health = q1(f32min(e->health + 1.0f, hmax)); e->clocks[5] = 0; }
  if (e->sleeping) {
    int woke = e->energy >= fmax;
    if (woke) { e->sleeping = 0; award(s, ws, 15); }
    if (ws->hurt) e->sleeping = 0;
  }
  if (!s->classic && e->resting) {
    if (ws->hurt) e->resting = 0;
    if (e->health >= hmax || starving) e->resting = 0;
  }
}

/* creatures.py:387-423 */
static void spawn_class(go_state *s, int64_t i, Env *e, WS *ws, int cls, int kind, double prob, int sub) {
  int af = e->pfloor;
  Lanes L = lanes_of(e, cls, af);
  int n_alive = 0;
  for (int l = 0; l < L.cap; ++l) n_alive += L.alive[l];
  float u = draw(ws, sub, 0);
  if (!((double)u < prob) || !(n_alive < L.cap) || kind < 0) return;
  float u1 = draw(ws, sub, 1), u2 = draw(ws, sub, 2);
  int off_r = (int)(int16_t)(u1 * 21.0f) - 10;
  int off_c = (int)(int16_t)(u2 * 21.0f) - 10;
  int dist = abs(off_r) > abs(off_c) ? abs(off_r) : abs(off_c);
  if (!(dist >= 5 && dist <= 10)) return;
  int r = e->prow + off_r, c = e->pcol + off_c;
  uint8_t b = gblock(s, i, af, r, c);
  if (!COLL_WALK[CR_COLL[kind]][b]) return;
  if (cls == 1 && !(b == B_PATH || af != 0)) return;
  int slot = -1;
  for (int l = 0; l < L.cap; ++l) if (!L.alive[l]) { slot = l; break; }
  L.pos[slot][0] = (int16_t)r; L.pos[slot][1] = (int16_t)c;
  L.hp[slot] = CR_HP[kind];
  L.type[slot] = (uint8_t)kind;
  if (cls != 2) L.cd[slot] = 0;
  L.alive[slot] = 1;
}

/* creatures.py:455-486 */
static void spawn_wave(go_state *s, Env *e, int wf) {
  int nr = e->necro_pos[0], nc = e->necro_pos[1];
  uint8_t mk = (uint8_t)MEL_KIND[wf], rk = (uint8_t)RAN_KIND[wf];
  static const int off[2][2] = {{2, -2}, {2, 2}};
  for (int l = 0; l < 2; ++l) {
    int r = nr + off[l][0], c = nc + off[l][1];
    if (r == e->prow && c == e->pcol) c += 1;
    e->mel_pos[8][l][0] = (int16_t)r; e->mel_pos[8][l][1] = (int16_t)c;
    e->mel_hp[8][l] = CR_HP[mk]; e->mel_type[8][l] = mk;
    e->mel_cd[8][l] = 2; e->mel_alive[8][l] = 1;
  }
  int aquatic = CR_COLL[rk] == COLL_AQUATIC;
  int r = aquatic ? s->H / 2 + 4 + 1 : nr + 3;
  int c = aquatic ? s->W / 2 - 5 + 1 : nc;
  e->ran_pos[8][0][0] = (int16_t)r; e->ran_pos[8][0][1] = (int16_t)c;
  e->ran_hp[8][0] = CR_HP[rk]; e->ran_type[8][0] = rk;
  e->ran_cd[8][0] = 6; e->ran_alive[8][0] = 1;
}

/* creatures.py:489-520 (player on floor 8, so the active lanes are floor 8) */
static void boss_logic(go_state *s, int64_t i, Env *e) {
  if (!(e->pfloor == 8 && e->boss_hp > 0.0f)) return;
  int enemies = e->mel_alive[8][0] + e->mel_alive[8][1] + e->mel_alive[8][2] +
                e->ran_alive[8][0] + e->ran_alive[8][1];
  if (enemies != 0) return;
  int first = e->boss_wave == 0;
  if (first) { spawn_wave(s, e, 0); e->boss_wave = 1; }
  int was_vuln = e->boss_vuln;
  if (!first && !was_vuln && e->boss_wave > 0) {
    e->boss_vuln = 1;
    e->boss_timer = 20;
    sblock(s, i, 8, e->necro_pos[0], e->necro_pos[1], B_NECROMANCER_VULN);
  }
  if (was_vuln && e->boss_wave < 8) {
    e->boss_timer -= 1;
    if (e->boss_timer == 0) {
      spawn_wave(s, e, e->boss_wave);
      e->boss_wave += 1;
      e->boss_vuln = 0;
      sblock(s, i, 8, e->necro_pos[0], e->necro_pos[1], B_NECROMANCER);
    }
  }
}

/* creatures.py:426-452 */
static void spawn_despawn(go_state *s, int64_t i, Env *e, WS *ws) {
  int af = e->pfloor;
  for (int cls = 0; cls < 3; ++cls) {
    Lanes L = lanes_of(e, cls, af);
    for (int l = 0; l < L.cap; ++l) {
      if (!L.alive[l]) continue;
      int d = abs(L.pos[l][0] - e->prow), d2 = abs(L.pos[l][1] - e->pcol);
      if (d2 > d) d = d2;
      if (!(d <= 12 || af == 8)) L.alive[l] = 0;
    }
  }
  int night = (e->time % 300) >= 150;
  spawn_class(s, i, e, ws, 0, MEL_KIND[af], MEL_PROB[night][af], 4);
  spawn_class(s, i, e, ws, 1, RAN_KIND[af], RAN_PROB[af], 5);
  spawn_class(s, i, e, ws, 2, PAS_KIND[af], PAS_PROB[af], 6);
  if (!s->classic) boss_logic(s, i, e);
}

/* creatures.py:525-541 */
static void grow_plants(go_state *s, int64_t i, Env *e) {
  for (int l = 0; l < 10; ++l) {
    if (!e->plant_alive[l]) continue;
    e->plant_age[l] = (uint16_t)(e->plant_age[l] + 1);
    int r = e->plant_pos[l][0], c = e->plant_pos[l][1];
    uint8_t b = gblock(s, i, 0, r, c);
    int is_plant = b == B_PLANT;
    int keep = is_plant || b == B_RIPE_PLANT;
    e->plant_alive[l] = (uint8_t)keep;
    if (keep && is_plant && e->plant_age[l] >= 60) sblock(s, i, 0, r, c, B_RIPE_PLANT);
  }
}

/* engine.py:706-746, envs [lo, hi).  flags in/out: the two-pass protocol */
static void ws_begin(const Env *e, WS *ws) {
  memset(ws->unlock, 0, sizeof(ws->unlock));
  ws->hurt = 0;
  ws->health0 = e->health;
  uint32_t k32 = (uint32_t)(e->rng_key & 0xFFFFFFFFu);
  ws->base = go_vmix32(k32 ^ (e->time * 0x9E3779B9u));
}

void gs_step_pass1(go_state *s, const int64_t *actions, WS *ws, int64_t lo, int64_t hi, int *flags) {
  int mel_any = 0, ran_any = 0;
  for (int64_t i = lo; i < hi; ++i) {
    Env *e = &s->env[i];
    ws_begin(e, &ws[i]);
    player_actions(s, i, e, &ws[i], (int)actions[i]);
    advance_projectiles(s, i, e, &ws[i]);
    int af = e->pfloor;
    mel_any |= e->mel_alive[af][0] | e->mel_alive[af][1] | e->mel_alive[af][2];
    ran_any |= e->ran_alive[af][0] | e->ran_alive[af][1];
  }
  flags[0] |= mel_any;
  flags[1] |= ran_any;
}

void gs_step_pass2(go_state *s, WS *ws, int64_t lo, int64_t hi, const int *flags,
                   double *reward, uint8_t *done, uint8_t *newly, float *delta) {
  for (int64_t i = lo; i < hi; ++i) {
    Env *e = &s->env[i];
    WS *w = &ws[i];
    creatures_act(s, i, e, w, flags[0], flags[1]);
    survival_tick(s, e, w);
    spawn_despawn(s, i, e, w);
    grow_plants(s, i, e);
    e->time += 1;
    double r = 0.0;
    for (int a = 0; a < s->A; ++a) {
      int nw = w->unlock[a] && !e->ach[a];
      if (newly) newly[i * s->A + a] = (uint8_t)nw;
      if (nw) {
        e->ach[a] = 1;
        r += (double)(s->classic ? 1 : ACH_TIER_EXT[a]);
      }
    }
    float d = e->health - w->health0;
    r = r + 0.1 * (double)d;
    if (reward) reward[i] = r;
    if (delta) delta[i] = d;
    e->done = (uint8_t)(e->health <= 0.0f || (int64_t)e->time >= s->max_len);
    if (done) done[i] = e->done;
  }
}

/* state.py:198-249 for one env */
void gs_install(go_state *s, int64_t i, const go_world *w, uint64_t key) {
  Env *e = &s->env[i];
  int F = s->F, n = s->H * s->W;
  for (int f = 0; f < 9; ++f)
    for (int j = 0; j < 6; ++j) {
      e->chest_pos[f][j][0] = e->chest_pos[f][j][1] = -1;
      e->chest_loot[f][j] = e->chest_qty[f][j] = e->chest_aux[f][j] = 0;
    }
  for (int f = 0; f < F; ++f) {
    memcpy(s->blocks + ((size_t)i * F + f) * n, w->blocks[f], n);
    memcpy(s->items + ((size_t)i * F + f) * n, w->items[f], n);
    e->ladder_down[f][0] = w->ladder_down[f][0]; e->ladder_down[f][1] = w->ladder_down[f][1];
    e->ladder_up[f][0] = w->ladder_up[f][0]; e->ladder_up[f][1] = w->ladder_up[f][1];
  }
  e->spawn0[0] = w->spawn[0]; e->spawn0[1] = w->spawn[1];
  memcpy(e->potion_map, w->potion, 6);
  e->params_seed = w->seed;
  e->prow = w->spawn[0]; e->pcol = w->spawn[1];
  if (!s->classic) {
    for (int f = 0; f < F; ++f)
      for (int j = 0; j < w->n_chests[f] && j < 6; ++j) {
        e->chest_pos[f][j][0] = w->chest[f][j][0];
        e->chest_pos[f][j][1] = w->chest[f][j][1];
        e->chest_loot[f][j] = (uint8_t)w->chest[f][j][2];
        e->chest_qty[f][j] = (uint8_t)w->chest[f][j][3];
        e->chest_aux[f][j] = (uint8_t)(go_hash2(key, 800 + (uint64_t)(f * 6 + j)) % 6);
      }
    e->necro_pos[0] = (int16_t)(s->H / 2 - 6);
    e->necro_pos[1] = (int16_t)(s->W / 2);
  }
  e->facing = 3; e->dex = 1; e->str_ = 1; e->intel = 1; e->xp = 0;
  e->sword_tier = 0; e->pick_tier = 0; e->has_bow = 0; e->sword_ench = 0; e->bow_ench = 0;
  e->learned_fire = 0; e->learned_ice = 0; e->sleeping = 0; e->resting = 0;
  e->inv_wood = e->inv_stone = e->inv_coal = e->inv_iron = e->inv_diamond = 0;
  e->inv_sapphire = e->inv_ruby = e->inv_sapling = e->inv_torch = e->inv_arrow = e->inv_book = 0;
  e->time = 0; e->boss_wave = 0; e->boss_vuln = 0; e->boss_timer = 0; e->done = 0;
  memset(e->inv_potion, 0, 6); memset(e->armour, 0, 4); memset(e->armour_ench, 0, 4);
  memset(e->ach, 0, 67); memset(e->clocks, 0, sizeof(e->clocks));
  memset(e->mel_pos, 0, sizeof(e->mel_pos)); memset(e->mel_hp, 0, sizeof(e->mel_hp));
  memset(e->mel_cd, 0, sizeof(e->mel_cd)); memset(e->mel_alive, 0, sizeof(e->mel_alive));
  memset(e->mel_type, 0, sizeof(e->mel_type));
  memset(e->ran_pos, 0, sizeof(e->ran_pos)); memset(e->ran_hp, 0, sizeof(e->ran_hp));
  memset(e->ran_cd, 0, sizeof(e->ran_cd)); memset(e->ran_alive, 0, sizeof(e->ran_alive));
  memset(e->ran_type, 0, sizeof(e->ran_type));
  memset(e->pas_pos, 0, sizeof(e->pas_pos)); memset(e->pas_hp, 0, sizeof(e->pas_hp));
  memset(e->pas_alive, 0, sizeof(e->pas_alive)); memset(e->pas_type, 0, sizeof(e->pas_type));
  memset(e->pproj_pos, 0, sizeof(e->pproj_pos)); memset(e->pproj_dir, 0, 3);
  memset(e->pproj_type, 0, 3); memset(e->pproj_ttl, 0, 3); memset(e->pproj_alive, 0, 3);
  memset(e->pproj_dmg, 0, sizeof(e->pproj_dmg));
  memset(e->eproj_pos, 0, sizeof(e->eproj_pos)); memset(e->eproj_dir, 0, 3);
  memset(e->eproj_type, 0, 3); memset(e->eproj_ttl, 0, 3); memset(e->eproj_alive, 0, 3);
  memset(e->eproj_dmg, 0, sizeof(e->eproj_dmg));
  memset(e->plant_pos, 0, sizeof(e->plant_pos)); memset(e->plant_age, 0, sizeof(e->plant_age));
  memset(e->plant_alive, 0, sizeof(e->plant_alive));
  memset(e->floors_visited, 0, 9); memset(e->floor_cleared, 0, 9);
  e->pfloor = 0;
  e->health = 10.0f; e->food = 13.0f; e->drink = 13.0f; e->energy = 13.0f; e->mana = 17.0f;
  e->rng_key = key;
  e->floors_visited[0] = 1;
  e->boss_hp = s->classic ? 0.0f : 60.0f;
}
