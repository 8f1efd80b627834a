/*
 * go_obs.c -- oracle restatement of obs.encode_symbolic_batch (obs.py:191-386)
 * and tiles.render_tiles (tiles.py:85-186).  TEST INFRASTRUCTURE ONLY.
 *
 * Batch coupling reproduced: light_window adds torch glow to every env of
 * the batch iff some env of the batch stands on a dark floor
 * (obs.py:236, `(ambient < 1.0).any()`).  encode_symbolic takes that flag;
 * render_tiles runs on a one-env view, so its flag is the env's own floor.
 */
#include "go_state.h"
#include "go_tables.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

int gs_any_dark(const go_state *s) {
  if (s->classic) return 0;
  for (int64_t i = 0; i < s->n; ++i)
    if (FLOOR_AMB[s->env[i].pfloor] < 1.0f) return 1;
  return 0;
}

/* obs.py:191-195 */
static float daylight(uint32_t time) {
  float phase = (float)(time % 300) / 300.0f;
  float m = phase < 0.5f ? phase : 0.5f;
  float arg = (float)3.141592653589793 * m;
  arg = arg * 2.0f;
  float lift = go_np_sinf(arg);
  float k = (float)(1.0 - 0.15);
  return (float)0.15 + k * (lift > 0.0f ? lift : 0.0f);
}

/* obs.py:227-250: light of view tile (vr, vc) */
static void light_window(const go_state *s, const Env *e, int64_t i, int glow_on, float *light) {
  int VR = s->VR, VC = s->VC, vr2 = VR / 2, vc2 = VC / 2, af = e->pfloor;
  float base = af == 0 ? daylight(e->time) : FLOOR_AMB[af];
  for (int k = 0; k < VR * VC; ++k) light[k] = base;
  if (glow_on) {
    /* obs.py:202-213 over a (VR+6)x(VC+6) item window: the result at a view
     * tile is max(0, max over torches within Chebyshev 3 of 1 - d/4) */
    for (int r = -vr2 - 3; r <= vr2 + 3; ++r)
      for (int c = -vc2 - 3; c <= vc2 + 3; ++c) {
        int rr = e->prow + r, cc = e->pcol + c;
        if (rr < 0 || rr >= s->H || cc < 0 || cc >= s->W) continue;
        if (s->items[(((size_t)i * s->F + af) * s->H + rr) * s->W + cc] != I_TORCH) continue;
        for (int a = r - 3; a <= r + 3; ++a)
          for (int b = c - 3; b <= c + 3; ++b) {
            if (a < -vr2 || a > vr2 || b < -vc2 || b > vc2) continue;
            int d = abs(a - r) > abs(b - c) ? abs(a - r) : abs(b - c);
            float g = 1.0f;
            for (int k = 0; k < d; ++k) g = g - 0.25f;
            float *L = &light[(a + vr2) * VC + (b + vc2)];
            if (g > *L) *L = g;
          }
      }
  }
  if (e->sleeping)
    for (int k = 0; k < VR * VC; ++k) light[k] = 0.0f;
}

static const int8_t CLASSIC_LOCAL[37] = {0, 0, 1, 2, 3, 4, 0, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14,
                                         0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};

/* obs.py:253-297 */
static void creature_grid(const go_state *s, const Env *e, int *grid) {
  int VR = s->VR, VC = s->VC, af = e->pfloor;
  int r0 = e->prow - VR / 2, c0 = e->pcol - VC / 2;
  memset(grid, 0, sizeof(int) * VR * VC);
#define PAINT(pos, alive, ch)                                          \
  do {                                                                 \
    int wr = (pos)[0] - r0, wc = (pos)[1] - c0;                        \
    if ((alive) && wr >= 0 && wr < VR && wc >= 0 && wc < VC) grid[wr * VC + wc] = (ch); \
  } while (0)
  if (s->classic) {
    static const int cmap[19] = {1, 3, 2};
    for (int l = 0; l < 3; ++l) PAINT(e->mel_pos[0][l], e->mel_alive[0][l], e->mel_type[0][l] < 3 ? cmap[e->mel_type[0][l]] : 0);
    for (int l = 0; l < 2; ++l) PAINT(e->ran_pos[0][l], e->ran_alive[0][l], e->ran_type[0][l] < 3 ? cmap[e->ran_type[0][l]] : 0);
    for (int l = 0; l < 3; ++l) PAINT(e->pas_pos[0][l], e->pas_alive[0][l], e->pas_type[0][l] < 3 ? cmap[e->pas_type[0][l]] : 0);
    for (int l = 0; l < 3; ++l) PAINT(e->eproj_pos[l], e->eproj_alive[l], 4);
  } else {
    for (int l = 0; l < 3; ++l) PAINT(e->mel_pos[af][l], e->mel_alive[af][l], e->mel_type[af][l] + 1);
    for (int l = 0; l < 2; ++l) PAINT(e->ran_pos[af][l], e->ran_alive[af][l], e->ran_type[af][l] + 1);
    for (int l = 0; l < 3; ++l) PAINT(e->pas_pos[af][l], e->pas_alive[af][l], e->pas_type[af][l] + 1);
    for (int l = 0; l < 3; ++l) PAINT(e->eproj_pos[l], e->eproj_alive[l], e->eproj_type[l] + 20);
    for (int l = 0; l < 3; ++l) PAINT(e->pproj_pos[l], e->pproj_alive[l], e->pproj_type[l] + 20);
  }
#undef PAINT
}

static float sq10(uint8_t v) { return sqrtf((float)v) / 10.0f; }

/* obs.py:343-386 for env i; out has obs_length floats */
void gs_encode_symbolic(const go_state *s, int64_t i, int batch_dark, float *out) {
  const Env *e = &s->env[i];
  int VR = s->VR, VC = s->VC, T = VR * VC, af = e->pfloor;
  int bch = s->classic ? 15 : 37, ich = s->classic ? 0 : 5, cch = s->classic ? 5 : 36;
  int stride = bch + ich + cch + 1;
  int L = s->classic ? 1345 : 8268;
  float light[99];
  int cre[99];
  memset(out, 0, sizeof(float) * L);
  light_window(s, e, i, !s->classic && batch_dark, light);
  creature_grid(s, e, cre);
  for (int t = 0; t < T; ++t) {
    int r = e->prow - VR / 2 + t / VC, c = e->pcol - VC / 2 + t % VC;
    int inb = r >= 0 && r < s->H && c >= 0 && c < s->W;
    size_t mi = (((size_t)i * s->F + af) * s->H + (inb ? r : 0)) * s->W + (inb ? c : 0);
    int blk = inb ? s->blocks[mi] : B_OOB;
    int itm = inb ? s->items[mi] : 0;
    float lit = light[t] >= 0.05f ? 1.0f : 0.0f;
    float *tv = out + (size_t)t * stride;
    tv[s->classic ? CLASSIC_LOCAL[blk] : blk] = lit;
    if (ich) tv[bch + itm] = lit;
    tv[bch + ich + cre[t]] = lit;
    tv[stride - 1] = light[t];
  }
  float *v = out + (size_t)T * stride;
  float day = (float)(e->time % 300) / 300.0f;
  int k = 0;
  if (s->classic) {
    v[k++] = sq10(e->inv_wood); v[k++] = sq10(e->inv_stone); v[k++] = sq10(e->inv_coal);
    v[k++] = sq10(e->inv_iron); v[k++] = sq10(e->inv_diamond); v[k++] = sq10(e->inv_sapling);
    v[k++] = (float)e->pick_tier / 4.0f; v[k++] = (float)e->sword_tier / 4.0f;
    v[k++] = e->health / 10.0f; v[k++] = e->food / 10.0f; v[k++] = e->drink / 10.0f;
    v[k++] = e->energy / 10.0f;
    for (int d = 0; d < 4; ++d) v[k++] = e->facing == d ? 1.0f : 0.0f;
    v[k++] = day;
    v[k++] = (float)e->sleeping;
    return;
  }
  v[k++] = sq10(e->inv_wood); v[k++] = sq10(e->inv_stone); v[k++] = sq10(e->inv_coal);
  v[k++] = sq10(e->inv_iron); v[k++] = sq10(e->inv_diamond); v[k++] = sq10(e->inv_sapphire);
  v[k++] = sq10(e->inv_ruby); v[k++] = sq10(e->inv_sapling); v[k++] = sq10(e->inv_torch);
  v[k++] = sq10(e->inv_arrow);
  for (int p = 0; p < 6; ++p) v[k++] = sq10(e->inv_potion[p]);
  v[k++] = (float)e->inv_book / 2.0f;
  v[k++] = (float)e->pick_tier / 4.0f; v[k++] = (float)e->sword_tier / 4.0f;
  v[k++] = (float)e->sword_ench;
  v[k++] = (float)e->has_bow;
  for (int p = 0; p < 4; ++p) v[k++] = (float)e->armour[p] / 2.0f;
  for (int p = 0; p < 4; ++p) v[k++] = (float)e->armour_ench[p];
  v[k++] = e->health / 10.0f; v[k++] = e->food / 10.0f; v[k++] = e->drink / 10.0f;
  v[k++] = e->energy / 10.0f; v[k++] = e->mana / 10.0f; v[k++] = (float)e->xp / 10.0f;
  v[k++] = (float)e->dex / 10.0f; v[k++] = (float)e->str_ / 10.0f; v[k++] = (float)e->intel / 10.0f;
  for (int d = 0; d < 4; ++d) v[k++] = e->facing == d ? 1.0f : 0.0f;
  v[k++] = day;
  v[k++] = (float)e->sleeping; v[k++] = (float)e->resting;
  v[k++] = (float)e->learned_fire; v[k++] = (float)e->learned_ice;
  v[k++] = (float)e->pfloor / 10.0f;
  v[k++] = (float)e->floor_cleared[af];
  v[k++] = (float)e->boss_vuln;
}

/* ------------------------------------------------------------- tiles.py */

static const uint8_t PALETTE[37][3] = {
  {0,0,0},{10,10,10},{64,160,66},{48,92,190},{120,120,120},{28,100,38},{134,97,55},
  {160,140,110},{60,60,64},{188,168,152},{130,220,228},{168,120,50},{150,80,60},
  {216,200,130},{230,90,16},{96,190,90},{180,210,70},{84,78,76},{4,4,4},{86,110,76},
  {142,134,128},{60,110,230},{210,40,80},{196,150,40},{110,170,220},{190,110,40},
  {180,220,240},{100,96,90},{150,60,20},{140,190,210},{240,140,90},{150,200,255},
  {90,20,120},{130,130,140},{118,118,130},{106,106,120},{200,60,230}};

static void creature_color(int classic, int ch, uint8_t rgb[3]) {
  int kind;
  if (classic) {
    if (ch == 4) { rgb[0] = rgb[1] = rgb[2] = 250; return; }
    kind = ch == 1 ? 0 : ch == 2 ? 2 : 1;
  } else {
    if (ch >= 20) { rgb[0] = rgb[1] = rgb[2] = 250; return; }
    kind = ch - 1;
  }
  if (kind == 0) { rgb[0] = 80; rgb[1] = 200; rgb[2] = 90; return; }
  if (kind == 1) { rgb[0] = 230; rgb[1] = 230; rgb[2] = 215; return; }
  if (kind == 2) { rgb[0] = 240; rgb[1] = 190; rgb[2] = 160; return; }
  rgb[0] = (uint8_t)(40 + 11 * kind); rgb[1] = (uint8_t)(255 - 12 * kind); rgb[2] = (uint8_t)(60 + 9 * kind);
}

static void fill(uint8_t *img, int W, int y0, int y1, int x0, int x1, const uint8_t rgb[3]) {
  for (int y = y0; y < y1; ++y)
    for (int x = x0; x < x1; ++x) {
      uint8_t *p = img + ((size_t)y * W + x) * 3;
      p[0] = rgb[0]; p[1] = rgb[1]; p[2] = rgb[2];
    }
}

/* tiles.py:141-144: Python round() is half-to-even on float64 */
static void bar(uint8_t *img, int W, int y, int x, int width, int height, double frac, const uint8_t rgb[3]) {
  double f = frac < 0.0 ? 0.0 : (frac > 1.0 ? 1.0 : frac);
  int fillw = (int)nearbyint(f * (double)width);
  static const uint8_t grey[3] = {30, 30, 30};
  int a = x + fillw;
  if (a > x + width) a = x + width;
  fill(img, W, y, y + height, x, a, rgb);
  fill(img, W, y, y + height, x + fillw, x + width, grey);
}

/* tiles.py:85-133 + 147-186; out is (VR+2)*px x (VC+side)*px x 3 */
void gs_render_pixels(const go_state *s, int64_t i, int px, uint8_t *out) {
  const Env *e = &s->env[i];
  int VR = s->VR, VC = s->VC, af = e->pfloor;
  int side = s->classic ? 0 : 2;
  int FH = (VR + 2) * px, FW = (VC + side) * px;
  memset(out, 0, (size_t)FH * FW * 3);
  float light[99];
  int cre[99];
  /* render_tiles sees a one-env batch: glow iff this env's floor is dark */
  light_window(s, e, i, !s->classic && FLOOR_AMB[af] < 1.0f, light);
  creature_grid(s, e, cre);
  int inset = px / 4 > 1 ? px / 4 : 1;
  static const uint8_t ITEMC[5][3] = {{255,255,255},{255,220,90},{20,20,25},{235,235,240},{70,30,30}};
  for (int t = 0; t < VR * VC; ++t) {
    int tr = t / VC, tc = t % VC;
    int r = e->prow - VR / 2 + tr, c = e->pcol - VC / 2 + tc;
    int inb = r >= 0 && r < s->H && c >= 0 && c < s->W;
    size_t mi = (((size_t)i * s->F + af) * s->H + (inb ? r : 0)) * s->W + (inb ? c : 0);
    int blk = inb ? s->blocks[mi] : B_OOB;
    int itm = inb ? s->items[mi] : 0;
    float sh = light[t] < 0.0f ? 0.0f : (light[t] > 1.0f ? 1.0f : light[t]);
    int dark = light[t] < 0.05f;
    uint8_t rgb[3];
    for (int k = 0; k < 3; ++k) rgb[k] = dark ? 0 : (uint8_t)(int)((float)PALETTE[blk][k] * sh);
    int y = tr * px, x = tc * px;
    fill(out, FW, y, y + px, x, x + px, rgb);
    if (dark) continue;
    if (itm) fill(out, FW, y + inset, y + px - inset, x + inset, x + px - inset, ITEMC[itm]);
    if (cre[t]) {
      uint8_t cc[3];
      creature_color(s->classic, cre[t], cc);
      fill(out, FW, y + inset, y + px - inset, x + inset, x + px - inset, cc);
    }
  }
  static const uint8_t PLAYER[3] = {250, 60, 60};
  {
    int y = (VR / 2) * px, x = (VC / 2) * px;
    fill(out, FW, y + inset, y + px - inset, x + inset, x + px - inset, PLAYER);
  }
  /* status strip (tiles.py:147-166) */
  static const uint8_t BARC[5][3] = {{220,60,60},{220,160,60},{70,130,230},{240,230,90},{150,90,220}};
  double hmax = (double)(9.0f + (float)(double)e->str_);
  double fmax = (double)(12.0f + (float)(double)e->dex);
  double stats[5];
  int ns = 4;
  stats[0] = (double)e->health / hmax; stats[1] = (double)e->food / fmax;
  stats[2] = (double)e->drink / fmax; stats[3] = (double)e->energy / fmax;
  if (!s->classic) { stats[4] = (double)e->mana / (double)(16.0f + (float)(double)e->intel); ns = 5; }
  int bar_h = (2 * px) / (ns + 1);
  if (bar_h < 2) bar_h = 2;
  int y0 = VR * px, width = VC * px;
  for (int k = 0; k < ns; ++k) bar(out, FW, y0 + 1 + k * bar_h, 1, width - 2, bar_h - 1, stats[k], BARC[k]);
  if (side) {
    /* tiles.py:169-186 */
    static const uint8_t GC[7][3] = {{200,200,210},{160,160,170},{120,140,200},{240,220,90},
                                     {90,220,140},{220,90,90},{140,120,240}};
    double g[7] = {(double)e->sword_tier / 4.0, (double)e->pick_tier / 4.0,
                   (double)(e->armour[0] + e->armour[1] + e->armour[2] + e->armour[3]) / 8.0,
                   (double)e->xp / 8.0, (double)e->dex / 5.0, (double)e->str_ / 5.0,
                   (double)e->intel / 5.0};
    int x0 = VC * px;
    for (int k = 0; k < 7; ++k) {
      int y = k * px;
      if (y + px > FH) break;
      bar(out, FW, y + 1, x0 + 1, 2 * px - 2, px - 2, g[k], GC[k]);
    }
  }
}
