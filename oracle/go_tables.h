/*
 * go_tables.h -- rule tables restated from constants.py (TEST INFRASTRUCTURE).
 * constants.py:17-567; tiles.py:26-82 (palette).
 */
#ifndef GO_TABLES_H
#define GO_TABLES_H
#include <stdint.h>

/* Block (constants.py:17-54) */
enum {
  B_INVALID, B_OOB, B_GRASS, B_WATER, B_STONE, B_TREE, B_WOOD, B_PATH, B_COAL,
  B_IRON, B_DIAMOND, B_TABLE, B_FURNACE, B_SAND, B_LAVA, B_PLANT, B_RIPE_PLANT,
  B_WALL, B_DARKNESS, B_WALL_MOSS, B_STALAGMITE, B_SAPPHIRE, B_RUBY, B_CHEST,
  B_FOUNTAIN, B_FIRE_GRASS, B_ICE_GRASS, B_GRAVEL, B_FIRE_TREE, B_ICE_SHRUB,
  B_ENCHANT_TABLE_FIRE, B_ENCHANT_TABLE_ICE, B_NECROMANCER, B_GRAVE, B_GRAVE2,
  B_GRAVE3, B_NECROMANCER_VULN, N_BLOCKS_T
};
/* Item (constants.py:60-66) */
enum { I_EMPTY, I_TORCH, I_LADDER_DOWN, I_LADDER_UP, I_LADDER_DOWN_BLOCKED };
/* ChestLoot (constants.py:364-370) */
enum { LOOT_NOTHING, LOOT_BOW, LOOT_BOOK, LOOT_POTION, LOOT_ARROWS, LOOT_TORCHES };
/* Collision */
enum { COLL_GROUND, COLL_FLYING, COLL_AMPHIBIAN, COLL_AQUATIC };

/* constants.py:422-430: GRASS PATH SAND FIRE_GRASS ICE_GRASS GRAVEL */
static const uint8_t WALKABLE_T[37] = {
  0,0,1,0,0,0,0,1,0,0, 0,0,0,1,0,0,0,0,0,0, 0,0,0,0,0,1,1,1,0,0, 0,0,0,0,0,0,0};

/* creature tables (constants.py:73-156, creatures.py:36-69) */
static const float CR_HP[19] = {5, 3, 3, 7, 5, 6, 9, 6, 4, 11, 8, 12, 12, 20, 6, 20, 14, 24, 16};
static const float CR_DMG[19][3] = {
  {2,0,0},{2,0,0},{0,0,0},{3,0,0},{3,0,0},{0,0,0},{4,0,0},{2,0,0},{0,0,0},{5,0,0},
  {4,0,0},{6,0,0},{4,0,0},{6,1,1},{4,3,3},{3,5,0},{3,5,0},{4,0,5},{4,0,4}};
static const float CR_DEF[19][3] = {
  {0,0,0},{0,0,0},{0,0,0},{0,0,0},{0,0,0},{0,0,0},{0,0,0},{0,0,0},{0,0,0},{0,0,0},
  {0,0,0},{50,0,0},{50,0,0},{20,0,0},{0,0,0},{90,100,0},{90,100,0},{90,0,100},{90,0,100}};
static const uint8_t CR_COLL[19] = {0,0,0,0,0,0,0,0,1,2,0,0,0,0,3,0,1,0,0};
static const int8_t MEL_KIND[9] = {0, 3, 6, 9, 11, 13, 15, 17, -1};
static const int8_t RAN_KIND[9] = {1, 4, 7, 10, 12, 14, 16, 18, -1};
static const int8_t PAS_KIND[9] = {2, 5, 8, 5, 5, 8, 8, -1, -1};
static const uint8_t RANGED_PROJ[19] = {0,3,0,0,4,0,0,3,0,0,5,0,3,0,6,0,7,0,8};
static const uint8_t DEFEAT_ACH[19] = {8,12,2,38,39,51,36,37,50,40,41,65,66,42,43,44,45,46,47};
static const float EAT_FOOD_T[19] = {0,0,6,0,0,4,0,0,2,0,0,0,0,0,0,0,0,0,0};
static const float DEALT_BARE[19] = {2,2,0,3,3,0,4,2,0,5,4,6,4,8,10,8,8,9,8};
static const uint8_t ACH_TIER_EXT[67] = {
  1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,3,3,3,3,3,5,5,5,8,8,8,3,3,3,3,
  5,5,5,5,8,8,8,8,8,8,3,3,3,3,3,5,5,5,5,3,3,3,3,5,5,5,5};
/* COLLISION_WALKABLE[coll][block] (constants.py:432-444) */
static const uint8_t COLL_WALK[4][37] = {
  {0,0,1,0,0,0,0,1,0,0,0,0,0,1,0,0,0,0,0,0,0,0,0,0,0,1,1,1,0,0,0,0,0,0,0,0,0},
  {0,0,1,1,0,0,0,1,0,0,0,0,0,1,1,0,0,0,0,0,1,0,0,0,0,1,1,1,0,0,0,0,0,0,0,0,0},
  {0,0,1,1,0,0,0,1,0,0,0,0,0,1,0,0,0,0,0,0,0,0,0,0,0,1,1,1,0,0,0,0,0,0,0,0,0},
  {0,0,0,1,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0,0}};
static const uint8_t BLOCKS_PROJ[37] = {
  1,1,0,0,1,1,1,0,1,1,1,1,1,0,0,0,0,1,1,1,1,1,1,1,1,0,0,0,1,1,1,1,1,1,1,1,1};
static const uint8_t PLACE_STONE_OK[37] = {
  0,0,1,1,0,0,0,1,0,0,0,0,0,1,1,0,0,0,0,0,0,0,0,0,0,1,1,1,0,0,0,0,0,0,0,0,0};
static const uint8_t PLACE_SOLID_OK[37] = {
  0,0,1,0,0,0,0,1,0,0,0,0,0,1,0,0,0,0,0,0,0,0,0,0,0,1,1,1,0,0,0,0,0,0,0,0,0};
static const int16_t DIR_OFF[4][2] = {{0, -1}, {0, 1}, {-1, 0}, {1, 0}};
static const float SWORD_BASE[5] = {1, 2, 3, 5, 8};
static const float FLOOR_AMB[9] = {1, 1, 0, 1, 1, 0, 1, 0, 0};
/* spawn probabilities (creatures.py:61-69), float64 */
static const double MEL_PROB[2][9] = {{0.008,0.05,0.05,0.05,0.05,0.05,0.05,0.05,0},
                                      {0.05,0.05,0.05,0.05,0.05,0.05,0.05,0.05,0}};
static const double RAN_PROB[9] = {0.02,0.02,0.02,0.02,0.02,0.02,0.02,0.02,0};
static const double PAS_PROB[9] = {0.1,0.1,0.1,0.1,0.1,0.1,0.1,0.1,0};
/* ENTER_FLOOR_ACHIEVEMENT (constants.py:329-338) */
static const uint8_t ENTER_ACH[9] = {255, 29, 28, 30, 31, 32, 33, 34, 35};

#endif
