// The world generator (gr_world.cu) compiled a second time with 256-thread
// CTAs for the extended tier, in namespace gr::wide: small batches (a few
// worlds per step) finish a floor sooner with more threads per floor.
#define GR_WG_WIDE 1
#define GR_WG_EXT_THREADS 256
#include "gr_world.cu"
