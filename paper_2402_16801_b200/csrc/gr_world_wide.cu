// The world generator (gr_world.cu) compiled a second time with 512-thread
// CTAs for the extended tier, in namespace gr::wide: small batches (a few
// worlds per step) finish a floor sooner with more threads per floor.
#define GR_WG_WIDE 1
#ifndef GR_WG_WIDE_THREADS
#define GR_WG_WIDE_THREADS 512
#endif
#define GR_WG_EXT_THREADS GR_WG_WIDE_THREADS
#include "gr_world.cu"
