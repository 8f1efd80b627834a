// dev probe: host write bandwidth into a 2.17 GB array with T threads
// (regular stores, non-temporal stores), as the dense e2e decode would need.
#define _POSIX_C_SOURCE 199309L
#include <time.h>
#include <immintrin.h>
#include <omp.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <stdint.h>
static double now() { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec + 1e-9 * t.tv_nsec; }
int main() {
  size_t n = (size_t)65536 * 8268;   // floats
  float* a = aligned_alloc(64, n * 4);
  memset(a, 1, n * 4);
  int T = omp_get_max_threads();
  for (int rep = 0; rep < 3; ++rep) {
    double t0 = now();
#pragma omp parallel for schedule(static)
    for (long r = 0; r < 65536; ++r) memset(a + r * 8268, 0, 8268 * 4);
    double t1 = now();
#pragma omp parallel for schedule(static)
    for (long r = 0; r < 65536; ++r) {
      float* row = a + r * 8268;
      __m512 z = _mm512_setzero_ps();
      long k = 0;
      long head = ((64 - ((uintptr_t)row & 63)) & 63) / 4;
      for (; k < head; ++k) row[k] = 0.f;
      for (; k + 16 <= 8268; k += 16) _mm512_stream_ps(row + k, z);
      for (; k < 8268; ++k) row[k] = 0.f;
    }
    _mm_sfence();
    double t2 = now();
    printf("threads %d: memset %.1f GB/s, stream %.1f GB/s\n", T, n * 4 / (t1 - t0) / 1e9, n * 4 / (t2 - t1) / 1e9);
  }
  return 0;
}
