// gr_glibc_sincos.h -- glibc's float64 sin / cos, bit for bit (hazard H3).
//
// The reference's cave noise calls numpy's float64 cos / sin (perlin.py:71-72
// with the float64 dtype of worldgen.py:424), which is glibc's libm.  Its
// results are not always correctly rounded (off by an ulp on ~1.5e-4 of the
// float32 angles in [0, 2*pi)), so reproducing the reference bit for bit
// means reproducing glibc's algorithm: sysdeps/ieee754/dbl-64/s_sin.c
// (glibc >= 2.28; this image ships 2.39) as x86-64 runs it.  On hosts with
// FMA + AVX2 the ifunc picks the __sin_fma / __cos_fma build, where GCC
// contracted a*b+c into fused multiply-adds; every fma below is one that
// build executes (read off its disassembly), every other operation is a
// separately rounded IEEE op.  Compiled as CUDA (-fmad=false, fma() = DFMA)
// or as C (-ffp-contract=off, fma() from libm), so the host build can be
// checked against the system libm exhaustively (tests/test_host_cpu.py).
//
// Domain: |x| < 105414350 (the reduce_sincos range); the caves only use
// float32 angles in [0, 2*pi).
#pragma once
#include <stdint.h>
#include <math.h>
#ifndef __CUDACC__
#include <string.h>
#endif

#if defined(__CUDACC__)
#define GL_FN __host__ __device__ __forceinline__
#define GL_TAB __constant__
#else
#define GL_FN static inline
#define GL_TAB static const
#endif

// __sincostab: {sn, ssn, cs, ccs} for k/128, k = 0..109
GL_TAB uint64_t GL_SINCOSTAB[440] = {
#include "gr_glibc_sincostab.inc"
};

GL_FN double gl_bits(uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)b);
#else
  double d;
  memcpy(&d, &b, 8);
  return d;
#endif
}
GL_FN uint64_t gl_word(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t b;
  memcpy(&b, &d, 8);
  return b;
#endif
}
GL_FN double gl_tab(int i) {
#if defined(__CUDA_ARCH__)
  return gl_bits(GL_SINCOSTAB[i]);
#else
  return gl_bits(GL_SINCOSTAB[i]);
#endif
}

// usncs.h / s_sin.c constants (values as stored in libm)
#define GL_SN3 (-0x1.5555555555515p-3)
#define GL_SN5 (0x1.11110e829872fp-7)
#define GL_CS2 (0x1p-1)
#define GL_CS4 (-0x1.5555555555535p-5)
#define GL_CS6 (0x1.6c16bedd9e239p-10)
#define GL_S1 (-0x1.5555555555555p-3)
#define GL_S2 (0x1.1111111110ecep-7)
#define GL_S3 (-0x1.a01a019db08b8p-13)
#define GL_S4 (0x1.71de27b9a7ed9p-19)
#define GL_S5 (-0x1.addffc2fcdf59p-26)
#define GL_BIG (0x1.8p45)
#define GL_TOINT (0x1.8p52)
#define GL_HPINV (0x1.45f306dc9c883p-1)
#define GL_MP1 (0x1.921fb58p0)
#define GL_MP2 (-0x1.dde973cp-27)
#define GL_PP3 (-0x1.cb3b398p-55)
#define GL_PP4 (-0x1.d747f23e32ed7p-83)
#define GL_HP0 (0x1.921fb54442d18p0)
#define GL_HP1 (0x1.1a62633145c07p-54)

// TAYLOR_SIN(xx, a, da): a + ((POLY(xx)*a - 0.5*da)*xx + da)
GL_FN double gl_taylor_sin(double xx, double a, double da) {
  double p = fma(fma(fma(fma(GL_S5, xx, GL_S4), xx, GL_S3), xx, GL_S2), xx, GL_S1);
  double t = fma(p, a, -(0.5 * da));
  return a + fma(xx, t, da);
}

// do_sin(x, dx)
GL_FN double gl_do_sin(double x, double dx) {
  const double xold = x;
  if (fabs(x) < 0.126) return gl_taylor_sin(x * x, x, dx);
  if (x <= 0) dx = -dx;
  const double ax = fabs(x);
  const double u = GL_BIG + ax;
  const double xr = ax - (u - GL_BIG);
  const int k = (int)((uint32_t)gl_word(u) << 2);
  const double xx = xr * xr;
  const double s = xr + fma(xr * xx, fma(xx, GL_SN5, GL_SN3), dx);
  const double c = fma(xr, dx, xx * fma(xx, fma(xx, GL_CS6, GL_CS4), GL_CS2));
  const double sn = gl_tab(k), ssn = gl_tab(k + 1), cs = gl_tab(k + 2), ccs = gl_tab(k + 3);
  const double cor = fma(s, cs, fma(-c, sn, fma(s, ccs, ssn)));
  return copysign(sn + cor, xold);
}

// do_cos(x, dx)
GL_FN double gl_do_cos(double x, double dx) {
  if (x < 0) dx = -dx;
  const double ax = fabs(x);
  const double u = GL_BIG + ax;
  const double xr = (ax - (u - GL_BIG)) + dx;
  const int k = (int)((uint32_t)gl_word(u) << 2);
  const double xx = xr * xr;
  const double s = fma(xr * xx, fma(xx, GL_SN5, GL_SN3), xr);
  const double c = xx * fma(xx, fma(xx, GL_CS6, GL_CS4), GL_CS2);
  const double sn = gl_tab(k), ssn = gl_tab(k + 1), cs = gl_tab(k + 2), ccs = gl_tab(k + 3);
  const double cor = fma(-s, sn, fma(-c, cs, fma(-s, ssn, ccs)));
  return cs + cor;
}

// reduce_sincos: x = n*pi/2 + (a + da), 136-bit accurate
GL_FN int gl_reduce(double x, double* a, double* da) {
  const double t = fma(x, GL_HPINV, GL_TOINT);
  const double xn = t - GL_TOINT;
  const int n = (int)((uint32_t)gl_word(t) & 3u);
  const double y = fma(-xn, GL_MP2, fma(-xn, GL_MP1, x));
  const double t2 = fma(-xn, GL_PP3, y);
  double db = fma(-xn, GL_PP3, y - t2);
  const double b = fma(-xn, GL_PP4, t2);
  db = db + fma(-xn, GL_PP4, t2 - b);
  *a = b;
  *da = db;
  return n;
}

GL_FN double gl_do_sincos(double a, double da, int n) {
  const double r = (n & 1) ? gl_do_cos(a, da) : gl_do_sin(a, da);
  return (n & 2) ? -r : r;
}

GL_FN uint32_t gl_hi_abs(double x) { return (uint32_t)(gl_word(x) >> 32) & 0x7fffffffu; }

// __sin
GL_FN double gl_sin(double x) {
  const uint32_t k = gl_hi_abs(x);
  if (k < 0x3e500000u) return x;
  if (k < 0x3feb6000u) return gl_do_sin(x, 0.0);
  if (k < 0x400368fdu) return copysign(gl_do_cos(GL_HP0 - fabs(x), GL_HP1), x);
  double a, da;
  const int n = gl_reduce(x, &a, &da);
  return gl_do_sincos(a, da, n);
}

// __cos
GL_FN double gl_cos(double x) {
  const uint32_t k = gl_hi_abs(x);
  if (k < 0x3e400000u) return 1.0;
  if (k < 0x3feb6000u) return gl_do_cos(x, 0.0);
  if (k < 0x400368fdu) {
    const double y = GL_HP0 - fabs(x);
    const double a = y + GL_HP1;
    const double da = (y - a) + GL_HP1;
    return gl_do_sin(a, da);
  }
  double a, da;
  const int n = gl_reduce(x, &a, &da);
  return gl_do_sincos(a, da, n + 1);
}
