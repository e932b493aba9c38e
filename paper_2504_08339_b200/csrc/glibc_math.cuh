// glibc_math.cuh -- bit-exact restatement of glibc 2.39's __log_fma and
// __cos_fma (x86_64 ifunc variants selected on FMA+AVX2 hosts) for the
// inputs RngStream::normal feeds them (rng.hpp:111-116):
//   log(u1), u1 = 1 - k*2^-53 in (0, 1]   (normal doubles, never special)
//   cos(x),  x  = fl(2*pi * k*2^-53) in [0, 2*pi)
// and the normal deviate itself, evaluated with the reference's rounding
// (no FMA contraction in the reference build, CMakeLists.txt:4-9).
//
// The operation sequence -- including exactly which multiply-adds the
// glibc FMA build fused -- was read off `objdump -d` of this image's
// libm.so.6 (H1); the constants and tables are copied from the
// same file at build time by gen_libm_tables.py.  Every arithmetic step is
// an explicitly rounded intrinsic, so nvcc cannot re-associate or contract.
// Used on the device by the mutation kernel and on the host by the
// validation test that compares it with the live libm.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

#include "libm_tables.inc"

namespace fnb {
namespace glibc {

#ifdef __CUDA_ARCH__
#define GM_FMA(a, b, c) __fma_rn((a), (b), (c))
#define GM_ADD(a, b) __dadd_rn((a), (b))
#define GM_SUB(a, b) __dsub_rn((a), (b))
#define GM_MUL(a, b) __dmul_rn((a), (b))
#define GM_SQRT(a) __dsqrt_rn(a)
// polynomial coefficients (constant indices): constant-bank operands of the DFMAs
__constant__ static const double kLogA[5] = FNB_LIBM_LOG_A;
__constant__ static const double kLogB[11] = FNB_LIBM_LOG_B;
// lookup tables (data-dependent indices): read-only global loads
__device__ static const double kLogTab[256] = FNB_LIBM_LOG_TAB;
__device__ static const double kSinCos[FNB_LIBM_SINCOSTAB_N] = FNB_LIBM_SINCOSTAB;
// the tables (6 KB) stay L1-resident next to the genome rows the mutation
// kernels stream through L1 (evict_last: evicted after normal-priority lines)
__device__ __forceinline__ double ld_table(const double* a) {
  double v;
  asm("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(a));
  return v;
}
#define GM_TAB(t, i) ld_table(&(t)[i])
#define GM_CT(t, i) ((t)[i])
#else
#define GM_FMA(a, b, c) std::fma((a), (b), (c))
#define GM_ADD(a, b) ((a) + (b))
#define GM_SUB(a, b) ((a) - (b))
#define GM_MUL(a, b) ((a) * (b))
#define GM_SQRT(a) std::sqrt(a)
static const double kLogA[5] = FNB_LIBM_LOG_A;
static const double kLogB[11] = FNB_LIBM_LOG_B;
static const double kLogTab[256] = FNB_LIBM_LOG_TAB;
static const double kSinCos[FNB_LIBM_SINCOSTAB_N] = FNB_LIBM_SINCOSTAB;
#define GM_TAB(t, i) ((t)[i])
#define GM_CT(t, i) ((t)[i])
#endif

__host__ __device__ __forceinline__ uint64_t bits(double x) {
#ifdef __CUDA_ARCH__
  return uint64_t(__double_as_longlong(x));
#else
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
#endif
}
__host__ __device__ __forceinline__ double from_bits(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double x;
  std::memcpy(&x, &u, 8);
  return x;
#endif
}

// __log_fma (optimized-routines log, LOG_TABLE_BITS = 7) for x in (0, 1]
__host__ __device__ inline double log(double x) {
  const uint64_t ix = bits(x);
  if (ix - 0x3fee000000000000ull < 0x3090000000000ull) {  // |x - 1| small: polynomial path
    if (ix == 0x3ff0000000000000ull) return 0.0;
    const double r = GM_SUB(x, FNB_LIBM_ONE);
    double p = GM_FMA(r, GM_CT(kLogB, 2), GM_CT(kLogB, 1));
    double q = GM_FMA(r, GM_CT(kLogB, 5), GM_CT(kLogB, 4));
    double s = GM_FMA(r, GM_CT(kLogB, 8), GM_CT(kLogB, 7));
    const double r2 = GM_MUL(r, r);
    p = GM_FMA(r2, GM_CT(kLogB, 3), p);
    q = GM_FMA(r2, GM_CT(kLogB, 6), q);
    const double r3 = GM_MUL(r, r2);
    s = GM_FMA(r2, GM_CT(kLogB, 9), s);
    s = GM_FMA(r3, GM_CT(kLogB, 10), s);
    q = GM_FMA(s, r3, q);
    p = GM_FMA(q, r3, p);
    const double t = GM_FMA(r, FNB_LIBM_TWO27, r);     // r + r*2^27
    const double rhi = GM_FMA(-FNB_LIBM_TWO27, r, t);  // (r + w) - w
    const double b0 = GM_CT(kLogB, 0);
    const double rhi2 = GM_MUL(rhi, rhi);
    const double rlo = GM_SUB(r, rhi);
    const double hi = GM_FMA(rhi2, b0, r);
    const double d = GM_SUB(r, hi);
    const double sum = GM_ADD(r, rhi);
    double lo = GM_FMA(rhi2, b0, d);
    lo = GM_FMA(GM_MUL(b0, rlo), sum, lo);
    const double y = GM_FMA(p, r3, lo);
    return GM_ADD(hi, y);
  }
  const uint64_t tmp = ix - 0x3fe6000000000000ull;
  const int i = int((tmp >> 45) & 127u);
  const int k = int(int64_t(tmp) >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
  const double invc = GM_TAB(kLogTab, 2 * i), logc = GM_TAB(kLogTab, 2 * i + 1);
  const double z = from_bits(iz);
  const double kd = double(k);
  const double w = GM_FMA(kd, FNB_LIBM_LN2HI, logc);
  const double r = GM_FMA(z, invc, FNB_LIBM_MINUS_ONE);
  const double p1 = GM_FMA(r, GM_CT(kLogA, 2), GM_CT(kLogA, 1));
  const double hi = GM_ADD(r, w);
  const double r2 = GM_MUL(r, r);
  double t = GM_SUB(w, hi);
  t = GM_ADD(t, r);
  double lo = GM_FMA(kd, FNB_LIBM_LN2LO, t);
  const double r3 = GM_MUL(r, r2);
  const double p2 = GM_FMA(r, GM_CT(kLogA, 4), GM_CT(kLogA, 3));
  lo = GM_FMA(r2, GM_CT(kLogA, 0), lo);
  const double q = GM_FMA(p2, r2, p1);
  const double y = GM_FMA(r3, q, lo);
  return GM_ADD(y, hi);
}

// do_cos(x, dx) of s_sin.c (FMA build), dx already sign-adjusted
__host__ __device__ __forceinline__ double do_cos_fma(double ax, double dxs) {
  const double u = GM_ADD(ax, FNB_LIBM_BIG);
  const double t = GM_SUB(u, FNB_LIBM_BIG);
  double xr = GM_SUB(ax, t);
  xr = GM_ADD(xr, dxs);
  const int idx = int(uint32_t(bits(u)) << 2);
  const double xx = GM_MUL(xr, xr);
  const double p = GM_FMA(xx, FNB_LIBM_SN5, FNB_LIBM_SN3);
  const double s = GM_FMA(GM_MUL(xr, xx), p, xr);
  double c6 = GM_FMA(xx, FNB_LIBM_CS6, FNB_LIBM_CS4);
  c6 = GM_FMA(xx, c6, FNB_LIBM_CS2);
  const double c = GM_MUL(xx, c6);
  const double sn = GM_TAB(kSinCos, idx), ssn = GM_TAB(kSinCos, idx + 1);
  const double cs = GM_TAB(kSinCos, idx + 2), ccs = GM_TAB(kSinCos, idx + 3);
  const double a1 = GM_FMA(-s, ssn, ccs);
  const double a2 = GM_FMA(-c, cs, a1);
  const double cor = GM_FMA(-s, sn, a2);
  return GM_ADD(cs, cor);
}

// do_sin(x, dx) of s_sin.c for |x| >= 0.126 (FMA build); dx sign-adjusted
__host__ __device__ __forceinline__ double do_sin_fma(double x, double dxs) {
  const double ax = fabs(x);
  const double u = GM_ADD(ax, FNB_LIBM_BIG);
  const double t = GM_SUB(u, FNB_LIBM_BIG);
  const double xr = GM_SUB(ax, t);
  const int idx = int(uint32_t(bits(u)) << 2);
  const double xx = GM_MUL(xr, xr);
  const double p = GM_FMA(xx, FNB_LIBM_SN5, FNB_LIBM_SN3);
  const double q = GM_FMA(GM_MUL(xr, xx), p, dxs);
  double c6 = GM_FMA(xx, FNB_LIBM_CS6, FNB_LIBM_CS4);
  c6 = GM_FMA(xx, c6, FNB_LIBM_CS2);
  const double s = GM_ADD(xr, q);
  const double cc = GM_MUL(xx, c6);
  const double c = GM_FMA(xr, dxs, cc);
  const double sn = GM_TAB(kSinCos, idx), ssn = GM_TAB(kSinCos, idx + 1);
  const double cs = GM_TAB(kSinCos, idx + 2), ccs = GM_TAB(kSinCos, idx + 3);
  const double a1 = GM_FMA(s, ccs, ssn);
  const double a2 = GM_FMA(-c, sn, a1);
  const double cor = GM_FMA(s, cs, a2);
  return copysign(GM_ADD(sn, cor), x);
}

// TAYLOR_SIN(x*x, x, dx) of s_sin.c (FMA build)
__host__ __device__ __forceinline__ double taylor_sin_fma(double a, double da) {
  const double xx = GM_MUL(a, a);
  double p = GM_FMA(xx, FNB_LIBM_S5, FNB_LIBM_S4);
  p = GM_FMA(xx, p, FNB_LIBM_S3);
  p = GM_FMA(xx, p, FNB_LIBM_S2);
  p = GM_FMA(xx, p, FNB_LIBM_S1);
  const double hd = GM_MUL(da, FNB_LIBM_CS2);  // 0.5 * da
  p = GM_FMA(p, a, -hd);
  const double t = GM_FMA(xx, p, da);
  return GM_ADD(a, t);
}

// __cos_fma for finite 0 <= x < 105414350 (the RngStream domain is [0, 2*pi)).
// Every argument range only prepares (a, da, kernel, sign) -- the same
// rounded operations as s_sin.c's branches -- and the three kernels each have
// one call site, so a warp whose lanes fall in different ranges runs at most
// do_cos + do_sin (+ the rare Taylor case) instead of one kernel copy per range.
__host__ __device__ inline double cos(double x) {
  const uint32_t k = uint32_t(bits(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;
  double a, da;
  int kern;  // 0 do_cos(a, da), 1 do_sin(a, da), 2 taylor_sin(a, da)
  bool neg = false;
  if (k < 0x3feb6000u) {
    a = fabs(x);
    da = x < 0.0 ? -0.0 : 0.0;
    kern = 0;
  } else if (k < 0x400368fdu) {
    const double y = GM_SUB(FNB_LIBM_HP0, fabs(x));
    a = GM_ADD(y, FNB_LIBM_HP1);
    da = GM_ADD(GM_SUB(y, a), FNB_LIBM_HP1);
    if (fabs(a) < FNB_LIBM_SMALL) {
      kern = 2;
    } else {
      kern = 1;
      if (a <= 0.0) da = -da;
    }
  } else {  // reduce_sincos
    const double t = GM_FMA(x, FNB_LIBM_HPINV, FNB_LIBM_TOINT);
    const double xn = GM_SUB(t, FNB_LIBM_TOINT);
    const int n = int(uint32_t(bits(t)) & 3u);
    double y = GM_FMA(-xn, FNB_LIBM_MP1, x);
    y = GM_FMA(-xn, FNB_LIBM_MP2, y);
    const double t2 = GM_FMA(-xn, FNB_LIBM_PP3, y);
    double db = GM_SUB(y, t2);
    db = GM_FMA(-xn, FNB_LIBM_PP3, db);
    const double b = GM_FMA(-xn, FNB_LIBM_PP4, t2);
    double e = GM_SUB(t2, b);
    e = GM_FMA(-xn, FNB_LIBM_PP4, e);
    db = GM_ADD(db, e);
    if ((n & 1) == 0) {  // do_sincos(b, db, n + 1) -> do_cos
      a = fabs(b);
      da = b < 0.0 ? -db : db;
      kern = 0;
    } else if (fabs(b) < FNB_LIBM_SMALL) {
      a = b;
      da = db;
      kern = 2;
    } else {
      a = b;
      da = b <= 0.0 ? -db : db;
      kern = 1;
    }
    neg = ((n + 1) & 2) != 0;
  }
  double res;
  if (kern == 0) res = do_cos_fma(a, da);
  else if (kern == 1) res = do_sin_fma(a, da);
  else res = taylor_sin_fma(a, da);
  return neg ? -res : res;
}

// RngStream::normal from its two uniforms (rng.hpp:111-116): u1 = 1 - U0,
// u2 = U1, mean + (sd * sqrt(-2 log u1)) * cos(2 pi u2), each op rounded.
__host__ __device__ inline double normal_from_uniforms(double uni0, double uni1, double mean, double sd) {
  const double u1 = GM_SUB(1.0, uni0);
  const double r = GM_SQRT(GM_MUL(-2.0, log(u1)));
  const double c = cos(GM_MUL(6.283185307179586476925286766559, uni1));
  return GM_ADD(mean, GM_MUL(GM_MUL(sd, r), c));
}

}  // namespace glibc
}  // namespace fnb
