// rt_math.cuh — lean FP64 elementary functions for the tree walk.
//
// The arguments the method produces have known domains — log of a uniform in
// (0,1), sinpi/cospi of 2v with v in (0,1), sqrt of a non-negative product,
// 1/d with d >= 1, exp of a non-positive number — so the special-case
// branches of general libm routines are unnecessary.  Accuracy target: a few
// ulp (<= ~4e-16 relative, or ~1e-18 absolute near zero), far inside the
// 1e-12 per-tree parity bound; checked against 64-bit-mantissa long double
// references on the host (tests/test_math.py) and on the device.
//
// Polynomial coefficients live in the constant bank (RTM_CONST) so DFMA reads
// them directly; the 2 KB log table is staged in shared memory by the kernel
// (its index is lane-divergent).  Functions are __host__ __device__ so the
// identical code is accuracy-tested on the CPU, where MUFU approximations are
// emulated in FP32.
#pragma once
#include <cstdint>
#include <cstring>
#include <cmath>

#include "rt_math_tables.h"

#if defined(__CUDACC__)
#define RTM_HD __host__ __device__ __forceinline__
#else
#define RTM_HD inline
#endif

namespace rtk {

RTM_HD uint64_t dbits(double x) {
#if defined(__CUDA_ARCH__)
  return static_cast<uint64_t>(__double_as_longlong(x));
#else
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
#endif
}

RTM_HD double dfrom(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(u));
#else
  double x;
  std::memcpy(&x, &u, 8);
  return x;
#endif
}

// MUFU.RCP64H / MUFU.RSQ64H seeds (~2^-22 relative); FP32 emulation on host.
RTM_HD double rcp_seed(double x) {
#if defined(__CUDA_ARCH__)
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
#else
  return static_cast<double>(1.0f / static_cast<float>(x));
#endif
}

RTM_HD double rsqrt_seed(double x) {
#if defined(__CUDA_ARCH__)
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
#else
  return static_cast<double>(1.0f / std::sqrt(static_cast<float>(x)));
#endif
}

RTM_HD double rint_d(double x) {
#if defined(__CUDA_ARCH__)
  return rint(x);
#else
  return std::nearbyint(x);
#endif
}

RTM_HD double fma_d(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return fma(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}

// log(x) for positive normal x.  x = 2^k z, z ∈ [0.6875, 1.375); table entry
// i (top 7 bits of bits(x) - bits(0.6875)) gives invc ≈ 1/c_i and
// logc = -log(invc); r = z·invc − 1 (one rounding, |r| <= 2^-7);
// log x = k ln2 + logc + r + r²·P(r).  11 FP64 ops + 1 I2F.
RTM_HD double log_tab(double x, const LogEntry* T) {
  // (all on the high word: bits(0.6875) has a zero low word, so the 64-bit
  // difference never borrows and z keeps x's low word)
  const uint64_t ix = dbits(x);
  const uint32_t hi = static_cast<uint32_t>(ix >> 32);
  const uint32_t tmp = hi - static_cast<uint32_t>(kLogOff >> 32);
  const int i = static_cast<int>((tmp >> 13) & 127u);
  const int k = static_cast<int32_t>(tmp) >> 20;
  const double z = dfrom((static_cast<uint64_t>(hi - (tmp & 0xfff00000u)) << 32) | (ix & 0xffffffffull));
  const LogEntry e = T[i];
  const double r = fma_d(z, e.invc, -1.0);
  double p = kLogPTop;
  p = fma_d(p, r, kLogPL[4]);
  p = fma_d(p, r, kLogPL[3]);
  p = fma_d(p, r, kLogPL[2]);
  p = fma_d(p, r, kLogPL[1]);
  p = fma_d(p, r, kLogPL[0]);
  const double r2 = r * r;
  const double t = fma_d(static_cast<double>(k), kLogPL[5], e.logc);   // kLogPL[5] = ln2
  return t + fma_d(r2, p, r);
}

// sin(pi f), cos(pi f) for |f| <= 1/4 (near-minimax in f², fit errors < 3e-18).
RTM_HD void sincospi_core(double f, double& s, double& c) {
  const double f2 = f * f;
  double ps = kSinPiTop;
  ps = fma_d(ps, f2, kSinPi[5]);
  ps = fma_d(ps, f2, kSinPi[4]);
  ps = fma_d(ps, f2, kSinPi[3]);
  ps = fma_d(ps, f2, kSinPi[2]);
  ps = fma_d(ps, f2, kSinPi[1]);
  ps = fma_d(ps, f2, kSinPi[0]);
  double pc = kCosPiTop;
  pc = fma_d(pc, f2, kCosPi[6]);
  pc = fma_d(pc, f2, kCosPi[5]);
  pc = fma_d(pc, f2, kCosPi[4]);
  pc = fma_d(pc, f2, kCosPi[3]);
  pc = fma_d(pc, f2, kCosPi[2]);
  pc = fma_d(pc, f2, kCosPi[1]);
  s = ps * f;
  c = fma_d(pc, f2, kCosPi[0]);
}

// sin(pi a), cos(pi a) for a ∈ [0, 2] on the 2^-52 grid (a = 2v, v = unif53):
// q = rint(2a), f = a − q/2 exactly (|f| <= 1/4), rotate by q quarter turns.
RTM_HD void sincospi2(double a, double& s_out, double& c_out) {
  const double q = rint_d(2.0 * a);
  const double f = fma_d(q, -0.5, a);
  double s, c;
  sincospi_core(f, s, c);
  const int qi = static_cast<int>(q) & 3;
  const bool swap = qi & 1;
  double so = swap ? c : s;
  double co = swap ? s : c;
  const uint64_t sneg = (qi & 2) ? 0x8000000000000000ull : 0ull;
  const uint64_t cneg = ((qi + 1) & 2) ? 0x8000000000000000ull : 0ull;
  s_out = dfrom(dbits(so) ^ sneg);
  c_out = dfrom(dbits(co) ^ cneg);
}

// cos(pi a) only, a ∈ [0, 2] on the 2^-52 grid: n = rint(a), f = a − n
// exactly (|f| <= 1/2), cos(pi a) = (−1)^n cos(pi f) with one even polynomial
// (no quadrant swap, half the work of sincospi2; absolute error < 1e-16).
RTM_HD double cospi2(double a) {
  const double n = rint_d(a);
  const double f = a - n;
  const double f2 = f * f;
  double p = kCosPiWTop;
  p = fma_d(p, f2, kCosPiW[7]);
  p = fma_d(p, f2, kCosPiW[6]);
  p = fma_d(p, f2, kCosPiW[5]);
  p = fma_d(p, f2, kCosPiW[4]);
  p = fma_d(p, f2, kCosPiW[3]);
  p = fma_d(p, f2, kCosPiW[2]);
  p = fma_d(p, f2, kCosPiW[1]);
  p = fma_d(p, f2, kCosPiW[0]);
  const uint64_t neg = (static_cast<uint64_t>(static_cast<int>(n)) & 1ull) << 63;
  return dfrom(dbits(p) ^ neg);
}

// The angles of the d = 3 Box–Muller draws, 2π·v with v = (2w+1)·2^-33 the
// 32-bit uniform of word w, reduced on the integer instead of in FP64 —
// bitwise the same q and f as sincospi2(2v) / cospi2(2v):
//   sincospi2: 2·(2v) = (w + 1/2)·2^-30, q = rint = ((w >> 29) + 1) >> 1,
//              f = 2v − q/2 = ((2w+1) − q·2^31)·2^-32, |f| <= 1/4;
//   cospi2:    2v = (w + 1/2)·2^-31, n = rint = ((w >> 30) + 1) >> 1,
//              f = 2v − n = ((2w+1) − n·2^32)·2^-32, |f| < 1/2;
// the differences d are odd and fit an int32, so they are the wrapped uint32
// differences reinterpreted.  The polynomials are evaluated in d itself with
// the coefficients pre-scaled by exact powers of two (k_n 2^(-64n), sin also
// 2^-32): Horner in d·d = 2^64 f·f then gives the same bits as in f·f.
RTM_HD void sincos2pi_u32(uint32_t w, double& s_out, double& c_out) {
  const uint32_t q = ((w >> 29) + 1u) >> 1;
  const double d = static_cast<double>(static_cast<int32_t>(2u * w + 1u - (q << 31)));
  const double D = d * d;
  double ps = kSinPi32Top;
  ps = fma_d(ps, D, kSinPi32[5]);
  ps = fma_d(ps, D, kSinPi32[4]);
  ps = fma_d(ps, D, kSinPi32[3]);
  ps = fma_d(ps, D, kSinPi32[2]);
  ps = fma_d(ps, D, kSinPi32[1]);
  ps = fma_d(ps, D, kSinPi32[0]);
  double pc = kCosPi32Top;
  pc = fma_d(pc, D, kCosPi32[6]);
  pc = fma_d(pc, D, kCosPi32[5]);
  pc = fma_d(pc, D, kCosPi32[4]);
  pc = fma_d(pc, D, kCosPi32[3]);
  pc = fma_d(pc, D, kCosPi32[2]);
  pc = fma_d(pc, D, kCosPi32[1]);
  const double s = ps * d;
  const double c = fma_d(pc, D, kCosPi32[0]);
  const int qi = static_cast<int>(q) & 3;
  const bool swap = qi & 1;
  double so = swap ? c : s;
  double co = swap ? s : c;
  const uint64_t sneg = (qi & 2) ? 0x8000000000000000ull : 0ull;
  const uint64_t cneg = ((qi + 1) & 2) ? 0x8000000000000000ull : 0ull;
  s_out = dfrom(dbits(so) ^ sneg);
  c_out = dfrom(dbits(co) ^ cneg);
}

RTM_HD double cos2pi_u32(uint32_t w) {
  const double d = static_cast<double>(static_cast<int32_t>(2u * w + 1u));
  const double D = d * d;
  double p = kCosPiW32Top;
  p = fma_d(p, D, kCosPiW32[7]);
  p = fma_d(p, D, kCosPiW32[6]);
  p = fma_d(p, D, kCosPiW32[5]);
  p = fma_d(p, D, kCosPiW32[4]);
  p = fma_d(p, D, kCosPiW32[3]);
  p = fma_d(p, D, kCosPiW32[2]);
  p = fma_d(p, D, kCosPiW32[1]);
  p = fma_d(p, D, kCosPiW32[0]);
  const uint64_t neg = static_cast<uint64_t>(((w >> 30) + 1u) & 2u) << 62;   // n odd
  return dfrom(dbits(p) ^ neg);
}

// sqrt(a), a >= 0: rsqrt seed, one Newton step (2^-44), one Heron correction.
RTM_HD double sqrt_nr(double a) {
  double y = rsqrt_seed(a);
  const double h = 0.5 * a;
  const double t = h * y;
  y = fma_d(y, fma_d(-t, y, 0.5), y);
  double s = a * y;
  const double r = fma_d(-s, s, a);
  s = fma_d(r, 0.5 * y, s);
  return a > 0.0 ? s : 0.0;
}

// sqrt(a) for a positive normal a (the Box–Muller radii: −2 ln v > 0 and
// h > 0 always): sqrt_nr without the a = 0 select.
RTM_HD double sqrt_pos(double a) {
  double y = rsqrt_seed(a);
  const double h = 0.5 * a;
  const double t = h * y;
  y = fma_d(y, fma_d(-t, y, 0.5), y);
  double s = a * y;
  const double r = fma_d(-s, s, a);
  return fma_d(r, 0.5 * y, s);
}

// 1/d for normal d > 0: rcp seed and one cubic correction y(1 + e + e²).
RTM_HD double rcp_nr(double d) {
  const double y = rcp_seed(d);
  const double e = fma_d(-d, y, 1.0);
  return fma_d(y, fma_d(e, e, e), y);
}

// exp(x) for x <= 0 (0 below -1075·ln2): x = k ln2 + r, |r| <= ln2/2, Taylor
// degree 13, scaled by 2^k in two exact steps (subnormal results allowed).
RTM_HD double exp_neg(double x) {
  const double xc = x < -745.5 ? -745.5 : x;
  const double kf = rint_d(xc * kLog2e);
  double r = fma_d(kf, -kExpLn2Hi, xc);
  r = fma_d(kf, -kExpLn2Lo, r);
  double p = kExp[13];
  p = fma_d(p, r, kExp[12]);
  p = fma_d(p, r, kExp[11]);
  p = fma_d(p, r, kExp[10]);
  p = fma_d(p, r, kExp[9]);
  p = fma_d(p, r, kExp[8]);
  p = fma_d(p, r, kExp[7]);
  p = fma_d(p, r, kExp[6]);
  p = fma_d(p, r, kExp[5]);
  p = fma_d(p, r, kExp[4]);
  p = fma_d(p, r, kExp[3]);
  p = fma_d(p, r, kExp[2]);
  p = fma_d(p, r, kExp[1]);
  p = fma_d(p, r, kExp[0]);
  const int k = static_cast<int>(kf);
  const int k1 = k / 2, k2 = k - k1;
  const double s1 = dfrom(static_cast<uint64_t>(1023 + k1) << 52);
  const double s2 = dfrom(static_cast<uint64_t>(1023 + k2) << 52);
  return x < -745.5 ? 0.0 : (p * s1) * s2;
}

// exp(x) for x <= 0 (0 below -745.5) with a 32-entry table T = kExpT32
// (staged in shared memory by the kernel: its index is lane-divergent):
// x = (32m + j) ln2/32 + r, |r| <= ln2/64, e^x = 2^m T_j (1 + (e^r − 1)),
// e^r − 1 by Taylor degree 6 — 13 FP64 operations against exp_neg's 19.
RTM_HD double exp_neg_tab(double x, const double* T) {
  const double xc = x < -745.5 ? -745.5 : x;
  const double kf = rint_d(xc * kExp32Inv);
  double r = fma_d(kf, -kExp32Hi, xc);
  r = fma_d(kf, -kExp32Lo, r);
  double q = kExpQ[5];
  q = fma_d(q, r, kExpQ[4]);
  q = fma_d(q, r, kExpQ[3]);
  q = fma_d(q, r, kExpQ[2]);
  q = fma_d(q, r, kExpQ[1]);
  q = fma_d(q, r, kExpQ[0]);
  const int k = static_cast<int>(kf);
  const double t = T[k & 31];
  const double p = fma_d(t, q * r, t);
  const int m = (k - (k & 31)) / 32;   // floor(k / 32), exact
  const int m1 = m / 2, m2 = m - m1;
  const double s1 = dfrom(static_cast<uint64_t>(1023 + m1) << 52);
  const double s2 = dfrom(static_cast<uint64_t>(1023 + m2) << 52);
  return x < -745.5 ? 0.0 : (p * s1) * s2;
}

// a · e^x for finite a and any x (the record-ring trees' C = Π e^X, DESIGN.md
// §4): the table-driven e^x = 2^m T_j (1 + (e^r − 1)) of exp_neg_tab with the
// power 2^m applied to the PRODUCT last, in two exact halves — neither e^x
// nor a needs to be representable on its own, only the result (x clamped to
// ±1400, where 2^m's halves are still normal).  Same rounding as a ·
// exp_neg_tab(x) wherever e^x is normal.
RTM_HD double mul_exp_tab(double a, double x, const double* T) {
  const double xc = x < -1400.0 ? -1400.0 : (x > 1400.0 ? 1400.0 : x);
  const double kf = rint_d(xc * kExp32Inv);
  double r = fma_d(kf, -kExp32Hi, xc);
  r = fma_d(kf, -kExp32Lo, r);
  double q = kExpQ[5];
  q = fma_d(q, r, kExpQ[4]);
  q = fma_d(q, r, kExpQ[3]);
  q = fma_d(q, r, kExpQ[2]);
  q = fma_d(q, r, kExpQ[1]);
  q = fma_d(q, r, kExpQ[0]);
  const int k = static_cast<int>(kf);
  const double t = T[k & 31];
  const double p = fma_d(t, q * r, t);
  const int m = (k - (k & 31)) / 32;   // floor(k / 32), exact; |m| <= 2020
  const int m1 = m / 2, m2 = m - m1;   // |m1|, |m2| <= 1010: 2^m1, 2^m2 normal
  const double s1 = dfrom(static_cast<uint64_t>(1023 + m1) << 52);
  const double s2 = dfrom(static_cast<uint64_t>(1023 + m2) << 52);
  return ((a * p) * s1) * s2;
}

}  // namespace rtk
