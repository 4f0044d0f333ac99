// pade.cuh — row a8: batched [L/M] Padé approximants at z = 1 (PAPER.md:295-301,
// 744-780), one warp per node, the system in registers (no local memory).
//
// Q(0) = 1, deg P <= L, deg Q <= M, Q·Σc_n z^n − P = O(z^{L+M+1}): the
// denominator solves the Toeplitz system Σ_{j=1..M} q_j c_{L+i−j} = −c_{L+i}
// (i = 1..M, c_{<0} = 0) by Gaussian elimination with partial pivoting (first
// maximal |pivot| on ties), p_a = Σ_{j<=min(a,M)} q_j c_{a−j}, u = P(1)/Q(1).
// Lane r holds row r of the augmented matrix in registers; the pivot search
// is two warp max-reductions on the bit pattern of |a| (non-negative doubles
// order as their bit patterns) plus a ballot; pivot rows are broadcast by
// shuffles.  The order M is a template parameter (one instantiation per M,
// loops fully unrolled for exactly that M): a launch fetches only the code of
// the M it uses.  (A first version unrolled every loop to M = 16 — 5,000
// instructions per node, instruction-fetch bound at ~18 us per 1024 nodes.)  The products and differences are rounded separately (no FMA
// contraction), in the order the plain definition states them.
//
// Flags (R12):
//   bit0  exact zero pivot in [L/M]: the value is then the largest regular
//         [L/M'], M' < M ([L/0], the partial sum c_0+…+c_L, always is) —
//         SPEC.md:403's fallback — and M' is stored in bits 8..15;
//   bit1  |Q(1)| <= 1e-14 |P(1)|;
//   bit2  Q changes sign on (0, 1] (256 equispaced points);
//   bit3  |u − Σ_{n<=K} c_n| > 10 se_sum (only when se_sum is given): the
//         resummed value and the partial sum disagree beyond the statistics
//         (divergence or an artificial pole).
#pragma once
#include <cstdint>

namespace rtk {

constexpr int kPadeMaxM = 16;
constexpr int kPadeThreads = 128;   // 4 nodes per CTA

__device__ __forceinline__ double pade_shfl(double v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

// c_idx for a per-lane index (0 outside [0, K]); every lane must call it
__device__ __forceinline__ double pade_coef(double cl, int idx, int K) {
  const double v = pade_shfl(cl, idx & 31);
  return (idx >= 0 && idx <= K) ? v : 0.0;
}

// The [L/MM] denominator with MM a compile-time constant (every loop fully
// unrolled, the rows in registers; only the instantiation a launch uses is
// fetched).  Lane r < MM owns row r.  Returns false on an exact zero pivot;
// else q[0..MM] (all lanes).
template <int MM>
__device__ __forceinline__ bool pade_denominator(double cl, int K, int L, int lane, double* q) {
  double A[MM];
#pragma unroll
  for (int j = 0; j < MM; ++j) A[j] = pade_coef(cl, L + lane - j, K);
  double rhs = -pade_coef(cl, L + lane + 1, K);
#pragma unroll
  for (int col = 0; col < MM; ++col) {
    const bool in = lane >= col && lane < MM;
    const unsigned long long bits =
        static_cast<unsigned long long>(__double_as_longlong(in ? fabs(A[col]) : 0.0));
    const unsigned hi = static_cast<unsigned>(bits >> 32), lo = static_cast<unsigned>(bits);
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
    if ((mhi | mlo) == 0u) return false;       // exact zero pivot (warp-uniform)
    const int piv = __ffs(__ballot_sync(0xffffffffu, in && hi == mhi && lo == mlo)) - 1;
    if (piv != col) {                          // warp-uniform: swap rows col and piv
      const int src = lane == col ? piv : (lane == piv ? col : lane);
#pragma unroll
      for (int j = col; j < MM; ++j) A[j] = pade_shfl(A[j], src);
      rhs = pade_shfl(rhs, src);
    }
    const bool upd = lane > col && lane < MM;
    const double f = A[col] / pade_shfl(A[col], col);
#pragma unroll
    for (int j = col; j < MM; ++j) {
      const double pj = pade_shfl(A[j], col);
      if (upd) A[j] = __dsub_rn(A[j], __dmul_rn(f, pj));
    }
    const double pr = pade_shfl(rhs, col);
    if (upd) rhs = __dsub_rn(rhs, __dmul_rn(f, pr));
  }
  // back substitution: q_{r+1} = (rhs_r − Σ_{k>r} A[r][k] q_{k+1}) / A[r][r]
  q[0] = 1.0;
#pragma unroll
  for (int r = MM - 1; r >= 0; --r) {
    double s = rhs;
#pragma unroll
    for (int k = r + 1; k < MM; ++k) s = __dsub_rn(s, __dmul_rn(A[k], q[k + 1]));
    q[r + 1] = pade_shfl(s / A[r], r);
  }
  return true;
}

template <int MM>
__device__ __forceinline__ void pade_tail(double cl, int K, int L, int M, int lane, const double* q,
                                          double se, bool want_se, double* out_u, uint32_t* out_fl) {
  // numerator coefficients, lane a: p_a = Σ_{j <= min(a, MM)} q_j c_{a−j}
  double pa = 0.0;
#pragma unroll
  for (int j = 0; j <= MM; ++j) {
    const double v = pade_coef(cl, lane - j, K);
    if (j <= lane) pa = __dadd_rn(pa, __dmul_rn(q[j], v));
  }
  // P(1), the partial sum: ascending order, as the definition sums (L <= K)
  double P1 = 0.0, us = 0.0, Q1 = 0.0;
  for (int a = 0; a <= K; ++a) {
    const double v = pade_shfl(pa, a), w = pade_shfl(cl, a);
    if (a <= L) P1 += v;
    us += w;
  }
#pragma unroll
  for (int j = 0; j <= MM; ++j) Q1 += q[j];
  const double u = P1 / Q1;
  uint32_t fl = MM < M ? (1u | (static_cast<uint32_t>(MM) << 8)) : 0u;
  if (fabs(Q1) <= 1e-14 * fabs(P1)) fl |= 2u;
  // sign change of Q on (0, 1]: lane takes z = (lane + 1 + 32 m)/256
  bool neg = false;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const double z = static_cast<double>(lane + 1 + 32 * m) * (1.0 / 256.0);
    double Qz = 0.0, zp = 1.0;
#pragma unroll
    for (int j = 0; j <= MM; ++j) {
      Qz = __dadd_rn(Qz, __dmul_rn(q[j], zp));
      zp = __dmul_rn(zp, z);
    }
    neg = neg || !(Qz > 0.0);
  }
  if (__any_sync(0xffffffffu, neg)) fl |= 4u;
  if (want_se && fabs(u - us) > 10.0 * se) fl |= 8u;
  *out_u = u;
  *out_fl = fl;
}

template <int MM>
__device__ __forceinline__ bool pade_try(double cl, int K, int L, int M, int lane, double se,
                                         bool want_se, double* u, uint32_t* fl) {
  double q[MM + 1];
  if (MM > 0 && !pade_denominator<MM>(cl, K, L, lane, q)) return false;
  q[0] = 1.0;
  pade_tail<MM>(cl, K, L, M, lane, q, se, want_se, u, fl);
  return true;
}

template <>
__device__ __forceinline__ bool pade_denominator<0>(double, int, int, int, double* q) {
  q[0] = 1.0;
  return true;
}

__global__ void __launch_bounds__(kPadeThreads)
pade_warp_kernel(const double* __restrict__ coeffs, int64_t n, int K, int L, int M,
                 const double* __restrict__ se_sum, double* __restrict__ out_u,
                 uint32_t* __restrict__ flags) {
  const int64_t node = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (node >= n) return;                      // warp-uniform
  const double cl = lane <= K ? coeffs[node * (K + 1) + lane] : 0.0;   // K <= 30
  const double se = se_sum != nullptr ? se_sum[node] : 0.0;
  const bool want = se_sum != nullptr;
  double u = 0.0;
  uint32_t fl = 0;
  // degenerate table: lower M until the system is regular (bit0)
  for (int Mu = M; Mu >= 0; --Mu) {
    bool ok = false;
    switch (Mu) {
#define RT_PADE_CASE(m) case m: ok = pade_try<m>(cl, K, L, M, lane, se, want, &u, &fl); break;
      RT_PADE_CASE(0) RT_PADE_CASE(1) RT_PADE_CASE(2) RT_PADE_CASE(3) RT_PADE_CASE(4)
      RT_PADE_CASE(5) RT_PADE_CASE(6) RT_PADE_CASE(7) RT_PADE_CASE(8) RT_PADE_CASE(9)
      RT_PADE_CASE(10) RT_PADE_CASE(11) RT_PADE_CASE(12) RT_PADE_CASE(13) RT_PADE_CASE(14)
      RT_PADE_CASE(15) RT_PADE_CASE(16)
#undef RT_PADE_CASE
      default: break;
    }
    if (ok) break;
  }
  if (lane == 0) {
    out_u[node] = u;
    if (flags) flags[node] = fl;
  }
}

}  // namespace rtk
