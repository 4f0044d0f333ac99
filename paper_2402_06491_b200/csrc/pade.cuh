// pade.cuh — row a8: batched [L/M] Padé approximants at z = 1 (PAPER.md:295-301,
// 744-780), one warp per node, everything in registers (no local memory).
//
// Q(0) = 1, deg P <= L, deg Q <= M, Q·Σc_n z^n − P = O(z^{L+M+1}): the
// denominator solves the Toeplitz system Σ_{j=1..M} q_j c_{L+i−j} = −c_{L+i}
// (i = 1..M, c_{<0} = 0) by Gaussian elimination with partial pivoting (first
// maximal |pivot| on ties), p_a = Σ_{j<=min(a,M)} q_j c_{a−j}, u = P(1)/Q(1).
// Lane r holds row r of the augmented matrix in registers; the pivot search
// is two warp max-reductions on the bit pattern of |a| (non-negative doubles
// order as their bit patterns) plus a ballot; pivot rows are broadcast by
// shuffles.  The products and differences are rounded separately (no FMA
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

__global__ void __launch_bounds__(kPadeThreads)
pade_warp_kernel(const double* __restrict__ coeffs, int64_t n, int K, int L, int M,
                 const double* __restrict__ se_sum, double* __restrict__ out_u,
                 uint32_t* __restrict__ flags) {
  const int64_t node = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (node >= n) return;                      // warp-uniform
  const double* c = coeffs + node * (K + 1);
  const double cl = lane <= K ? c[lane] : 0.0;   // K <= 30: one coefficient per lane
  // c_idx for a per-lane index (0 outside [0, K]); every lane must call it
  auto coef = [&](int idx) -> double {
    const double v = pade_shfl(cl, idx & 31);
    return (idx >= 0 && idx <= K) ? v : 0.0;
  };

  double q[kPadeMaxM + 1];
  q[0] = 1.0;
#pragma unroll
  for (int j = 1; j <= kPadeMaxM; ++j) q[j] = 0.0;
  int Mu = M;
  for (; Mu > 0; --Mu) {                      // degenerate table: lower M (bit0)
    double A[kPadeMaxM];
#pragma unroll
    for (int j = 0; j < kPadeMaxM; ++j) {
      const double v = coef(L + lane - j);
      A[j] = (j < Mu) ? v : 0.0;
    }
    double rhs = -coef(L + lane + 1);
    bool singular = false;
#pragma unroll
    for (int col = 0; col < kPadeMaxM; ++col) {
      if (col >= Mu) break;                   // warp-uniform
      const bool in = lane >= col && lane < Mu;
      const unsigned long long bits =
          static_cast<unsigned long long>(__double_as_longlong(in ? fabs(A[col]) : 0.0));
      const unsigned hi = static_cast<unsigned>(bits >> 32), lo = static_cast<unsigned>(bits);
      const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
      const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
      if ((mhi | mlo) == 0u) { singular = true; break; }   // exact zero pivot
      const unsigned cand = __ballot_sync(0xffffffffu, in && hi == mhi && lo == mlo);
      const int piv = __ffs(cand) - 1;
      if (piv != col) {                       // warp-uniform: swap rows col and piv
        const int src = lane == col ? piv : (lane == piv ? col : lane);
#pragma unroll
        for (int j = 0; j < kPadeMaxM; ++j)
          if (j >= col) A[j] = pade_shfl(A[j], src);
        rhs = pade_shfl(rhs, src);
      }
      const bool upd = lane > col && lane < Mu;
      const double f = A[col] / pade_shfl(A[col], col);
#pragma unroll
      for (int j = 0; j < kPadeMaxM; ++j) {
        if (j < col) continue;
        const double pj = pade_shfl(A[j], col);
        if (upd) A[j] = __dsub_rn(A[j], __dmul_rn(f, pj));
      }
      const double pr = pade_shfl(rhs, col);
      if (upd) rhs = __dsub_rn(rhs, __dmul_rn(f, pr));
    }
    if (singular) continue;
    // back substitution: q_{r+1} = (rhs_r − Σ_{k>r} A[r][k] q_{k+1}) / A[r][r]
#pragma unroll
    for (int r = kPadeMaxM - 1; r >= 0; --r) {
      if (r >= Mu) continue;                  // warp-uniform
      double s = rhs;
#pragma unroll
      for (int k = r + 1; k < kPadeMaxM; ++k)
        if (k < Mu) s = __dsub_rn(s, __dmul_rn(A[k], q[k + 1]));
      q[r + 1] = pade_shfl(s / A[r], r);
    }
    break;
  }
  // numerator coefficients, lane a: p_a = Σ_{j <= min(a, M')} q_j c_{a−j}
  double pa = 0.0;
  const int jm = min(lane, Mu);
#pragma unroll
  for (int j = 0; j <= kPadeMaxM; ++j) {
    const double v = coef(lane - j);
    if (j <= jm) pa = __dadd_rn(pa, __dmul_rn(q[j], v));
  }
  // P(1), Q(1), the partial sum: ascending order, as the definition sums
  double P1 = 0.0, us = 0.0, Q1 = 0.0;
  for (int a = 0; a < 32; ++a) {
    const double v = pade_shfl(pa, a), w = pade_shfl(cl, a);
    if (a <= L) P1 += v;
    if (a <= K) us += w;
  }
#pragma unroll
  for (int j = 0; j <= kPadeMaxM; ++j)
    if (j <= Mu) Q1 += q[j];
  const double u = P1 / Q1;
  uint32_t fl = Mu < M ? (1u | (static_cast<uint32_t>(Mu) << 8)) : 0u;
  if (fabs(Q1) <= 1e-14 * fabs(P1)) fl |= 2u;
  // sign change of Q on (0, 1]: lane takes z = (lane + 1 + 32 m)/256
  bool neg = false;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const double z = static_cast<double>(lane + 1 + 32 * m) / 256.0;
    double Qz = 0.0, zp = 1.0;
#pragma unroll
    for (int j = 0; j <= kPadeMaxM; ++j) {
      if (j <= Mu) {
        Qz = __dadd_rn(Qz, __dmul_rn(q[j], zp));
        zp = __dmul_rn(zp, z);
      }
    }
    neg = neg || !(Qz > 0.0);
  }
  if (__any_sync(0xffffffffu, neg)) fl |= 4u;
  if (se_sum != nullptr && fabs(u - us) > 10.0 * se_sum[node]) fl |= 8u;
  if (lane == 0) {
    out_u[node] = u;
    if (flags) flags[node] = fl;
  }
}

}  // namespace rtk
