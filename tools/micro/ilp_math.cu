// Microbenchmark (experiment, not product): the tree walk's per-particle math
// (2 Philox blocks, R29 one-log Gamma split, d = 3 Box–Muller, Lorentzian g)
// for NP independent particles per thread per iteration, the next label of
// each chain derived from its outputs (a serial chain like the walk's).
// Question: does NP = 2 (constants shared between two chains, half the
// occupancy) beat NP = 1 per particle?
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2402_06491_b200/csrc/philox.cuh"
#include "../../paper_2402_06491_b200/csrc/rt_math.cuh"
using namespace rtk;

struct MP { RoundKeys rk; double inv_lambda, two_d, inv_scale2, amp; int iters; };

template <int NP, int MINB>
__global__ void __launch_bounds__(128, MINB) kmath(const __grid_constant__ MP P, double* out) {
  __shared__ LogEntry ltab[128];
  for (int q = threadIdx.x; q < 128; q += blockDim.x) ltab[q] = kLogTable[q];
  __syncthreads();
  uint32_t lab[NP];
  double y[NP][3], tau[NP], acc[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    lab[p] = blockIdx.x * blockDim.x + threadIdx.x + p * 7919u;
    y[p][0] = y[p][1] = y[p][2] = 0.1 * p; tau[p] = 1.0; acc[p] = 0.0;
  }
  for (int it = 0; it < P.iters; ++it) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const uint4 r0 = philox4x32_10(it, 7u, lab[p], 0u, P.rk);
      const uint4 r1 = philox4x32_10(it, 7u, lab[p], 1u << 24, P.rk);
      const double u12 = unif32(r0.x) * unif32(r0.y);
      const double v1 = unif32(min(r1.y, r1.z)), v2 = unif32(max(r1.y, r1.z));
      const double G = -log_tab(u12 * unif32(r1.x), ltab);
      const double e0 = G * v1, e1 = G * (v2 - v1), e2 = G * (1.0 - v2);
      const double S = e0 * P.inv_lambda;
      const bool leaf = S > tau[p];
      const double h2d = (leaf ? tau[p] : S) * P.two_d;
      const double rad = sqrt_pos(fma(2.0 * e1, h2d, 1e-300));
      double sn, cs;
      sincos2pi_u32(r0.w, sn, cs);
      y[p][0] = fma(rad, cs, y[p][0]);
      y[p][1] = fma(rad, sn, y[p][1]);
      y[p][2] = fma(sqrt_pos(2.0 * e2 * h2d), cos2pi_u32(r1.w), y[p][2]);
      double r2 = y[p][0] * y[p][0];
      r2 = fma(y[p][1], y[p][1], r2);
      r2 = fma(y[p][2], y[p][2], r2);
      const double g = P.amp * rcp_nr(fma(r2, P.inv_scale2, 1.0));
      acc[p] += g;
      tau[p] = leaf ? 1.0 : tau[p] - S;
      lab[p] = (leaf ? lab[p] * 3u : lab[p] * 5u) ^ r0.z;
    }
  }
  double s = 0.0;
#pragma unroll
  for (int p = 0; p < NP; ++p) s += acc[p] + y[p][0];
  if (s == 1.2345) out[0] = s;
}

template <int NP, int MINB>
double run(MP P, double* d) {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kmath<NP, MINB>, 128, 0);
  const int grid = nsm * per;
  kmath<NP, MINB><<<grid, 128>>>(P, d);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kmath<NP, MINB><<<grid, 128>>>(P, d);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double parts = double(grid) * 128 * P.iters * NP;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kmath<NP, MINB>);
  printf("NP=%d MINB=%d: %d regs, %d CTAs/SM, %.3f ms, %.3e particles/s\n", NP, MINB, fa.numRegs, per, ms,
         parts / (ms * 1e-3));
  return parts / (ms * 1e-3);
}

int main() {
  MP P; P.rk = make_round_keys(12345); P.inv_lambda = 1.0; P.two_d = 2.0; P.inv_scale2 = 1.0; P.amp = 0.5;
  P.iters = 2000;
  double* d; cudaMalloc(&d, 8);
  run<1, 8>(P, d); run<1, 12>(P, d); run<2, 4>(P, d); run<2, 6>(P, d); run<2, 8>(P, d); run<4, 2>(P, d); run<4, 4>(P, d);
  return 0;
}
