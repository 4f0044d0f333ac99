// shared_eval.cuh — shared trees (NEXT row f4), phase 2.
//
// Phase 1 (tree_walk_kernel<…, SH = true>) walked every tree ONCE for all
// nodes and stored its summary (order bin, weight product W, leaf count) and
// its leaf displacements δ_l from the root.  Here a CTA of 64 threads takes
// 128 nodes (two per thread) and a block of consecutive trees; every thread
// runs the same trees in index order, so control flow is identical across
// the warp and the tree data are warp-uniform loads (L1/L2 broadcasts):
//   C_i = W · Π_l g(x_i + δ_l)  (leaves at x_i + δ),
// accumulated into the node's order bin (ΣC, ΣC²; counts are node-free).
// The loop is the g evaluations themselves — FP64-pipe bound.  Results per
// (node, tree block) go to the per-node task partials that the shared task
// reduction sums in block order (deterministic).
#pragma once
#include <cstdint>

#include "tree_walk.cuh"

namespace rtk {

constexpr int kEvalThreads = 64;

struct EvalParams {
  const TreeSum* tsum;
  const double* leaves;      // [M][lmax][DIM]
  int32_t lmax;
  int64_t M;                 // trees in this chunk
  int32_t tpb;               // trees per block (blockIdx.y)
  const double* points;      // [n_points][DIM]
  int32_t n_points;
  int32_t K, nb;
  double amp, inv_scale, inv_scale2;
  double* partials;          // [n_points][tpn_total][nb][3]
  int64_t tpn_total, q0;     // per-node task count, first block index of this chunk
  TreeRec* recs;             // REC: [n_points][n_rec]
  int64_t n_rec;
  int32_t rec_shift;
  uint32_t rel0;             // REC: tree index of this chunk relative to the call's first tree
};

// Each thread owns kNpt nodes (tree data loaded once serve them all; 1 for
// small node counts so no thread idles); leaves are loaded four at a time and
// the next tree's summary is prefetched, so the global-load latency is
// overlapped with the g evaluations.
template <int DIM, int GK, bool REC, int kNpt>
__global__ void __launch_bounds__(kEvalThreads)
shared_eval_kernel(const __grid_constant__ EvalParams E) {
  extern __shared__ double acc[];                 // [nb][2][kNpt][kEvalThreads]
  __shared__ int cnt[32];
  const int tid = threadIdx.x;
  int node[kNpt];
  bool valid[kNpt];
  double x[kNpt][DIM];
#pragma unroll
  for (int a = 0; a < kNpt; ++a) {
    node[a] = (blockIdx.x * kNpt + a) * kEvalThreads + tid;
    valid[a] = node[a] < E.n_points;
#pragma unroll
    for (int k = 0; k < DIM; ++k) x[a][k] = valid[a] ? E.points[static_cast<int64_t>(node[a]) * DIM + k] : 0.0;
  }
  constexpr int AS = kNpt * kEvalThreads;         // acc stride per (bin, moment)
  if constexpr (!REC) {
    for (int q = tid; q < E.nb * 2 * AS; q += kEvalThreads) acc[q] = 0.0;
    if (tid < 32) cnt[tid] = 0;
    __syncthreads();
  }
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * E.tpb;
  const int64_t j1 = min(E.M, j0 + E.tpb);
  TreeSum nxt = E.tsum[j0];                       // warp-uniform, prefetched
  for (int64_t j = j0; j < j1; ++j) {
    const TreeSum ts = nxt;
    if (j + 1 < j1) nxt = E.tsum[j + 1];
    if constexpr (REC) {
      const uint32_t rel = E.rel0 + static_cast<uint32_t>(j);
      if ((rel & ((1u << E.rec_shift) - 1u)) != 0u) continue;
    }
    double prod[kNpt];
#pragma unroll
    for (int a = 0; a < kNpt; ++a) prod[a] = ts.W;
    if (ts.bin <= E.K) {
      const double* lf = E.leaves + j * E.lmax * DIM;
      for (int l = 0; l < ts.nl; l += 4) {
        double d4[4][DIM];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int k = 0; k < DIM; ++k) d4[u][k] = (l + u < ts.nl) ? lf[(l + u) * DIM + k] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (l + u < ts.nl) {
#pragma unroll
            for (int a = 0; a < kNpt; ++a) {
              double xe[DIM];
#pragma unroll
              for (int k = 0; k < DIM; ++k) xe[k] = x[a][k] + d4[u][k];
              prod[a] *= g_eval<DIM, GK>(xe, E.amp, E.inv_scale, E.inv_scale2);
            }
          }
        }
      }
      if constexpr (!REC) {
#pragma unroll
        for (int a = 0; a < kNpt; ++a) {
          double* s1 = acc + (ts.bin * 2 + 0) * AS + a * kEvalThreads + tid;
          double* s2 = acc + (ts.bin * 2 + 1) * AS + a * kEvalThreads + tid;
          *s1 += prod[a];
          *s2 = fma(prod[a], prod[a], *s2);
        }
      }
    }
    if constexpr (REC) {
      const uint32_t rel = E.rel0 + static_cast<uint32_t>(j);
#pragma unroll
      for (int a = 0; a < kNpt; ++a) {
        if (valid[a]) {
          TreeRec r;
          r.ne = ts.ne; r.leaves = ts.nl; r.particles = ts.parts; r.pruned = ts.bin > E.K ? 1 : 0;
          r.C = ts.bin > E.K ? 0.0 : prod[a];
          E.recs[static_cast<int64_t>(node[a]) * E.n_rec + (rel >> E.rec_shift)] = r;
        }
      }
    } else {
      if (tid == 0) cnt[ts.bin] += 1;
    }
  }
  if constexpr (!REC) {
    __syncthreads();
#pragma unroll
    for (int a = 0; a < kNpt; ++a) {
      if (valid[a]) {
        double* o = E.partials + (static_cast<int64_t>(node[a]) * E.tpn_total + E.q0 + blockIdx.y) * E.nb * 3;
        for (int b = 0; b < E.nb; ++b) {
          o[b * 3 + 0] = acc[(b * 2 + 0) * AS + a * kEvalThreads + tid];
          o[b * 3 + 1] = acc[(b * 2 + 1) * AS + a * kEvalThreads + tid];
          o[b * 3 + 2] = static_cast<double>(cnt[b]);
        }
      }
    }
  }
}

}  // namespace rtk
