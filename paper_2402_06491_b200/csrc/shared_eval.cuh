// shared_eval.cuh — shared trees (NEXT row f4), phase 2.
//
// Phase 1 (tree_walk_kernel<…, SH = true>) walked every tree ONCE for all
// nodes and stored its summary (order bin, weight product W, leaf count) and
// its leaf displacements δ_l from the root.  bin_sort_kernel orders each
// block of consecutive trees stably by order bin; then a CTA of 64 threads
// takes 128 nodes (two per thread) and one tree block; every thread runs the
// same trees in the same order, so control flow is identical across the warp
// and the tree data are warp-uniform loads (L1/L2 broadcasts):
//   C_i = W · Π_l g(x_i + δ_l)  (leaves at x_i + δ),
// accumulated per order bin (ΣC, ΣC²; counts are node-free) in registers,
// one bin run at a time.  Results per (node, tree block) go to the per-node
// task partials that the shared task reduction sums in block order
// (deterministic).  Gaussian g: phase 1 stored each tree's leaf mean μ and
// scatter V instead of its leaves, and C_i = W amp^L e^{−(L|x_i+μ|² + V)/s²}
// is ONE exponential per (node, tree) whatever the leaf count (the identity
// Σ_l |x+δ_l|² = L|x+μ|² + Σ_l |δ_l−μ|²; both terms ≥ 0, so no cancellation
// against the node position); the CTA stages 64 trees' (W, L, μ, V) in
// shared memory at a time.
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
  TreeSum* sorted;           // [M] the chunk's summaries, stably sorted by bin within each block
  int32_t* boff;             // [blocks][nb + 1] each block's bin runs in `sorted`
};

// Per tree block (tpb consecutive trees), a stable counting sort of the trees
// by order bin — one warp per block: match_any groups equal bins, ranks are
// ballot prefix counts, so trees of a bin keep their index order (the sort,
// and so the summation order of phase 2, is a function of the chunk alone).
// sorted[r].parts carries the tree's index in the chunk (phase 2 needs
// neither the split nor the particle count).
__global__ void __launch_bounds__(32) bin_sort_kernel(const __grid_constant__ EvalParams E) {
  __shared__ int base[64];
  const int lane = threadIdx.x;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * E.tpb;
  const int64_t j1 = min(E.M, j0 + E.tpb);
  for (int b = lane; b < E.nb; b += 32) base[b] = 0;
  __syncwarp();
  for (int64_t j = j0 + lane; j - lane < j1; j += 32) {      // histogram
    const bool in = j < j1;
    const int b = in ? E.tsum[j].bin : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, b);
    if (in && (peers & lt) == 0u) base[b] += __popc(peers);  // one leader per bin
    __syncwarp();
  }
  if (lane == 0) {                                           // exclusive scan (nb <= 64)
    int acc = 0;
    int32_t* bo = E.boff + static_cast<int64_t>(blockIdx.x) * (E.nb + 1);
    for (int b = 0; b < E.nb; ++b) { const int c = base[b]; base[b] = acc; bo[b] = acc; acc += c; }
    bo[E.nb] = acc;
  }
  __syncwarp();
  for (int64_t j = j0 + lane; j - lane < j1; j += 32) {      // stable scatter
    const bool in = j < j1;
    TreeSum ts;
    ts.bin = -1;
    if (in) ts = E.tsum[j];
    const unsigned peers = __match_any_sync(0xffffffffu, ts.bin);
    if (in) {
      const int pos = base[ts.bin] + __popc(peers & lt);
      RT_CHECK(pos >= 0 && pos < j1 - j0);
      ts.parts = static_cast<int32_t>(j);
      E.sorted[j0 + pos] = ts;
    }
    __syncwarp();
    if (in && (peers & lt) == 0u) base[ts.bin] += __popc(peers);
    __syncwarp();
  }
}

// Phase 2.  Each thread owns kNpt nodes (tree data loaded once serve them
// all; 1 for small node counts so no thread idles).  Non-REC: the block's
// trees are visited bin by bin in the sorted order, so the order-bin sums of
// a (node, block) are plain register accumulators, written out at the end of
// each bin's run — no shared memory, so occupancy is set by registers.  The
// next tree's summary is prefetched and leaves are loaded four at a time, so
// the global-load latency overlaps the g evaluations.  REC: every tree in
// index order, one record per (node, tree).
template <int DIM, int GK, bool REC, int kNpt>
__global__ void __launch_bounds__(kEvalThreads)
shared_eval_kernel(const __grid_constant__ EvalParams E) {
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
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * E.tpb;
  const int64_t j1 = min(E.M, j0 + E.tpb);
  __shared__ double sExp[32];                  // Gaussian g: the table exp's 2^(j/32)
  if constexpr (sh_moments<GK>()) {
    if (tid < 32) sExp[tid] = kExpT32[tid];
    __syncthreads();
  }

  // C_i = W Π_l g(x_i + δ_l) of tree ts (leaf slots of chunk tree jl)
  // Gaussian g: W amp^L e^{−(L|x+μ|² + V)/s²} (W carries amp^L; μ, V from
  // phase 1) — both terms non-negative, so the exponent is accurate to a few
  // ulps of itself wherever the node lies
  auto gauss_prod = [&](double W, int nl, const double (&m)[DIM + 1], double (&prod)[kNpt]) {
    const double V = m[DIM], L = static_cast<double>(nl);
#pragma unroll
    for (int a = 0; a < kNpt; ++a) {
      double q = 0.0;
#pragma unroll
      for (int k = 0; k < DIM; ++k) {
        const double z = x[a][k] + m[k];
        q = fma(z, z, q);
      }
      prod[a] = W * exp_neg_tab(-(fma(L, q, V) * E.inv_scale2), sExp);
    }
  };
  auto tree_prod = [&](const TreeSum& ts, int64_t jl, double (&prod)[kNpt]) {
    if constexpr (sh_moments<GK>()) {
      double m[DIM + 1];
#pragma unroll
      for (int k = 0; k <= DIM; ++k) m[k] = E.leaves[jl * (DIM + 1) + k];
      gauss_prod(ts.W, ts.nl, m, prod);
      return;
    }
#pragma unroll
    for (int a = 0; a < kNpt; ++a) prod[a] = ts.W;
    const double* lf = E.leaves + jl * E.lmax * DIM;
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
  };

  if constexpr (REC) {
    for (int64_t j = j0; j < j1; ++j) {
      const uint32_t rel = E.rel0 + static_cast<uint32_t>(j);
      if ((rel & ((1u << E.rec_shift) - 1u)) != 0u) continue;
      const TreeSum ts = E.tsum[j];
      double prod[kNpt];
      if (ts.bin <= E.K) tree_prod(ts, j, prod);
#pragma unroll
      for (int a = 0; a < kNpt; ++a) {
        if (valid[a]) {
          TreeRec r;
          r.ne = ts.ne; r.leaves = ts.nl; r.particles = ts.parts; r.pruned = ts.bin > E.K ? 1 : 0;
          r.C = ts.bin > E.K ? 0.0 : prod[a];
          E.recs[static_cast<int64_t>(node[a]) * E.n_rec + (rel >> E.rec_shift)] = r;
        }
      }
    }
  } else {
    const int32_t* bo = E.boff + static_cast<int64_t>(blockIdx.y) * (E.nb + 1);
    const TreeSum* srt = E.sorted + j0;
    int64_t ob[kNpt];
#pragma unroll
    for (int a = 0; a < kNpt; ++a)
      ob[a] = (static_cast<int64_t>(valid[a] ? node[a] : 0) * E.tpn_total + E.q0 + blockIdx.y) * E.nb * 3;
    const int n_kept = bo[E.K + 1];                  // runs of bins 0..K, then the pruned run
    if constexpr (sh_moments<GK>()) {
      // Gaussian g: the CTA stages 64 trees' (W, L, μ, V) in shared memory at
      // a time — one coalesced gather by all threads instead of a dependent
      // global load per tree per warp — then every thread walks them in order
      __shared__ double sW[kEvalThreads], sM[DIM + 1][kEvalThreads];
      __shared__ int sL[kEvalThreads];
      double s1[kNpt], s2[kNpt];
#pragma unroll
      for (int a = 0; a < kNpt; ++a) { s1[a] = 0.0; s2[a] = 0.0; }
      int b = 0, bend = bo[1];
      auto flush = [&]() {                           // bin b's run is complete
        const double cnt = static_cast<double>(bo[b + 1] - bo[b]);
#pragma unroll
        for (int a = 0; a < kNpt; ++a) {
          if (valid[a]) {
            double* o = E.partials + ob[a] + b * 3;
            o[0] = s1[a]; o[1] = s2[a]; o[2] = cnt;
          }
          s1[a] = 0.0; s2[a] = 0.0;
        }
        ++b;
        bend = bo[b + 1];
      };
      for (int r0 = 0; r0 < n_kept; r0 += kEvalThreads) {   // (CTA-uniform bounds)
        const int nt = min(kEvalThreads, n_kept - r0);
        __syncthreads();
        if (tid < nt) {
          const TreeSum ts = srt[r0 + tid];
          sW[tid] = ts.W;
          sL[tid] = ts.nl;
          const double* m = E.leaves + static_cast<int64_t>(ts.parts) * (DIM + 1);
#pragma unroll
          for (int k = 0; k <= DIM; ++k) sM[k][tid] = m[k];
        }
        __syncthreads();
        for (int u = 0; u < nt; ++u) {
          while (r0 + u >= bend) flush();
          double m[DIM + 1];
#pragma unroll
          for (int k = 0; k <= DIM; ++k) m[k] = sM[k][u];
          double prod[kNpt];
          gauss_prod(sW[u], sL[u], m, prod);
#pragma unroll
          for (int a = 0; a < kNpt; ++a) {
            s1[a] += prod[a];
            s2[a] = fma(prod[a], prod[a], s2[a]);
          }
        }
      }
      while (b <= E.K) flush();                      // the last run and the empty bins after it
    } else {
      TreeSum nxt;
      if (n_kept > 0) nxt = srt[0];
      int r = 0;
      for (int b = 0; b <= E.K; ++b) {
        const int r1 = bo[b + 1];
        double s1[kNpt], s2[kNpt];
#pragma unroll
        for (int a = 0; a < kNpt; ++a) { s1[a] = 0.0; s2[a] = 0.0; }
        for (; r < r1; ++r) {
          const TreeSum ts = nxt;
          if (r + 1 < n_kept) nxt = srt[r + 1];        // warp-uniform, prefetched
          double prod[kNpt];
          tree_prod(ts, ts.parts, prod);
#pragma unroll
          for (int a = 0; a < kNpt; ++a) {
            s1[a] += prod[a];
            s2[a] = fma(prod[a], prod[a], s2[a]);
          }
        }
        const double cnt = static_cast<double>(r1 - bo[b]);
#pragma unroll
        for (int a = 0; a < kNpt; ++a) {
          if (valid[a]) {
            double* o = E.partials + ob[a] + b * 3;
            o[0] = s1[a]; o[1] = s2[a]; o[2] = cnt;
          }
        }
      }
    }
    const double cpr = static_cast<double>(bo[E.nb] - bo[E.K + 1]);   // pruned trees: count only
#pragma unroll
    for (int a = 0; a < kNpt; ++a) {
      if (valid[a]) {
        double* o = E.partials + ob[a] + (E.K + 1) * 3;
        o[0] = 0.0; o[1] = 0.0; o[2] = cpr;
      }
    }
  }
}

}  // namespace rtk
