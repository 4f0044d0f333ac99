// tree_walk.cuh — the random-tree walk kernel (rows a3–a7).
//
// One lane = one tree at a time; one warp = a static stream of (node, tree)
// tasks.  Each loop iteration advances EVERY lane by exactly one particle, so
// the expensive part of an iteration (3 Philox blocks, log, Box–Muller,
// sqrt — PAPER.md:197-204 exponential clock, PAPER.md:174-191 Brownian
// increment) runs with all 32 lanes converged whatever the trees look like;
// only the short leaf / split / pop tails diverge.  A lane whose tree ends
// takes the next tree of the warp's stream in the same iteration
// (ballot + popc compaction), so no lane idles until the stream runs dry.
//
// Depth-first order (child 0 first): the pending sibling
// groups form a per-lane stack in shared memory (SoA [level][field][lane],
// conflict-free), with levels >= LV in a per-warp global spill area.
// A group stores the split position y, remaining horizon τ_c and a packed
// (next child label | remaining count << 56).
//
// Order binning: a finished tree appends
// (bin | slot << 5, C) to a 64-entry per-warp ring in shared memory; when 32
// records are pending the warp "transposes" them: lane b owns order bin b and
// accumulates, in ring order, the records whose bin is b (ΣC, ΣC², count in
// registers; deterministic).  When all trees of a task are recorded, lane b
// writes the task's bin b to partials[task][b] (atomic-free); a second kernel
// sums each node's tasks in task order.  Two task slots let the stream run
// past a task boundary while the previous task's last trees finish.
#pragma once
#include <cstdint>

#include "philox.cuh"

namespace rtk {

constexpr int kWarpsPerCta = 4;
constexpr int kThreads = 32 * kWarpsPerCta;
constexpr int kRing = 64;
constexpr uint64_t kLabelMask = (1ull << 56) - 1;

struct TreeRec {   // mirrors rt_tree_rec
  int32_t ne, leaves, particles, pruned;
  double C;
};

struct WalkParams {
  RoundKeys rk;
  double inv_lambda, sigma, amp, inv_scale, inv_scale2, t;
  double w[9];
  uint32_t thr[9];      // T_k - 1 for support entries (ascending)
  int32_t kval[9];
  int32_t n_support, beta, K, nb;   // nb = K + 2 bins (K+1 = pruned)
  const double* points;
  int64_t n_trees, tree_offset, T, tpn, n_tasks;
  double* partials;     // [n_tasks][nb][3]
  double* spill;        // [warps][spill_levels][DIM+2][32]
  int32_t spill_levels;
  TreeRec* recs;
  int32_t rec_shift;
  int64_t n_rec;
  unsigned long long* stats;   // trees, pruned, particles, leaves, splits
};

template <int DIM, int GK>
__device__ __forceinline__ double g_eval(const double (&x)[DIM], const WalkParams& P) {
  if constexpr (GK == 0) {
    return P.amp;
  } else if constexpr (GK == 1) {
    return P.amp * 0.5 * (1.0 + tanh(x[0] * P.inv_scale));
  } else {
    double r2 = x[0] * x[0];
    if constexpr (DIM >= 2) r2 = fma(x[1], x[1], r2);
    if constexpr (DIM >= 3) r2 = fma(x[2], x[2], r2);
    if constexpr (GK == 2) return P.amp * exp(-r2 * P.inv_scale2);
    else return P.amp / fma(r2, P.inv_scale2, 1.0);
  }
}

template <int DIM, int LV>
struct LaneStack {
  static constexpr int NF = DIM + 2;
  double* smem;     // this warp's [LV][NF][32]
  double* gmem;     // this warp's spill [levels][NF][32]
  int lane;
  __device__ __forceinline__ void push(int lvl, const double (&y)[DIM], double tau, uint64_t pk) {
    if (lvl < LV) {
      double* b = smem + lvl * NF * 32 + lane;
#pragma unroll
      for (int k = 0; k < DIM; ++k) b[k * 32] = y[k];
      b[DIM * 32] = tau;
      b[(DIM + 1) * 32] = __longlong_as_double(static_cast<long long>(pk));
    } else {
      double* b = gmem + (lvl - LV) * NF * 32 + lane;
#pragma unroll
      for (int k = 0; k < DIM; ++k) b[k * 32] = y[k];
      b[DIM * 32] = tau;
      b[(DIM + 1) * 32] = __longlong_as_double(static_cast<long long>(pk));
    }
  }
  __device__ __forceinline__ void top(int lvl, double (&y)[DIM], double& tau, uint64_t& pk) const {
    const double* b = (lvl < LV) ? smem + lvl * NF * 32 + lane
                                 : gmem + (lvl - LV) * NF * 32 + lane;
#pragma unroll
    for (int k = 0; k < DIM; ++k) y[k] = b[k * 32];
    tau = b[DIM * 32];
    pk = static_cast<uint64_t>(__double_as_longlong(b[(DIM + 1) * 32]));
  }
  __device__ __forceinline__ void set_packed(int lvl, uint64_t pk) {
    double* b = (lvl < LV) ? smem + lvl * NF * 32 + lane : gmem + (lvl - LV) * NF * 32 + lane;
    b[(DIM + 1) * 32] = __longlong_as_double(static_cast<long long>(pk));
  }
};

template <int DIM, int LV>
constexpr int smem_bytes() {
  return kWarpsPerCta * (LV * (DIM + 2) * 32 * 8 + kRing * (8 + 4));
}

__device__ __forceinline__ int64_t task_size(const WalkParams& P, int64_t task) {
  const int64_t q = task % P.tpn;
  const int64_t rem = P.n_trees - q * P.T;
  return rem < P.T ? rem : P.T;
}

template <int DIM, int GK, int LV, bool REC>
__global__ void __launch_bounds__(kThreads, 4) tree_walk_kernel(const __grid_constant__ WalkParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int NF = DIM + 2;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  double* const stk_all = reinterpret_cast<double*>(smem_raw);
  double* const ringC = stk_all + kWarpsPerCta * LV * NF * 32 + wib * kRing;
  int* const ringCode =
      reinterpret_cast<int*>(stk_all + kWarpsPerCta * LV * NF * 32 + kWarpsPerCta * kRing) +
      wib * kRing;
  const int64_t gwarp = static_cast<int64_t>(blockIdx.x) * kWarpsPerCta + wib;
  const int64_t W = static_cast<int64_t>(gridDim.x) * kWarpsPerCta;

  LaneStack<DIM, LV> stack{stk_all + wib * LV * NF * 32,
                           P.spill + gwarp * static_cast<int64_t>(P.spill_levels) * NF * 32, lane};

  // order bin `lane` of the two task slots
  double s1a = 0.0, s2a = 0.0, s1b = 0.0, s2b = 0.0;
  uint32_t na = 0, nbn = 0;

  // warp-uniform stream state
  int64_t iss_task = gwarp, iss_next = 0, iss_size = 0, iss_node = 0, iss_j0 = 0;
  int iss_slot = 0;
  bool stream_end = iss_task >= P.n_tasks;
  if (!stream_end) {
    iss_size = task_size(P, iss_task);
    iss_node = iss_task / P.tpn;
    iss_j0 = P.tree_offset + (iss_task - iss_node * P.tpn) * P.T;
  }
  int64_t slot_task0 = stream_end ? -1 : iss_task, slot_task1 = -1;
  int64_t slot_left0 = iss_size, slot_left1 = 0;
  int ring_head = 0, ring_cnt = 0;

  // lane state
  bool active = false;
  int slot = 0;
  uint32_t ti = 0, tj = 0;
  double y[DIM];
#pragma unroll
  for (int k = 0; k < DIM; ++k) y[k] = 0.0;
  double tau = 0.0, Pi = 1.0;
  uint64_t label = 1;
  int ne = 0, leaves = 0, sp = 0, parts = 0;

  unsigned long long st_particles = 0, st_leaves = 0, st_splits = 0;
  uint32_t st_pruned = 0, st_trees = 0;

  while (true) {
    // ---------------- assign trees to idle lanes (warp-uniform control) -----
    unsigned idle = __ballot_sync(0xffffffffu, !active);
    while (idle != 0u && !stream_end) {
      const int64_t avail = iss_size - iss_next;
      if (avail == 0) {
        const int64_t nt = iss_task + W;
        if (nt >= P.n_tasks) { stream_end = true; break; }
        const int ns = iss_slot ^ 1;
        if ((ns == 0 ? slot_task0 : slot_task1) != -1) break;   // previous task still open
        iss_task = nt; iss_next = 0; iss_slot = ns;
        iss_size = task_size(P, nt);
        iss_node = nt / P.tpn;
        iss_j0 = P.tree_offset + (nt - iss_node * P.tpn) * P.T;
        if (ns == 0) { slot_task0 = nt; slot_left0 = iss_size; }
        else { slot_task1 = nt; slot_left1 = iss_size; }
        continue;
      }
      const int nidle = __popc(idle);
      const int take = avail < nidle ? static_cast<int>(avail) : nidle;
      const int rank = __popc(idle & lt_mask);
      if (!active && rank < take) {
        ti = static_cast<uint32_t>(iss_node);
        tj = static_cast<uint32_t>(iss_j0 + iss_next + rank);
        slot = iss_slot;
#pragma unroll
        for (int k = 0; k < DIM; ++k) y[k] = P.points[iss_node * DIM + k];
        tau = P.t; label = 1; Pi = 1.0; ne = 0; leaves = 0; sp = 0; parts = 0;
        active = true;
      }
      iss_next += take;
      idle = __ballot_sync(0xffffffffu, !active);
    }
    if (!__any_sync(0xffffffffu, active)) break;

    // ---------------- one particle per active lane ---------------------------
    bool done = false, pruned = false;
    if (active) {
      ++parts;
      const uint32_t c2 = static_cast<uint32_t>(label);
      const uint32_t c3 = static_cast<uint32_t>(label >> 32);
      const uint4 r0 = philox4x32_10(tj, ti, c2, c3, P.rk);
      const uint4 r1 = philox4x32_10(tj, ti, c2, c3 | (1u << 24), P.rk);
      // exponential clock S ~ λ e^{-λS}
      const double S = -log(unif53(r0.x, r0.y)) * P.inv_lambda;
      const bool leaf = S > tau;                 // 1{S > t}
      const double h = leaf ? tau : S;
      // Box–Muller normals (R8)
      double xi[DIM];
      {
        const double v1 = unif53(r1.x, r1.y), v2 = unif53(r1.z, r1.w);
        const double rad = sqrt(-2.0 * log(v1));
        double sn, cs;
        sincospi(2.0 * v2, &sn, &cs);
        xi[0] = rad * cs;
        if constexpr (DIM >= 2) xi[1] = rad * sn;
      }
      if constexpr (DIM == 3) {
        const uint4 r2 = philox4x32_10(tj, ti, c2, c3 | (2u << 24), P.rk);
        const double v3 = unif53(r2.x, r2.y), v4 = unif53(r2.z, r2.w);
        xi[2] = sqrt(-2.0 * log(v3)) * cospi(2.0 * v4);
      }
      const double stepk = P.sigma * sqrt(h);
      double x[DIM];
#pragma unroll
      for (int k = 0; k < DIM; ++k) x[k] = fma(stepk, xi[k], y[k]);

      bool pop = false;
      if (leaf) {
        Pi *= g_eval<DIM, GK>(x, P);             // g at the leaf
        ++leaves;
        pop = true;
      } else {
        ++ne;                                    // splitting event
        if (ne > P.K) {
          done = true; pruned = true;            // prune
        } else if (P.n_support == 0) {
          Pi = 0.0; done = true;                 // purely linear f: the ring kills the tree
        } else {
          const uint32_t c32 = r0.z;
          int s = 0;
          for (int q = 0; q + 1 < P.n_support; ++q) s += (c32 > P.thr[q]) ? 1 : 0;
          const int k = P.kval[s];
          Pi *= P.w[s];                          // h^(α) = c'_α
          if (k == 0) {
            pop = true;
          } else {
            const double tc = tau - S;
            const uint64_t base = label << P.beta;
            if (k > 1) {
              stack.push(sp, x, tc, (base | 1ull) | (static_cast<uint64_t>(k - 1) << 56));
              ++sp;
            }
#pragma unroll
            for (int q = 0; q < DIM; ++q) y[q] = x[q];
            tau = tc;
            label = base;                        // child 0 first
          }
        }
      }
      if (pop) {
        if (sp == 0) {
          done = true;
        } else {
          uint64_t pk;
          stack.top(sp - 1, y, tau, pk);
          label = pk & kLabelMask;
          const uint32_t rem = static_cast<uint32_t>(pk >> 56);
          if (rem == 1u) --sp;
          else stack.set_packed(sp - 1, pk + 1ull - (1ull << 56));
        }
      }
      if (done) {
        st_particles += static_cast<unsigned long long>(parts);
        st_leaves += static_cast<unsigned long long>(leaves);
        st_splits += static_cast<unsigned long long>(ne);
        ++st_trees;
        if (pruned) ++st_pruned;
        if constexpr (REC) {
          const uint32_t rel = tj - static_cast<uint32_t>(P.tree_offset);
          if ((rel & ((1u << P.rec_shift) - 1u)) == 0u) {
            TreeRec r;
            r.ne = ne; r.leaves = leaves; r.particles = parts; r.pruned = pruned ? 1 : 0;
            r.C = pruned ? 0.0 : Pi;
            P.recs[static_cast<int64_t>(ti) * P.n_rec + (rel >> P.rec_shift)] = r;
          }
        }
      }
    }

    // ---------------- record finished trees; flush; close tasks -------------
    const unsigned fin = __ballot_sync(0xffffffffu, done);
    if (fin != 0u) {
      if (done) {
        const int e = (ring_head + ring_cnt + __popc(fin & lt_mask)) & (kRing - 1);
        ringCode[e] = (pruned ? (P.K + 1) : ne) | (slot << 5);
        ringC[e] = pruned ? 0.0 : Pi;
        active = false;
      }
      const unsigned fin1 = __ballot_sync(0xffffffffu, done && slot == 1);
      ring_cnt += __popc(fin);
      slot_left1 -= __popc(fin1);
      slot_left0 -= __popc(fin) - __popc(fin1);
      __syncwarp();
      const bool c0 = slot_task0 >= 0 && slot_left0 == 0;
      const bool c1 = slot_task1 >= 0 && slot_left1 == 0;
      if (c0 || c1 || ring_cnt >= 32) {
        const int nflush = (c0 || c1) ? ring_cnt : 32;
        for (int r = 0; r < nflush; ++r) {
          const int e = (ring_head + r) & (kRing - 1);
          const int code = ringCode[e];
          const double C = ringC[e];
          if ((code & 31) == lane) {
            if (code >> 5) { s1b += C; s2b = fma(C, C, s2b); ++nbn; }
            else { s1a += C; s2a = fma(C, C, s2a); ++na; }
          }
        }
        ring_head = (ring_head + nflush) & (kRing - 1);
        ring_cnt -= nflush;
        __syncwarp();
        if (c0) {
          if (lane < P.nb) {
            double* o = P.partials + (slot_task0 * P.nb + lane) * 3;
            o[0] = s1a; o[1] = s2a; o[2] = static_cast<double>(na);
          }
          s1a = 0.0; s2a = 0.0; na = 0; slot_task0 = -1;
        }
        if (c1) {
          if (lane < P.nb) {
            double* o = P.partials + (slot_task1 * P.nb + lane) * 3;
            o[0] = s1b; o[1] = s2b; o[2] = static_cast<double>(nbn);
          }
          s1b = 0.0; s2b = 0.0; nbn = 0; slot_task1 = -1;
        }
      }
    }
  }

  // ---------------- counters ------------------------------------------------
  unsigned long long v[5] = {st_trees, st_pruned, st_particles, st_leaves, st_splits};
#pragma unroll
  for (int q = 0; q < 5; ++q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 5; ++q) atomicAdd(P.stats + q, v[q]);
  }
}

}  // namespace rtk
