// tree_walk.cuh — the random-tree walk kernel (rows a3–a7).
//
// One lane = one tree at a time; one warp = a static stream of (node, tree)
// tasks.  Each loop iteration advances EVERY lane by exactly one particle, so
// the expensive part of an iteration (2–3 Philox blocks, logs, Box–Muller,
// sqrt — PAPER.md:197-204 exponential clock, PAPER.md:174-191 Brownian
// increment) runs with all 32 lanes converged whatever the trees look like;
// the tree logic after it is short predicated straight-line code.  A lane
// whose tree ends takes the next tree of the warp's stream in the next
// iteration (ballot + popc compaction), so no lane idles until the stream
// runs dry.
//
// Depth-first order (child 0 first): the pending sibling
// groups form a per-lane stack in shared memory (SoA [level][field][lane],
// conflict-free), with levels >= LV in a per-warp global spill area (rare:
// LV is sized from the depth distribution).  A group stores the
// split position y, remaining horizon τ_c and a packed (next child label |
// remaining count << 56).
//
// Order binning: a finished tree appends
// (bin, C) to its task slot's 64-entry per-warp ring in shared memory and
// bumps the slot's integer bin count (shared atomic: exact in any order);
// when 32 records are pending the warp "transposes" them: lane b owns order
// bin b and accumulates, in ring order, the records whose bin is b (ΣC, ΣC²;
// deterministic).  When all trees of a task are recorded, lane b writes the
// task's bin b to partials[task][b] (atomic-free); a second kernel sums each
// node's tasks in task order.  Two task slots let the stream run past a task
// boundary while the previous task's last trees finish.
#pragma once
#include <cstdint>

#include "philox.cuh"
#include "rt_math.cuh"

namespace rtk {

constexpr int kWarpsPerCta = 4;
constexpr int kThreads = 32 * kWarpsPerCta;
constexpr int kRing = 64;
constexpr uint64_t kLabelMask = (1ull << 56) - 1;
// per-warp record rings [2 slots][kRing] (C, bin), bin sums [2][2][32], counts [2][32]
constexpr int kWarpExtra = 2 * kRing * 8 + 2 * 2 * 32 * 8 + 2 * kRing * 4 + 2 * 32 * 4;

// Stack levels kept in shared memory per lane, and resident CTAs per SM (the
// register budget 65536 / (128 v) and the 228 KB of shared memory).  The
// record-emitting trace variant gets one CTA less so it never spills; it is
// launched on the production kernel's grid, so both give identical sums.
template <int DIM> struct Levels;
template <> struct Levels<1> { static constexpr int v = 7; };
template <> struct Levels<2> { static constexpr int v = 5; };
template <> struct Levels<3> { static constexpr int v = 6; };
template <int DIM, bool REC> struct MinCtas {
  static constexpr int v = (DIM == 3 ? 5 : 6) - (REC ? 1 : 0);
};

struct TreeRec {   // mirrors rt_tree_rec
  int32_t ne, leaves, particles, pruned;
  double C;
};

struct WalkParams {
  RoundKeys rk;
  double inv_lambda, two_d, amp, inv_scale, inv_scale2, t;
  double w[9];
  uint32_t thr[9];      // T_k - 1 for support entries (ascending); 0xffffffff past the end
  int32_t kval[9];
  int32_t n_support, beta, K, nb;   // nb = K + 2 bins (K+1 = pruned)
  const double* points;
  int32_t n_trees, T, tpn, n_tasks;   // trees per node (< 2^31), per task, tasks per node, tasks
  uint32_t tree_offset;               // first tree index (tree indices are uint32)
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
    if constexpr (GK == 2) return P.amp * exp_neg(-r2 * P.inv_scale2);
    else return P.amp * rcp_nr(fma(r2, P.inv_scale2, 1.0));
  }
}

template <int DIM>
__host__ __device__ constexpr int stack_bytes_per_warp() {
  return Levels<DIM>::v * (DIM + 2) * 32 * 8;
}

template <int DIM>
__host__ __device__ constexpr int smem_bytes() {
  return 128 * 16 /* log table */ + kWarpsPerCta * (stack_bytes_per_warp<DIM>() + kWarpExtra) +
         9 * 8 + 9 * 4 /* offspring weights and sizes */;
}

template <int DIM, int GK, bool REC>
__global__ void __launch_bounds__(kThreads, MinCtas<DIM, REC>::v)
tree_walk_kernel(const __grid_constant__ WalkParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int NF = DIM + 2;
  constexpr int LV = Levels<DIM>::v;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;

  // ---- shared memory carve-up -------------------------------------------
  LogEntry* const ltab = reinterpret_cast<LogEntry*>(smem_raw);
  unsigned char* const wbase = smem_raw + 128 * 16 + wib * (stack_bytes_per_warp<DIM>() + kWarpExtra);
  double* const ssp = reinterpret_cast<double*>(wbase) + lane;            // [LV][NF][32]
  double* const ringC = reinterpret_cast<double*>(wbase + stack_bytes_per_warp<DIM>());
  double* const bsum = ringC + 2 * kRing;                                 // [slot][ΣC, ΣC²][32]
  int* const ringBin = reinterpret_cast<int*>(bsum + 2 * 2 * 32);         // [slot][kRing]
  int* const bcnt = ringBin + 2 * kRing;                                  // [slot][32]
  double* const wtab = reinterpret_cast<double*>(smem_raw + 128 * 16 +
      kWarpsPerCta * (stack_bytes_per_warp<DIM>() + kWarpExtra));        // [9] weights
  int* const ktab = reinterpret_cast<int*>(wtab + 9);                     // [9] offspring k
  for (int q = threadIdx.x; q < 128; q += kThreads) ltab[q] = kLogTable[q];
  if (threadIdx.x < 9) {
    wtab[threadIdx.x] = P.w[threadIdx.x];
    ktab[threadIdx.x] = P.kval[threadIdx.x];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) bsum[q * 32 + lane] = 0.0;
  bcnt[lane] = 0;
  bcnt[32 + lane] = 0;
  __syncthreads();

  const int gwarp = blockIdx.x * kWarpsPerCta + wib;
  const int W = gridDim.x * kWarpsPerCta;
  double* const gsp = P.spill + static_cast<int64_t>(gwarp) * P.spill_levels * NF * 32 + lane;

  // ---- warp-uniform stream state (32-bit) ----------------------------------
  // the task being issued: id, trees issued / in it, its first tree index and
  // its node's coordinates
  int iss_task = gwarp, iss_next = 0, iss_size = 0, iss_slot = 0;
  uint32_t iss_j0 = 0u, iss_node = 0u;
  double iss_y[DIM];
  bool stream_end = iss_task >= P.n_tasks;
  auto open_task = [&](int task) {
    const int node = task / P.tpn;
    const int q = task - node * P.tpn;
    iss_size = min(P.T, P.n_trees - q * P.T);
    iss_node = static_cast<uint32_t>(node);
    iss_j0 = static_cast<uint32_t>(P.tree_offset) + static_cast<uint32_t>(q * P.T);
#pragma unroll
    for (int k = 0; k < DIM; ++k) iss_y[k] = P.points[node * DIM + k];
  };
#pragma unroll
  for (int k = 0; k < DIM; ++k) iss_y[k] = 0.0;
  if (!stream_end) open_task(iss_task);
  int slot_task0 = stream_end ? -1 : iss_task, slot_task1 = -1;
  int slot_left0 = iss_size, slot_left1 = 0;
  int ring_head0 = 0, ring_cnt0 = 0, ring_head1 = 0, ring_cnt1 = 0;

  // ---- lane state ----------------------------------------------------------
  bool active = false;
  int slot = 0;
  uint32_t ti = 0, tj = 0;
  double y[DIM];
#pragma unroll
  for (int k = 0; k < DIM; ++k) y[k] = 0.0;
  double tau = 0.0, Pi = 1.0;
  uint64_t label = 1;
  int ne = 0, sp = 0;
  int leaves = 0, parts = 0;           // per-tree counts (trace variant only)
  uint32_t c_part = 0u, c_leaf = 0u;   // particles / leaves since the last task close

  while (true) {
    // ---------------- assign trees to idle lanes (warp-uniform control) -----
    unsigned idle = __ballot_sync(0xffffffffu, !active);
    while (idle != 0u && !stream_end) {
      const int avail = iss_size - iss_next;
      if (avail == 0) {
        const int nt = iss_task + W;
        if (nt >= P.n_tasks) { stream_end = true; break; }
        const int ns = iss_slot ^ 1;
        if ((ns == 0 ? slot_task0 : slot_task1) != -1) break;   // previous task still open
        iss_task = nt; iss_next = 0; iss_slot = ns;
        open_task(nt);
        if (ns == 0) { slot_task0 = nt; slot_left0 = iss_size; }
        else { slot_task1 = nt; slot_left1 = iss_size; }
        continue;
      }
      const int nidle = __popc(idle);
      const int take = min(avail, nidle);
      const int rank = __popc(idle & lt_mask);
      if (!active && rank < take) {
        ti = iss_node;
        tj = iss_j0 + static_cast<uint32_t>(iss_next + rank);
        slot = iss_slot;
#pragma unroll
        for (int k = 0; k < DIM; ++k) y[k] = iss_y[k];
        tau = P.t; label = 1; Pi = 1.0; ne = 0; sp = 0;
        if constexpr (REC) { leaves = 0; parts = 0; }
        active = true;
      }
      iss_next += take;
      idle = __ballot_sync(0xffffffffu, !active);
    }
    if (!__any_sync(0xffffffffu, active)) break;

    // ---------------- one particle per lane (converged) ----------------------
    const uint32_t c2 = static_cast<uint32_t>(label);
    const uint32_t c3 = static_cast<uint32_t>(label >> 32);
    const uint4 r0 = philox4x32_10(tj, ti, c2, c3, P.rk);
    const uint4 r1 = philox4x32_10(tj, ti, c2, c3 | (1u << 24), P.rk);
    // exponential clock S ~ λ e^{-λS}
    const double S = -log_tab(unif53(r0.x, r0.y), ltab) * P.inv_lambda;
    const bool leaf = S > tau;                  // 1{S > t}
    const double h2d = (leaf ? tau : S) * P.two_d;   // variance 2D·h of the increment
    // Box–Muller with the lifetime folded into the radius (R8):
    // σ sqrt(h) · sqrt(-2 log v1) · (cos, sin)(2π v2)
    double x[DIM];
    {
      const double v1 = unif53(r1.x, r1.y), v2 = unif53(r1.z, r1.w);
      const double rad = sqrt_nr(-2.0 * log_tab(v1, ltab) * h2d);
      double sn, cs;
      sincospi2(2.0 * v2, sn, cs);
      x[0] = fma(rad, cs, y[0]);
      if constexpr (DIM >= 2) x[1] = fma(rad, sn, y[1]);
    }
    if constexpr (DIM == 3) {
      const uint4 r2 = philox4x32_10(tj, ti, c2, c3 | (2u << 24), P.rk);
      const double v3 = unif53(r2.x, r2.y), v4 = unif53(r2.z, r2.w);
      const double rad2 = sqrt_nr(-2.0 * log_tab(v3, ltab) * h2d);
      x[2] = fma(rad2, cospi2(2.0 * v4), y[2]);
    }
    // categorical offspring choice from the integer thresholds (R9)
    const uint32_t c32 = r0.z;
    int s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q + 1 >= P.n_support) break;          // warp-uniform (kernel parameter)
      s += (c32 > P.thr[q]) ? 1 : 0;
    }
    const double gv = g_eval<DIM, GK>(x, P);    // g at the leaf
    const int k = ktab[s];
    const double wk = wtab[s];

    // ---------------- tree logic: predicated straight-line code ---------------
    const bool split = active && !leaf;
    ne += split ? 1 : 0;                         // splitting events
    const bool pruned = split && ne > P.K;       // prune
    const bool kill = split && !pruned && P.n_support == 0;   // purely linear f
    const bool branch = split && !pruned && !kill;
    // g at a leaf; h^(α) = c'_α at a split; 0 if killed
    const double fac = leaf ? gv : (kill ? 0.0 : wk);
    if (active) Pi *= fac;
    c_part += active ? 1u : 0u;
    c_leaf += (active && leaf) ? 1u : 0u;
    if constexpr (REC) {
      parts += active ? 1 : 0;
      leaves += (active && leaf) ? 1 : 0;
    }
    const bool child = branch && k > 0;          // continue with child 0
    const bool push = child && k > 1;            // k-1 younger siblings wait
    const bool pop = (active && leaf) || (branch && k == 0);
    const double tc = tau - S;
    const uint64_t base = label << P.beta;
    if (push) {
      const uint64_t pk = (base | 1ull) | (static_cast<uint64_t>(k - 1) << 56);
      if (sp < LV) {
#pragma unroll
        for (int q = 0; q < DIM; ++q) ssp[(sp * NF + q) * 32] = x[q];
        ssp[(sp * NF + DIM) * 32] = tc;
        ssp[(sp * NF + DIM + 1) * 32] = __longlong_as_double(static_cast<long long>(pk));
      } else {
        double* b = gsp + (sp - LV) * (NF * 32);
#pragma unroll
        for (int q = 0; q < DIM; ++q) b[q * 32] = x[q];
        b[DIM * 32] = tc;
        b[(DIM + 1) * 32] = __longlong_as_double(static_cast<long long>(pk));
      }
      ++sp;
    }
    if (child) {
#pragma unroll
      for (int q = 0; q < DIM; ++q) y[q] = x[q];
      tau = tc;
      label = base;
    }
    bool done = pruned || kill || (pop && sp == 0);
    if (pop && sp > 0) {
      const int lvl = sp - 1;
      uint64_t pk;
      if (lvl < LV) {
#pragma unroll
        for (int q = 0; q < DIM; ++q) y[q] = ssp[(lvl * NF + q) * 32];
        tau = ssp[(lvl * NF + DIM) * 32];
        pk = static_cast<uint64_t>(__double_as_longlong(ssp[(lvl * NF + DIM + 1) * 32]));
      } else {
        const double* b = gsp + (lvl - LV) * (NF * 32);
#pragma unroll
        for (int q = 0; q < DIM; ++q) y[q] = b[q * 32];
        tau = b[DIM * 32];
        pk = static_cast<uint64_t>(__double_as_longlong(b[(DIM + 1) * 32]));
      }
      label = pk & kLabelMask;
      if ((pk >> 56) == 1ull) {
        sp = lvl;                               // last sibling: drop the group
      } else {
        const double npk = __longlong_as_double(static_cast<long long>(pk + 1ull - (1ull << 56)));
        if (lvl < LV) ssp[(lvl * NF + DIM + 1) * 32] = npk;
        else gsp[((lvl - LV) * NF + DIM + 1) * 32] = npk;
      }
    }

    if constexpr (REC) {
      const uint32_t rel = tj - static_cast<uint32_t>(P.tree_offset);
      if (done && (rel & ((1u << P.rec_shift) - 1u)) == 0u) {
        TreeRec r;
        r.ne = ne; r.leaves = leaves; r.particles = parts; r.pruned = pruned ? 1 : 0;
        r.C = pruned ? 0.0 : Pi;
        P.recs[static_cast<int64_t>(ti) * P.n_rec + (rel >> P.rec_shift)] = r;
      }
    }

    // ---------------- record finished trees; flush; close tasks -------------
    const unsigned fin = __ballot_sync(0xffffffffu, done);
    if (fin != 0u) {
      const unsigned fin1 = __ballot_sync(0xffffffffu, done && slot == 1);
      const unsigned fin0 = fin & ~fin1;
      if (done) {
        const int bin = pruned ? (P.K + 1) : ne;
        const int e = slot ? (ring_head1 + ring_cnt1 + __popc(fin1 & lt_mask)) & (kRing - 1)
                           : (ring_head0 + ring_cnt0 + __popc(fin0 & lt_mask)) & (kRing - 1);
        ringBin[slot * kRing + e] = bin;
        ringC[slot * kRing + e] = pruned ? 0.0 : Pi;
        atomicAdd(bcnt + slot * 32 + bin, 1);   // integer: exact in any order
        active = false;
      }
      ring_cnt0 += __popc(fin0);
      ring_cnt1 += __popc(fin1);
      slot_left0 -= __popc(fin0);
      slot_left1 -= __popc(fin1);
      __syncwarp();
      const bool cl0 = slot_task0 >= 0 && slot_left0 == 0;
      const bool cl1 = slot_task1 >= 0 && slot_left1 == 0;
#pragma unroll
      for (int sl = 0; sl < 2; ++sl) {
        const bool close = sl ? cl1 : cl0;
        int& head = sl ? ring_head1 : ring_head0;
        int& cnt = sl ? ring_cnt1 : ring_cnt0;
        if (close || cnt >= 32) {
          // transpose: lane b accumulates, in ring order, the records of bin b
          const int nflush = close ? cnt : 32;
          double a1 = bsum[(sl * 2 + 0) * 32 + lane], a2 = bsum[(sl * 2 + 1) * 32 + lane];
          const int* rb = ringBin + sl * kRing;
          const double* rc = ringC + sl * kRing;
          for (int r = 0; r < nflush; ++r) {
            const int e = (head + r) & (kRing - 1);
            const int b = rb[e];
            const double C = rc[e];
            if (b == lane) {
              a1 += C;
              a2 = fma(C, C, a2);
            }
          }
          head = (head + nflush) & (kRing - 1);
          cnt -= nflush;
          if (close) {
            const int task = sl ? slot_task1 : slot_task0;
            if (lane < P.nb) {
              double* o = P.partials + (static_cast<int64_t>(task) * P.nb + lane) * 3;
              o[0] = a1; o[1] = a2; o[2] = static_cast<double>(bcnt[sl * 32 + lane]);
            }
            bcnt[sl * 32 + lane] = 0;
            a1 = 0.0; a2 = 0.0;
            if (sl) slot_task1 = -1; else slot_task0 = -1;
            // fold the lanes' 32-bit event counters into the 64-bit totals
            unsigned long long v0 = c_part, v1 = c_leaf;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              v0 += __shfl_xor_sync(0xffffffffu, v0, o);
              v1 += __shfl_xor_sync(0xffffffffu, v1, o);
            }
            if (lane == 0) {
              atomicAdd(P.stats + 2, v0);
              atomicAdd(P.stats + 3, v1);
            }
            c_part = 0u;
            c_leaf = 0u;
          }
          bsum[(sl * 2 + 0) * 32 + lane] = a1;
          bsum[(sl * 2 + 1) * 32 + lane] = a2;
          __syncwarp();
        }
      }
    }
  }
  // (trees, pruned trees and splits follow exactly from the bin counts and are
  // added by the task-reduction kernel; every task close folded c_part/c_leaf)
}

}  // namespace rtk
