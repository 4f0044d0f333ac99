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
// (bin | task slot << 5, C) to a 64-entry per-warp ring in shared memory and
// bumps its slot's integer bin count (shared atomic: exact in any order);
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
// per-warp record ring [kRing] (C, bin | slot << 5), bin sums [2 slots][2][32],
// counts [2][32]; the ring is flushed completely once >= 32 records are pending
constexpr int kWarpExtra = kRing * 8 + 2 * 2 * 32 * 8 + kRing * 4 + 2 * 32 * 4;

// Stack levels kept in shared memory per lane, and resident CTAs per SM (the
// register budget 65536 / (128 v) and the 228 KB of shared memory).  The
// record-emitting trace variant gets one CTA less so it never spills; it is
// launched on the production kernel's grid, so both give identical sums.
template <int DIM> struct Levels;
template <> struct Levels<1> { static constexpr int v = 7; };
template <> struct Levels<2> { static constexpr int v = 5; };
template <> struct Levels<3> { static constexpr int v = 5; };
template <int DIM, bool REC> struct MinCtas {
  static constexpr int v = (DIM == 3 ? 6 : 7) - (REC ? 1 : 0);
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
  double* const bsum = ringC + kRing;                                     // [slot][ΣC, ΣC²][32]
  int* const ringBin = reinterpret_cast<int*>(bsum + 2 * 2 * 32);         // [kRing]
  int* const bcnt = ringBin + kRing;                                      // [slot][32]
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
  // per task slot: task id and trees not yet recorded (kFree: slot unused)
  constexpr int kFree = -(1 << 30);
  int slot_task0 = stream_end ? -1 : iss_task, slot_task1 = -1;
  int slot_left0 = stream_end ? kFree : iss_size, slot_left1 = kFree;
  int ring_cnt = 0;    // pending records (always flushed completely)
  int ring_mask = 0;   // bit s: some pending record belongs to task slot s

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

  // Hand the next trees of the warp's stream to idle lanes (warp-uniform).
  // Lanes only become idle when trees finish, so this runs at start-up and
  // after a tree-completion event.
  auto assign = [&]() {
    unsigned idle = __ballot_sync(0xffffffffu, !active);
    while (idle != 0u && !stream_end) {
      const int avail = iss_size - iss_next;
      if (avail == 0) {
        const int nt = iss_task + W;
        if (nt >= P.n_tasks) { stream_end = true; break; }
        const int ns = iss_slot ^ 1;
        if ((ns == 0 ? slot_left0 : slot_left1) != kFree) break;   // previous task still open
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
  };
  assign();

  while (true) {
    if (stream_end) {                                  // warp-uniform
      if (!__any_sync(0xffffffffu, active)) break;
    }

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
    if constexpr (DIM <= 2) {
      const double v1 = unif53(r1.x, r1.y), v2 = unif53(r1.z, r1.w);
      const double rad = sqrt_nr(-2.0 * log_tab(v1, ltab) * h2d);
      double sn, cs;
      sincospi2(2.0 * v2, sn, cs);
      x[0] = fma(rad, cs, y[0]);
      if constexpr (DIM >= 2) x[1] = fma(rad, sn, y[1]);
    } else {
      // d = 3 from the same two blocks (R8): radii uniforms from
      // block-1 (w1:w0), (w3:w2); angles from 32-bit uniforms — block-0 w3 and
      // the word of the 12 low bits the 53-bit uniforms leave unused
      const double v1 = unif53(r1.x, r1.y), v2 = unif32(r0.w);
      const double v3 = unif53(r1.z, r1.w);
      const uint32_t w4 = ((r0.x & 0xFFFu) << 20) | ((r1.x & 0xFFFu) << 8) | ((r1.z & 0xFFFu) >> 4);
      const double v4 = unif32(w4);
      const double rad = sqrt_nr(-2.0 * log_tab(v1, ltab) * h2d);
      double sn, cs;
      sincospi2(2.0 * v2, sn, cs);
      x[0] = fma(rad, cs, y[0]);
      x[1] = fma(rad, sn, y[1]);
      const double rad2 = sqrt_nr(-2.0 * log_tab(v3, ltab) * h2d);
      x[2] = fma(rad2, cospi2(2.0 * v4), y[2]);
    }
    // categorical offspring choice from the integer thresholds (R9)
    // (thresholds past the support are 0xffffffff, so the sum needs no bound)
    const uint32_t c32 = r0.z;
    int s = (c32 > P.thr[0]) + (c32 > P.thr[1]) + (c32 > P.thr[2]) + (c32 > P.thr[3]);
    if (P.n_support > 5) {                      // warp-uniform, rare
#pragma unroll
      for (int q = 4; q < 8; ++q) s += (c32 > P.thr[q]) ? 1 : 0;
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
    const bool push = branch && k > 1;           // k-1 younger siblings wait
    const bool pop = (active && leaf) || (branch && k == 0);
    const double tc = tau - S;
    const uint64_t base = label << P.beta;
    // push the younger siblings: shared-memory levels inline, the rare deep
    // levels (global) behind a warp-uniform test so they cost nothing otherwise
    const uint64_t push_pk = (base | 1ull) | (static_cast<uint64_t>(k - 1) << 56);
    if (push && sp < LV) {
#pragma unroll
      for (int q = 0; q < DIM; ++q) ssp[(sp * NF + q) * 32] = x[q];
      ssp[(sp * NF + DIM) * 32] = tc;
      ssp[(sp * NF + DIM + 1) * 32] = __longlong_as_double(static_cast<long long>(push_pk));
    }
    if (__any_sync(0xffffffffu, push && sp >= LV)) {
      if (push && sp >= LV) {
        double* b = gsp + (sp - LV) * (NF * 32);
#pragma unroll
        for (int q = 0; q < DIM; ++q) b[q * 32] = x[q];
        b[DIM * 32] = tc;
        b[(DIM + 1) * 32] = __longlong_as_double(static_cast<long long>(push_pk));
      }
    }
    sp += push ? 1 : 0;
    // continue with child 0 (lanes that pop overwrite this below; lanes whose
    // tree ended are re-initialised at assignment)
#pragma unroll
    for (int q = 0; q < DIM; ++q) y[q] = x[q];
    tau = tc;
    label = base;
    const bool done = pruned || kill || (pop && sp == 0);
    const int lvl = sp - 1;
    const bool pop_s = pop && sp > 0 && lvl < LV;
    uint64_t pk = 0;
    if (pop_s) {
#pragma unroll
      for (int q = 0; q < DIM; ++q) y[q] = ssp[(lvl * NF + q) * 32];
      tau = ssp[(lvl * NF + DIM) * 32];
      pk = static_cast<uint64_t>(__double_as_longlong(ssp[(lvl * NF + DIM + 1) * 32]));
    }
    if (__any_sync(0xffffffffu, pop && lvl >= LV)) {
      if (pop && lvl >= LV) {
        const double* b = gsp + (lvl - LV) * (NF * 32);
#pragma unroll
        for (int q = 0; q < DIM; ++q) y[q] = b[q * 32];
        tau = b[DIM * 32];
        pk = static_cast<uint64_t>(__double_as_longlong(b[(DIM + 1) * 32]));
        if ((pk >> 56) != 1ull)
          gsp[((lvl - LV) * NF + DIM + 1) * 32] =
              __longlong_as_double(static_cast<long long>(pk + 1ull - (1ull << 56)));
      }
    }
    if (pop && sp > 0) {
      label = pk & kLabelMask;
      if ((pk >> 56) == 1ull) sp = lvl;         // last sibling: drop the group
      else if (lvl < LV)
        ssp[(lvl * NF + DIM + 1) * 32] =
            __longlong_as_double(static_cast<long long>(pk + 1ull - (1ull << 56)));
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
        const int e = ring_cnt + __popc(fin & lt_mask);
        ringBin[e] = bin | (slot << 5);
        ringC[e] = pruned ? 0.0 : Pi;
        atomicAdd(bcnt + slot * 32 + bin, 1);   // integer: exact in any order
        active = false;
      }
      const int n1 = __popc(fin1), n0 = __popc(fin) - n1;
      ring_cnt += n0 + n1;
      ring_mask |= (n1 ? 2 : 0) | (n0 ? 1 : 0);
      slot_left0 -= n0;
      slot_left1 -= n1;
      __syncwarp();
      const bool cl0 = slot_left0 == 0;
      const bool cl1 = slot_left1 == 0;
      if (cl0 || cl1 || ring_cnt >= 32) {
        // transpose all pending records: lane b accumulates, in ring order, the
        // records of bin b (one slot in the common case, both near task ends)
        if (ring_mask != 3) {
          const int sl = ring_mask >> 1;
          double a1 = bsum[(sl * 2 + 0) * 32 + lane], a2 = bsum[(sl * 2 + 1) * 32 + lane];
          const int code = lane | (sl << 5);
          for (int r = 0; r < ring_cnt; ++r) {
            const int b = ringBin[r];
            const double C = ringC[r];
            if (b == code) {
              a1 += C;
              a2 = fma(C, C, a2);
            }
          }
          bsum[(sl * 2 + 0) * 32 + lane] = a1;
          bsum[(sl * 2 + 1) * 32 + lane] = a2;
        } else {
          double a1 = bsum[lane], a2 = bsum[32 + lane];
          double b1 = bsum[64 + lane], b2 = bsum[96 + lane];
          for (int r = 0; r < ring_cnt; ++r) {
            const int b = ringBin[r];
            const double C = ringC[r];
            if (b == lane) {
              a1 += C;
              a2 = fma(C, C, a2);
            }
            if (b == (lane | 32)) {
              b1 += C;
              b2 = fma(C, C, b2);
            }
          }
          bsum[lane] = a1; bsum[32 + lane] = a2;
          bsum[64 + lane] = b1; bsum[96 + lane] = b2;
        }
        ring_cnt = 0;
        ring_mask = 0;
        __syncwarp();
      }
#pragma unroll
      for (int sl = 0; sl < 2; ++sl) {
        const bool close = sl ? cl1 : cl0;
        if (close) {
          double a1 = bsum[(sl * 2 + 0) * 32 + lane], a2 = bsum[(sl * 2 + 1) * 32 + lane];
          {
            const int task = sl ? slot_task1 : slot_task0;
            if (lane < P.nb) {
              double* o = P.partials + (static_cast<int64_t>(task) * P.nb + lane) * 3;
              o[0] = a1; o[1] = a2; o[2] = static_cast<double>(bcnt[sl * 32 + lane]);
            }
            bcnt[sl * 32 + lane] = 0;
            a1 = 0.0; a2 = 0.0;
            if (sl) { slot_task1 = -1; slot_left1 = kFree; }
            else { slot_task0 = -1; slot_left0 = kFree; }
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
      assign();                                // finished lanes take new trees
    }
  }
  // (trees, pruned trees and splits follow exactly from the bin counts and are
  // added by the task-reduction kernel; every task close folded c_part/c_leaf)
}

}  // namespace rtk
