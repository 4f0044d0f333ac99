// tree_walk.cuh — the random-tree walk kernel (rows a3–a7).
//
// One lane = one tree at a time; one warp = a dynamic stream of tasks (T
// consecutive trees of one node, fetched with one atomicAdd each).  Each loop iteration advances EVERY lane by exactly one particle, so
// the expensive part of an iteration (2 Philox blocks, one log for the clock
// and the Box–Muller radii, sincos, sqrt — PAPER.md:197-204 exponential
// clock, PAPER.md:174-191 Brownian increment) runs with all 32 lanes converged whatever the trees look like;
// the tree logic after it is short predicated straight-line code.  A lane
// whose tree ends takes the next tree of the warp's stream in the same
// iteration (ballot + popc rank), so no lane idles until the stream runs dry.
//
// Depth-first order (child 0 first).  The pending sibling
// groups of all 32 trees of a warp live in ONE per-warp pool of stack
// entries in shared memory (SoA [field][entry]); each lane's stack is a
// linked list through the entries' `prev` index, and entries are handed out
// and returned through a per-warp free list with ballot ranks.  A per-lane
// fixed-depth stack must be sized for each lane's deepest excursion; the
// pool only for the warp's SUM of depths, which is far more concentrated
// (cfg4: mean 58, p99.99 89 entries for 32 lanes, where per-lane stacks of 5
// levels overflowed in 29 % of iterations — DESIGN.md §4).  Should the pool
// run dry, further entries come from a per-warp area in global memory (slow
// path, warp-uniform branch; exercised by the tests through rt_set_pool).
// A group stores the split position y, remaining horizon τ_c and a packed
// (next child label | remaining count << 56).
//
// Order binning: a lane whose tree finishes adds
// C, C² and 1 to ITS OWN accumulators of the tree's order bin, lane-private
// words in global memory ([warp][bin][ΣC, ΣC², n][lane], L2-resident) updated
// with fire-and-forget atomic adds (RED): one writer per word and program
// order, so the sums are deterministic.  When all trees of a task are
// recorded, every lane reads back and clears its words (L2 loads) and the
// warp adds the 32 lanes' sums of each bin in a fixed butterfly order into
// partials[task][bin]; a second kernel sums each node's tasks in a fixed order.
// Each task runs from a clean start (all lanes begin it together), so its
// partials depend on the task alone: results are bitwise reproducible for a
// fixed task size, whatever the grid or warp timing.  With Gaussian data
// (UseRing) the finished trees go through a per-warp record ring first, so
// that the tree's one exponential (Π_l g = amp^L e^{−Σ|x_l|²/s²}) is
// evaluated with all 32 lanes busy: lane i flushes record i into its own
// accumulators, 32 records at a time.
#pragma once
#include <cstdint>
#include <cstdio>
#include <type_traits>

#include "philox.cuh"
#include "rt_math.cuh"

// Debug build (librt_debug.so, -DRT_DEBUG_BOUNDS): device bounds checks on
// every computed index into the stack pool, free lists, overflow area,
// lane-private bin sums, shared-tree slots and partials — the GPU pool offers no compute-sanitizer,
// so the parity tests are re-run against this build (tests/test_gpu_bounds.py).
#if defined(RT_DEBUG_BOUNDS)
#define RT_CHECK(c)                                                              \
  do {                                                                           \
    if (!(c)) {                                                                  \
      printf("RT_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);             \
      __trap();                                                                  \
    }                                                                            \
  } while (0)
#else
#define RT_CHECK(c) do {} while (0)
#endif

namespace rtk {

constexpr int kWarpsPerCta = 4;
constexpr int kThreads = 32 * kWarpsPerCta;
constexpr uint64_t kLabelMask = (1ull << 56) - 1;

// Shared trees with Gaussian data (GK = 2) store per tree, instead of its
// leaf displacements, their mean μ and scatter V = Σ_l |δ_l − μ|² (DIM + 1
// doubles): Π_l amp e^{−|x+δ_l|²/s²} = amp^L e^{−(L|x+μ|² + V)/s²}, one
// exponential per (node, tree) in phase 2.
template <int GK> __host__ __device__ constexpr bool sh_moments() { return GK == 2; }

// Stack-pool entries per warp in shared memory (<= 255: 8-bit free list) and
// resident CTAs per SM.  Sized from the warp's depth-sum distribution (see
// the header) and the 228 KB of shared memory / 64 K registers per SM.  The
// record-emitting trace variant gets one CTA less so it never spills; it is
// launched on the production kernel's grid, so both give identical sums.
// Kernels with the finished-tree record ring (Gaussian data, see DeferG)
// give its 1 KB per warp up from the pool.
// (RT_POOL_D<d> / RT_CTAS_D<d>: compile-time overrides for occupancy sweeps)
#ifndef RT_POOL_D1
#define RT_POOL_D1 182
#endif
#ifndef RT_POOL_D2
#define RT_POOL_D2 168
#endif
#ifndef RT_POOL_D3
#define RT_POOL_D3 138
#endif
#ifndef RT_CTAS_D1
#define RT_CTAS_D1 8
#endif
#ifndef RT_CTAS_D2
#define RT_CTAS_D2 8
#endif
#ifndef RT_CTAS_D3
#define RT_CTAS_D3 8
#endif
constexpr int kRing = 64;   // finished-tree record ring slots per warp (ring kernels)
template <int DIM> struct PoolBase;
template <> struct PoolBase<1> { static constexpr int v = RT_POOL_D1; };
template <> struct PoolBase<2> { static constexpr int v = RT_POOL_D2; };
template <> struct PoolBase<3> { static constexpr int v = RT_POOL_D3; };
// RV = deferred values per ring record beside the tree product (RingVals):
// the ring's kRing × (8 (1 + RV) + 1) bytes come out of the pool's
// (DIM+2)·8 + 3 per entry
template <int RV> __host__ __device__ constexpr int ring_bytes() { return RV > 0 ? kRing * (8 * (1 + RV) + 1) : 0; }
template <int DIM, int RV> struct PoolCap {
  static constexpr int v = PoolBase<DIM>::v - (ring_bytes<RV>() + (DIM + 2) * 8 + 2) / ((DIM + 2) * 8 + 3);
};
template <int DIM, bool REC> struct MinCtas {
  static constexpr int v = (DIM == 1 ? RT_CTAS_D1 : DIM == 2 ? RT_CTAS_D2 : RT_CTAS_D3) - (REC ? 1 : 0);
};

struct TreeRec {   // mirrors rt_tree_rec
  int32_t ne, leaves, particles, pruned;
  double C;
};

// Shared trees (f4): what phase 2 needs of a tree — its order bin (K+1 if
// pruned), leaf count, splits, particles and the node-free weight product W
// (root factor × split weights × Strategy B's 1/q per leaf).
struct TreeSum {
  int32_t bin, nl, ne, parts;
  double W;
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
  int32_t pool_cap;                   // shared-memory pool entries used (<= PoolCap)
  double* partials;     // [n_tasks][nb][3]
  double* gpool;        // [warps][gcap][DIM+2]  overflow stack entries
  double* lacc;         // [warps][nb][3][32] lane-private order-bin sums (ΣC, ΣC², count)
  int32_t* gaux;        // [warps][2][gcap]      overflow prev links, free list
  int32_t gcap;         // overflow entries per warp (32 (K+1): every stack bound)
  TreeRec* recs;
  int32_t rec_shift;
  int64_t n_rec;
  unsigned long long* stats;   // trees, pruned, particles, leaves, splits
  unsigned int* task_ctr;      // dynamic task counter (zeroed before the launch)
  // NEXT rows f2/f3: split-weight factors beyond the constant
  // w_k — bit0 variable coefficients, bit1 Strategy A's e^{(k-1)λτ_c} (0 on
  // the default path: one warp-uniform test per iteration)
  int32_t wmode;
  uint32_t var_s;              // bit s: support entry s has a variable coefficient
  double lam, root;            // λ; per-tree root factor (e^{λt} with the shift, else 1)
  int32_t coef_axis;
  double coef_inv_s2, coef_t0;
  uint32_t tq;                 // Strategy B: leaf iff block-0 word 3 < tq
  double inv_q;                // Strategy B: 1/q̂
  int32_t n_points;            // nodes (shared trees: the stats are per (node, tree))
  // shared trees (f4), phase 1: per-tree summaries and leaf displacements of
  // trees [tree_offset, tree_offset + n_trees): tsum[j], leaves[j][lmax][DIM]
  // (Gaussian g: leaves[j][DIM + 1] = μ, V — see sh_moments)
  struct TreeSum* tsum;
  double* leaves;
  int32_t lmax;
  unsigned long long* wtime;   // debug (RT_WARP_TIMES): [warps][4] start, end, smid, iterations; or null
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Per-warp bookkeeping that only the completion path touches.
struct WarpState {
  double iss_y[3];          // coordinates of the current task's node
  int gtop, gfree;          // overflow area: bump pointer, free-list size
  double* gpool;            // the warp's overflow area (read in the slow paths only,
  int* gprev;               //   so the compiler does not keep or rematerialise them)
  double* lacc[32];         // each lane's accumulator base (its [bin 0][ΣC] word)
};

// The initial data g: constant, tanh step, Gaussian,
// Lorentzian (the BASELINE.json configs' shapes).
template <int DIM, int GK>
__device__ __forceinline__ double g_eval(const double (&x)[DIM], double amp, double inv_scale,
                                         double inv_scale2) {
  if constexpr (GK == 0) {
    return amp;
  } else if constexpr (GK == 1) {
    return amp * 0.5 * (1.0 + tanh(x[0] * inv_scale));
  } else {
    double r2 = x[0] * x[0];
    if constexpr (DIM >= 2) r2 = fma(x[1], x[1], r2);
    if constexpr (DIM >= 3) r2 = fma(x[2], x[2], r2);
    if constexpr (GK == 2) return amp * exp_neg(-r2 * inv_scale2);
    else return amp * rcp_nr(fma(r2, inv_scale2, 1.0));
  }
}

template <int DIM, int GK>
__device__ __forceinline__ double g_eval(const double (&x)[DIM], const WalkParams& P) {   // g(x)
  return g_eval<DIM, GK>(x, P.amp, P.inv_scale, P.inv_scale2);
}

// g in single precision for the FP32-position variant (RT_PREC_FP32_POS):
// MUFU exp2 (__expf) and single-precision reciprocals.
template <int DIM, int GK>
__device__ __forceinline__ float g_eval_f(const float (&x)[DIM], const WalkParams& P) {
  const float amp = static_cast<float>(P.amp);
  if constexpr (GK == 0) {
    return amp;
  } else if constexpr (GK == 1) {
    // 0.5 (1 + tanh z) = 1 / (1 + e^{-2z}): no cancellation for z << 0 in FP32
    return amp * __frcp_rn(1.0f + __expf(-2.0f * x[0] * static_cast<float>(P.inv_scale)));
  } else {
    float r2 = x[0] * x[0];
    if constexpr (DIM >= 2) r2 = fmaf(x[1], x[1], r2);
    if constexpr (DIM >= 3) r2 = fmaf(x[2], x[2], r2);
    const float is2 = static_cast<float>(P.inv_scale2);
    if constexpr (GK == 2) return amp * __expf(-r2 * is2);
    else return amp * __frcp_rn(fmaf(r2, is2, 1.0f));
  }
}

// Deferred factors (independent trees, FP64 positions; the "ring" kernels).
// Exponential and rational factors of a tree's product are carried in closed
// form — an exponent sum X and a denominator product D, C = Π · e^X / D —
// and evaluated once per TREE, when the finished tree's record (order bin,
// Π, X[, D]) is flushed from a per-warp ring of kRing records, 32 at a time,
// one record per lane (every lane busy on it, instead of the evaluation in
// every particle iteration):
//   Gaussian data g = amp e^{-|x|²/s²}: Π_l g(x_l) = amp^L e^{−Σ_l |x_l|²/s²}
//     — a leaf multiplies amp into Π and adds −|x|²/s² to X;
//   (general kernels, NEXT rows f2) Strategy A's shift factor e^{(k−1)λτ_c}
//     per split adds (k−1)λτ_c to X; a variable coefficient
//     b_k e^{−y_a²/s²}/(τ_c + t0) adds −y_a²/s² to X and multiplies τ_c + t0
//     into D.
// Measured: cfg2 +6.4 %, cfg3 +3.6 %; the same ring with the Lorentzian's
// denominator product Π(1 + |x|²/s²) made cfg4 0.9 % slower (its reciprocal
// is cheap, the ring is not free), so other data evaluate g at the leaf.
// RingVals: 0 no ring, 1 Π and X (Gaussian, GEN = false), 2 Π, X and D (GEN).
template <int GK, bool F32, bool SH, bool GEN> __host__ __device__ constexpr int RingVals() {
  return (F32 || SH) ? 0 : (GEN ? 2 : (GK == 2 ? 1 : 0));
}

// per-warp shared memory: pool fields [DIM+2][cap] doubles, (ring: record
// values [1 + RV][kRing] doubles), state, prev [cap] int16, free list [cap]
// u8, (ring: record bins [kRing] u8)
template <int DIM, int RV>
__host__ __device__ constexpr int warp_smem_bytes() {
  return PoolCap<DIM, RV>::v * ((DIM + 2) * 8 + 2 + 1) + ring_bytes<RV>() + static_cast<int>(sizeof(WarpState));
}

template <int DIM, int RV>
__host__ __device__ constexpr int warp_stride() {
  return (warp_smem_bytes<DIM, RV>() + 15) / 16 * 16;
}

template <int DIM, int RV>
__host__ __device__ constexpr int smem_bytes() {
  return 128 * 16 /* log table */ + kWarpsPerCta * warp_stride<DIM, RV>() +
         9 * 8 + 9 * 4 + 4 /* offspring weights and sizes */ + 32 * 8 /* exp table */;
}

// n += 1 if c, as one predicated add (ptxas otherwise emits add + select)
__device__ __forceinline__ void inc_if(bool c, int& n) {
  asm("{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %1, 0;\n\t@p add.s32 %0, %0, 1;\n\t}"
      : "+r"(n) : "r"(static_cast<int>(c)));
}

// Fire-and-forget FP64 add to a global word (RED; the generic atomicAdd on a
// pointer read from shared memory would also test for the shared window)
__device__ __forceinline__ void red_add(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// The same with an L2 eviction-priority hint: the lane-private bin sums
// (65 MB at cfg4) are the kernel's only re-used global data, so they are
// kept resident (evict_last) while the once-written task partials stream
// past them (evict_first), instead of being written back to DRAM.
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void red_add_keep(double* p, double v, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// F32 = the FP32-position / FP64-accumulate variant (cfg5, BASELINE.json
// configs[4]): the clock S, the leaf test, horizons, weights, the tree
// product and all sums stay FP64 (tree structure identical to the FP64
// path); positions, the Brownian increment and g are single precision.
// SB = Strategy B: a particle is a leaf with probability
// q (ξ = 0, weight g/q), else it splits after the uniform fraction S of its
// horizon with weight τ c_k/((1-q) p_k) and its children inherit τ(1-S).
// SH = shared trees (NEXT row f4), phase 1: the random numbers
// omit the node index, so every node sees the same trees; a task is a tree
// range; lanes walk trees carrying the displacement δ from the root and write
// each tree's summary (TreeSum) and leaf displacements; phase 2
// (shared_eval.cuh) evaluates all nodes.  Constant coefficients only.
// GEN = false: the common equations — no f2/f3 weight factors (wmode = 0)
// and one to three offspring kinds — without the warp-uniform tests for the
// rest (the same arithmetic; chosen by the launcher).
template <int DIM, int GK, bool REC, bool F32, bool SB, bool SH, bool GEN = true>
__global__ void __launch_bounds__(kThreads, MinCtas<DIM, REC>::v)
tree_walk_kernel(const __grid_constant__ WalkParams P) {
  using PT = typename std::conditional<F32, float, double>::type;   // position type
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int NF = DIM + 2;
  constexpr int RV = RingVals<GK, F32, SH, GEN>();
  constexpr bool RING = RV > 0;
  constexpr int CAP = PoolCap<DIM, RV>::v;
  // lane, its lower-lanes mask and the warp's shared-memory offset are read
  // through opaque moves, so the compiler keeps them in registers instead of
  // rematerialising them from threadIdx every iteration
  int lane;
  unsigned lt_mask;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane));
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(lt_mask));
  const int wib = threadIdx.x >> 5;

  // ---- shared memory carve-up -------------------------------------------
  LogEntry* const ltab = reinterpret_cast<LogEntry*>(smem_raw);
  const int wstride = warp_stride<DIM, RV>();
  unsigned woff;
  asm volatile("mov.u32 %0, %1;" : "=r"(woff) : "r"(128 * 16 + wib * wstride));
  unsigned char* const wbase = smem_raw + woff;
  double* const pool = reinterpret_cast<double*>(wbase);                   // [NF][CAP]
  double* const rval = pool + NF * CAP;                                    // ring: [kRing] tree products
  double* const rexp = rval + kRing;                                       // ring: [kRing] exponent sums X
  double* const rden = rexp + kRing;                                       // ring (RV = 2): [kRing] denominators D
  WarpState* const ws = reinterpret_cast<WarpState*>(rval + (RING ? kRing * (1 + RV) : 0));
  int16_t* const prevS = reinterpret_cast<int16_t*>(ws + 1);               // [CAP]
  uint8_t* const freeS = reinterpret_cast<uint8_t*>(prevS + CAP);           // [CAP]
  uint8_t* const rbin = freeS + CAP;                                       // ring: [kRing] order bins
  double* const wtab = reinterpret_cast<double*>(smem_raw + 128 * 16 +
      kWarpsPerCta * wstride);                                           // [9] weights
  int* const ktab = reinterpret_cast<int*>(wtab + 9);                     // [9] offspring k
  double* const etab = wtab + 14;                                         // [32] 2^(j/32)
  for (int q = threadIdx.x; q < 128; q += kThreads) ltab[q] = kLogTable[q];
  if constexpr ((GK == 2 && !F32) || RING) {
    if (threadIdx.x < 32) etab[threadIdx.x] = kExpT32[threadIdx.x];
  }
  if (threadIdx.x < 9) {
    wtab[threadIdx.x] = P.w[threadIdx.x];
    ktab[threadIdx.x] = P.kval[threadIdx.x];
  }
  const int cap = P.pool_cap;
  for (int q = lane; q < cap; q += 32) freeS[q] = static_cast<uint8_t>(q);

  const int gwarp = blockIdx.x * kWarpsPerCta + wib;
  if (P.wtime != nullptr && lane == 0) P.wtime[4 * gwarp] = global_ns();
  if (lane == 0) {
    ws->gpool = P.gpool + static_cast<int64_t>(gwarp) * P.gcap * NF;
    ws->gprev = P.gaux + static_cast<int64_t>(gwarp) * 2 * P.gcap;
  }
  ws->lacc[lane] = SH ? nullptr : P.lacc + static_cast<int64_t>(gwarp) * P.nb * 96 + lane;
  __syncwarp();
  // lane-private order-bin accumulators in global memory: [bin][ΣC, ΣC², n][lane]
  // (the lane's base read back from shared memory where used: one 64-bit
  // load and one wide multiply-add per address, no register held)
  auto lacc = [&]() -> double* { return *static_cast<double* volatile*>(&ws->lacc[lane]); };
  if constexpr (!SH) {
    double* a = lacc();
    for (int b = 0; b < P.nb; ++b) { a[b * 96] = 0.0; a[b * 96 + 32] = 0.0; a[b * 96 + 64] = 0.0; }
  }
  // overflow-area bases, re-read from shared memory where used (volatile: no
  // hoisting into the fast path)
  auto gpool = [&]() -> double* { return *static_cast<double* volatile*>(&ws->gpool); };
  auto gprev = [&]() -> int* { return *static_cast<int* volatile*>(&ws->gprev); };
  auto gfl = [&]() -> int* { return gprev() + P.gcap; };

  // ---- warp-uniform stream state -------------------------------------------
  // The warp fetches tasks dynamically (one atomicAdd per task) and runs each
  // task from a clean start: all 32 lanes take the task's first trees
  // together and the task is closed only when its last tree is recorded.  A
  // task's processing — and so its partial sums — is then a function of the
  // task alone, whichever warp runs it and whatever ran before (bitwise
  // deterministic for a fixed task size T, any grid).  Dynamic fetching
  // absorbs the warp scheduler's unequal issue rates.
  uint32_t iss_next = 0u, iss_end = 0u, iss_node = 0u;
  int task = -1, left = 0;             // current task, its trees not yet recorded
  int task_q = 0;                      // the task's tree-range index
  bool stream_end = false;
  auto next_task = [&]() {             // all lanes, converged
    int t = 0;
    if (lane == 0) t = static_cast<int>(atomicAdd(P.task_ctr, 1u));
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= P.n_tasks) { stream_end = true; return; }
    task = t;
    const int node = t / P.tpn;          // SH: always 0 (tasks are tree ranges)
    const int q = t - node * P.tpn;
    const int size = min(P.T, P.n_trees - q * P.T);
    task_q = q;
    iss_node = static_cast<uint32_t>(node);
    iss_next = static_cast<uint32_t>(P.tree_offset) + static_cast<uint32_t>(q * P.T);
    iss_end = iss_next + static_cast<uint32_t>(size);
    left = size;
    __syncwarp();
    if constexpr (SH) {
      // the walk carries δ from the root: no node coordinates
    } else if (lane == 0) {
#pragma unroll
      for (int k = 0; k < DIM; ++k) ws->iss_y[k] = P.points[static_cast<int64_t>(node) * DIM + k];
    }
    __syncwarp();
  };
  int nfree = cap;     // free shared-memory pool entries
  int n_glob = 0;      // overflow entries in use (warp-uniform)

  // ---- lane state ----------------------------------------------------------
  bool active = false;
  uint32_t tj = 0;   // (the node is the task's: warp-uniform iss_node)
  PT y[DIM];
#pragma unroll
  for (int k = 0; k < DIM; ++k) y[k] = PT(0);
  double tau = 0.0, Pi = 1.0;
  double gexp = 0.0, gden = 1.0;       // ring: the tree's deferred exponent X and denominator D (RingVals)
  uint64_t label = 1;
  int ne = 0, top = -1;                // top: the lane's top stack entry (-1: empty)
  int leaves = 0, parts = 0;           // per-tree counts (trace variant only)
  int c_leaf = 0;                      // leaves since the last task close
  double m1[DIM], m2 = 0.0;            // SH, Gaussian g: Σ δ_l and Σ |δ_l|² of the tree's leaves
#pragma unroll
  for (int k = 0; k < DIM; ++k) m1[k] = 0.0;

  auto start_tree = [&](uint32_t j) {  // a fresh tree j of the current task
    tj = j;
#pragma unroll
    for (int k = 0; k < DIM; ++k) y[k] = SH ? PT(0) : static_cast<PT>(ws->iss_y[k]);   // SH: δ = 0
    tau = P.t; label = 1; Pi = GEN ? P.root : 1.0; ne = 0; top = -1;   // (GEN = false: no shift, root factor 1)
    if constexpr (RING) gexp = 0.0;
    if constexpr (RV == 2) gden = 1.0;
    if constexpr (REC || SH) { leaves = 0; parts = 0; }
    if constexpr (SH && sh_moments<GK>()) {
#pragma unroll
      for (int k = 0; k < DIM; ++k) m1[k] = 0.0;
      m2 = 0.0;
    }
    active = true;
  };

  // The tree's contribution C = Π e^X / D from its record (RingVals)
  // (Π e^X with the power of two applied last: no overflow of e^X alone)
  auto tree_c = [&](double pi, double x, double dn) -> double {
    if constexpr (RING) {
      const double a = RV == 2 ? pi * rcp_nr(dn) : pi;
      return mul_exp_tab(a, x, etab);
    } else {
      return pi;
    }
  };
  // Record ring: rn records from slot rhead on (warp-uniform counters).
  // flush(m): lane i < m adds record rhead + i — C, C² and 1 — to ITS OWN
  // accumulators of the record's bin with fire-and-forget REDs (one writer
  // per word, program order: deterministic for a task's fixed record order).
  const uint64_t pol = l2_evict_last_policy();   // (warp-uniform: a uniform register)
  int rhead = 0, rn = 0;
  auto flush = [&](int m) {
    __syncwarp();
    if (lane < m) {
      const int sl = (rhead + lane) & (kRing - 1);
      const int b = rbin[sl];
      RT_CHECK(b >= 0 && b < P.nb);
      const double c = tree_c(rval[sl], rexp[sl], RV == 2 ? rden[sl] : 1.0);
      double* a = lacc() + b * 96;
      red_add_keep(a, c, pol);
      red_add_keep(a + 32, c * c, pol);
      red_add_keep(a + 64, 1.0, pol);
    }
    rhead = (rhead + m) & (kRing - 1);
    rn -= m;
    __syncwarp();
  };

  // All trees of the task are recorded: write its partials (lane b = bin b),
  // fold the event counters, fetch the next task and start its first trees.
  auto close_and_next = [&]() {
    if constexpr (SH) {
      // phase 1 writes tree summaries only (phase 2 accumulates per node)
    } else {
      // each lane reads back (L2: its own atomics) and clears its sums, the
      // warp adds the 32 lanes' in a fixed butterfly order, lane 0 writes
      RT_CHECK(task >= 0 && task < P.n_tasks);
      if constexpr (RING) {
        if (rn > 0) flush(rn);                     // the task's last records
      }
      __threadfence();                             // this lane's REDs are performed before its read-back
      double* a = lacc();
      for (int b = 0; b < P.nb; ++b) {
        double v1 = __ldcg(a + b * 96), v2 = __ldcg(a + b * 96 + 32), v3 = __ldcg(a + b * 96 + 64);
        a[b * 96] = 0.0; a[b * 96 + 32] = 0.0; a[b * 96 + 64] = 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          v1 += __shfl_xor_sync(0xffffffffu, v1, o);
          v2 += __shfl_xor_sync(0xffffffffu, v2, o);
          v3 += __shfl_xor_sync(0xffffffffu, v3, o);
        }
        if (lane == 0) {
          double* o = P.partials + (static_cast<int64_t>(task) * P.nb + b) * 3;
          const bool prb = b == P.K + 1;           // pruned bin: count only
          __stcs(o, prb ? 0.0 : v1); __stcs(o + 1, prb ? 0.0 : v2); __stcs(o + 2, v3);
        }
      }
    }
    // (shared trees: every node sees each walked particle and leaf)
    // (particles = leaves + splits: every processed particle either reaches
    // its horizon or splits — the aborting split included — so the host
    // derives them; splits come exactly from the bin counts)
    const unsigned long long scale = SH ? static_cast<unsigned long long>(P.n_points) : 1ull;
    unsigned long long v1 = static_cast<unsigned long long>(c_leaf) * scale;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    if (lane == 0) atomicAdd(P.stats + 3, v1);
    c_leaf = 0;
    next_task();
    if (!stream_end) {
      const uint32_t take = min(iss_end - iss_next, 32u);
      if (static_cast<uint32_t>(lane) < take) start_tree(iss_next + static_cast<uint32_t>(lane));
      iss_next += take;
    }
  };

  // ---- stack-pool slow path (overflow entries in global memory) -----------
  // entry e < cap lives in shared memory, e >= cap at gpool[e - cap]
  auto fld = [&](int e, int f) -> double* {
    return e < cap ? pool + f * CAP + e : gpool() + static_cast<int64_t>(e - cap) * NF + f;
  };
  auto prev_of = [&](int e) -> int { return e < cap ? static_cast<int>(prevS[e]) : gprev()[e - cap]; };
  // return entry e of every lane with rel set to the free lists
  auto release_generic = [&](bool rel, int e) {
    const unsigned rs = __ballot_sync(0xffffffffu, rel && e < cap);
    const unsigned rg = __ballot_sync(0xffffffffu, rel && e >= cap);
    const int gf = ws->gfree;
    __syncwarp();
    if (rel) RT_CHECK(e >= 0 && e < cap + P.gcap);
    if (rel && e < cap) RT_CHECK(nfree + __popc(rs & lt_mask) < cap);
    if (rel && e >= cap) RT_CHECK(gf + __popc(rg & lt_mask) < P.gcap);
    if (rel && e < cap) freeS[nfree + __popc(rs & lt_mask)] = static_cast<uint8_t>(e);
    if (rel && e >= cap) gfl()[gf + __popc(rg & lt_mask)] = e - cap;
    nfree += __popc(rs);
    n_glob -= __popc(rg);
    if (lane == 0) ws->gfree = gf + __popc(rg);
    __syncwarp();
  };

  if (lane == 0) ws->gtop = ws->gfree = 0;
  __syncthreads();
  next_task();
  if (!stream_end) {
    const uint32_t take = min(iss_end - iss_next, 32u);
    if (static_cast<uint32_t>(lane) < take) start_tree(iss_next + static_cast<uint32_t>(lane));
    iss_next += take;
  }

  while (true) {
    if (stream_end) {                                  // warp-uniform
      if (!__any_sync(0xffffffffu, active)) break;
    }

    // ---------------- one particle per lane (converged) ----------------------
    const uint32_t c2 = static_cast<uint32_t>(label);
    const uint32_t c3 = static_cast<uint32_t>(label >> 32);
    const uint32_t c1 = SH ? 0u : iss_node;     // the task's node (shared trees: none)
    const uint4 r0 = philox4x32_10(tj, c1, c2, c3, P.rk);
    const uint4 r1 = philox4x32_10(tj, c1, c2, c3 | (1u << 24), P.rk);
    bool leaf;
    double tc, h2d;                             // children's horizon, 2D·lifetime
    if constexpr (SB) {
      // ξ = 0 (leaf) iff block-0 word 3 < tq; S ~ U(0,1) the split fraction
      leaf = r0.w < P.tq;
      const double Sf = unif53(r0.x, r0.y);
      h2d = (leaf ? tau : tau * Sf) * P.two_d;
      tc = tau * (1.0 - Sf);
      // Brownian increment: textbook Box–Muller from 53-bit uniforms (R8)
      if constexpr (DIM <= 2) {
        const double v1 = unif53(r1.x, r1.y), v2 = unif53(r1.z, r1.w);
        const double rad = sqrt_pos(-2.0 * log_tab(v1, ltab) * h2d);
        if constexpr (DIM == 1) {
          y[0] = fma(rad, cospi2(2.0 * v2), y[0]);
        } else {
          double sn, cs;
          sincospi2(2.0 * v2, sn, cs);
          y[0] = fma(rad, cs, y[0]);
          y[1] = fma(rad, sn, y[1]);
        }
      } else {                                   // block-0 word 3 is ξ: angles from block 2
        const uint4 r2 = philox4x32_10(tj, c1, c2, c3 | (2u << 24), P.rk);
        const double rad = sqrt_pos(-2.0 * log_tab(unif53(r1.x, r1.y), ltab) * h2d);
        double sn, cs;
        sincos2pi_u32(r2.x, sn, cs);
        y[0] = fma(rad, cs, y[0]);
        y[1] = fma(rad, sn, y[1]);
        const double rad2 = sqrt_pos(-2.0 * log_tab(unif53(r1.z, r1.w), ltab) * h2d);
        y[2] = fma(rad2, cos2pi_u32(r2.y), y[2]);
      }
    } else {
      // The exponential clock and the Box–Muller radii from ONE log (DESIGN.md
      // R29): G = −ln(U_1⋯U_{m+1}) ~ Gamma(m+1), split by the spacings of m
      // sorted uniforms into m+1 iid Exp(1) — e0 the clock's, e1 (and e2 for
      // d = 3) the radii's (r² = 2e).  d ≤ 2: U1, U2, the spacing uniform and
      // the offspring draw from block 0, the angle word from block 1;
      // d = 3: U3, the two spacing uniforms and the second angle from block 1.
      const double u12 = unif32(r0.x) * unif32(r0.y);
      double e0, e1, e2 = 0.0;
      if constexpr (DIM <= 2) {
        const double v = unif32(r0.w);
        const double G = -log_tab(u12, ltab);
        e0 = G * v;
        e1 = G * (1.0 - v);
      } else {
        const double v1 = unif32(min(r1.y, r1.z)), v2 = unif32(max(r1.y, r1.z));
        const double G = -log_tab(u12 * unif32(r1.x), ltab);
        e0 = G * v1;
        e1 = G * (v2 - v1);                     // (0 when the two words tie)
        e2 = G * (1.0 - v2);
      }
      // exponential clock S ~ λ e^{-λS}
      const double S = e0 * P.inv_lambda;
      leaf = S > tau;                           // 1{S > t}
      h2d = (leaf ? tau : S) * P.two_d;         // variance 2D·h of the increment
      tc = tau - S;
      if constexpr (F32) {
        // the same variates in single precision on the MUFU approximations
        // (sin/cos at |x| <= π, sqrt: ~2^-21)
        constexpr float k2Pi = 6.28318530717958648f, kPi = 3.14159265358979324f;
        const float hf = static_cast<float>(h2d);
        const float rad = __fsqrt_rn(2.0f * static_cast<float>(e1) * hf);
        // cos(2πv) = −cos(2πv − π), sin(2πv) = −sin(2πv − π), argument in [−π, π)
        if constexpr (DIM == 1) {
          y[0] = fmaf(-rad, __cosf(fmaf(k2Pi, static_cast<float>(unif32(r1.x)), -kPi)), y[0]);
        } else {
          float sn, cs;
          __sincosf(fmaf(k2Pi, static_cast<float>(unif32(DIM == 2 ? r1.x : r0.w)), -kPi), &sn, &cs);
          y[0] = fmaf(-rad, cs, y[0]);
          y[1] = fmaf(-rad, sn, y[1]);
          if constexpr (DIM == 3) {
            const float rad2 = __fsqrt_rn(2.0f * static_cast<float>(e2) * hf);
            y[2] = fmaf(-rad2, __cosf(fmaf(k2Pi, static_cast<float>(unif32(r1.w)), -kPi)), y[2]);
          }
        }
      } else if constexpr (DIM == 1) {          // the cosine normal only
        y[0] = fma(sqrt_pos(2.0 * e1 * h2d), cos2pi_u32(r1.x), y[0]);
      } else if constexpr (DIM == 2) {
        const double rad = sqrt_pos(2.0 * e1 * h2d);
        double sn, cs;
        sincos2pi_u32(r1.x, sn, cs);
        y[0] = fma(rad, cs, y[0]);
        y[1] = fma(rad, sn, y[1]);
      } else {
        // (e1 = 0 when the two spacing words tie — probability 2^-32: the
        // 2^-996 (≈ 1.5e-300, an FP64 immediate) keeps the root positive and
        // changes nothing else, since it is absorbed by any 2·e1·h2d > 1e-284)
        const double rad = sqrt_pos(fma(2.0 * e1, h2d, 0x1p-996));
        double sn, cs;
        sincos2pi_u32(r0.w, sn, cs);
        y[0] = fma(rad, cs, y[0]);
        y[1] = fma(rad, sn, y[1]);
        y[2] = fma(sqrt_pos(2.0 * e2 * h2d), cos2pi_u32(r1.w), y[2]);
      }
    }
    // categorical offspring choice from the integer thresholds (R9)
    // (thresholds past the support are 0xffffffff, so the sum needs no bound)
    // (the last support entry's threshold is 2^32 - 1: with n entries only
    // n - 1 compares can fire — two for the configs' three-term f)
    const uint32_t c32 = r0.z;
    int s = 0;
    inc_if(c32 > P.thr[0], s);
    inc_if(c32 > P.thr[1], s);
    if (GEN && P.n_support > 3) {               // warp-uniform
      inc_if(c32 > P.thr[2], s);
      inc_if(c32 > P.thr[3], s);
      if (P.n_support > 5) {                    // warp-uniform, rare
#pragma unroll
        for (int q = 4; q < 8; ++q) inc_if(c32 > P.thr[q], s);
      }
    }
    double gv;                                  // g at the leaf
    if constexpr (F32) {
      gv = static_cast<double>(g_eval_f<DIM, GK>(y, P));
    } else if constexpr (RING && GK == 2) {    // Gaussian: exponent deferred to the record (RingVals)
      double r2 = y[0] * y[0];
      if constexpr (DIM >= 2) r2 = fma(y[1], y[1], r2);
      if constexpr (DIM >= 3) r2 = fma(y[2], y[2], r2);
      gv = P.amp;
      const double e = fma(-r2, P.inv_scale2, gexp);
      gexp = leaf ? e : gexp;
    } else if constexpr (GK == 2) {             // Gaussian (shared trees: unused)
      double r2 = y[0] * y[0];
      if constexpr (DIM >= 2) r2 = fma(y[1], y[1], r2);
      if constexpr (DIM >= 3) r2 = fma(y[2], y[2], r2);
      gv = P.amp * exp_neg_tab(-r2 * P.inv_scale2, etab);
    } else {
      gv = g_eval<DIM, GK>(y, P);
    }
    const int k = ktab[s];
    double wk = wtab[s];
    if constexpr (SB) wk *= tau;                // η(τ) = τ
    if (RV == 2 && P.wmode != 0) {              // warp-uniform: f2/f3 weight factors, deferred
      // into the tree's X and D (RingVals): the same factors, evaluated once per tree
      double x = 0.0, dn = 1.0;
      if ((P.var_s >> s) & 1u) {                // c_k(y, τ_c) = b_k e^{-y_a²/s²}/(τ_c + t0)
        double ya = static_cast<double>(y[0]);   // (no dynamic register indexing)
        if constexpr (DIM >= 2) if (P.coef_axis == 1) ya = static_cast<double>(y[1]);
        if constexpr (DIM >= 3) if (P.coef_axis == 2) ya = static_cast<double>(y[2]);
        x = -(ya * ya) * P.coef_inv_s2;
        dn = tc + P.coef_t0;
      }
      if (P.wmode & 2) x = fma(static_cast<double>(k - 1) * P.lam, tc, x);   // e^{(k-1)λτ_c}
      gexp = leaf ? gexp : gexp + x;
      gden = leaf ? gden : gden * dn;
    } else if (GEN && P.wmode != 0) {           // warp-uniform: f2/f3 weight factors
      double f = 1.0;
      if ((P.var_s >> s) & 1u) {                // c_k(y, τ_c) = b_k e^{-y_a²/s²}/(τ_c + t0)
        double ya = static_cast<double>(y[0]);   // (no dynamic register indexing)
        if constexpr (DIM >= 2) if (P.coef_axis == 1) ya = static_cast<double>(y[1]);
        if constexpr (DIM >= 3) if (P.coef_axis == 2) ya = static_cast<double>(y[2]);
        f = exp_neg(-(ya * ya) * P.coef_inv_s2) * rcp_nr(tc + P.coef_t0);
      }
      if (P.wmode & 2) {                        // e^{(k-1)λτ_c}
        const double a = static_cast<double>(k - 1) * P.lam * tc;
        f *= a >= 0.0 ? rcp_nr(exp_neg(-a)) : exp_neg(a);
      }
      wk *= f;
    }

    // ---------------- tree logic: predicated straight-line code ---------------
    const bool split = active && !leaf;
    inc_if(!leaf, ne);                           // splitting events (an idle lane's ne is unused)
    const bool pruned = split && ne > P.K;       // prune
    // a pruned tree (ne = K+1, the pruned bin) and a killed one (purely linear
    // f: no offspring, bin ne) both end here with a zero product
    const bool dead = split && (ne > P.K || (GEN && P.n_support == 0));   // (GEN = false: support non-empty)
    const bool branch = split && !dead;
    // g at a leaf; h^(α) = c'_α at a split
    // SH: g is applied per node in phase 2 (Gaussian: its amplitude here)
    const double gl = SH ? (sh_moments<GK>() ? P.amp : 1.0) : gv;
    // (a killed tree's wk is 0 — entry 0 of an empty support; a pruned tree
    // keeps a nonzero product, routed to the pruned bin whose sums are
    // discarded at task close)
    const double fac = leaf ? (SB ? gl * P.inv_q : gl) : wk;
    Pi *= fac;                                   // (an idle lane's product is never recorded)
    inc_if(active && leaf, c_leaf);
    if constexpr (REC || SH) {
      inc_if(active, parts);
      if constexpr (!SH) inc_if(active && leaf, leaves);   // SH counts at the store below
    }
    const bool push = branch && k > 1;           // k-1 younger siblings wait
    const bool pop = (active && leaf) || (branch && k == 0);
    const bool has = pop && top >= 0;            // resume the top group's next child
    const bool done = dead || (pop && top < 0);
    // child 0 continues from the split point y with horizon τ_c (popping
    // lanes overwrite y, τ, label below; finished lanes are re-initialised)
    tau = tc;
    const uint64_t base = label << P.beta;
    const uint64_t push_pk = (base | 1ull) | (static_cast<uint64_t>(k - 1) << 56);
    label = base;

    // ---------------- shared trees, phase 1: store the leaf displacement -------
    // (before the pops overwrite y): leaves[j][l] = δ of the tree's l-th leaf
    if constexpr (SH) {
      if (active && leaf) {
        if constexpr (sh_moments<GK>()) {
          double r2 = 0.0;
#pragma unroll
          for (int k = 0; k < DIM; ++k) {
            const double yk = static_cast<double>(y[k]);
            m1[k] += yk;
            r2 = fma(yk, yk, r2);
          }
          m2 += r2;
        } else {
          RT_CHECK(leaves < P.lmax && tj - static_cast<uint32_t>(P.tree_offset) < static_cast<uint32_t>(P.n_trees));
          double* const o = P.leaves + (static_cast<int64_t>(tj - static_cast<uint32_t>(P.tree_offset)) *
                                            P.lmax + leaves) * DIM;
#pragma unroll
          for (int k = 0; k < DIM; ++k) o[k] = static_cast<double>(y[k]);
        }
        ++leaves;
      }
    }

    // ---------------- stack: push / pop / release -----------------------------
    // pushes first (they read y before pops overwrite it); entries released in
    // this iteration are reused from the next one
    const unsigned alc = __ballot_sync(0xffffffffu, push);
    const int nalc = __popc(alc);
    if (n_glob == 0 && nalc <= nfree) {          // warp-uniform fast path
      if (push) {
        RT_CHECK(nfree - 1 - __popc(alc & lt_mask) >= 0);
        const int e = freeS[nfree - 1 - __popc(alc & lt_mask)];
        RT_CHECK(e >= 0 && e < cap);
#pragma unroll
        for (int q = 0; q < DIM; ++q) pool[q * CAP + e] = static_cast<double>(y[q]);
        pool[DIM * CAP + e] = tau;
        pool[(DIM + 1) * CAP + e] = __longlong_as_double(static_cast<long long>(push_pk));
        prevS[e] = static_cast<int16_t>(top);
        top = e;
      }
      nfree -= nalc;
      bool last = false;
      if (has) {
#pragma unroll
        RT_CHECK(top >= 0 && top < cap);
        for (int q = 0; q < DIM; ++q) y[q] = static_cast<PT>(pool[q * CAP + top]);
        tau = pool[DIM * CAP + top];
        const uint64_t pk = static_cast<uint64_t>(__double_as_longlong(pool[(DIM + 1) * CAP + top]));
        label = pk & kLabelMask;
        last = (pk >> 56) == 1ull;
        if (!last)
          pool[(DIM + 1) * CAP + top] = __longlong_as_double(static_cast<long long>(pk + 1ull - (1ull << 56)));
      }
      const bool rel = has && last;              // group exhausted: free its entry
      const unsigned rl = __ballot_sync(0xffffffffu, rel);
      __syncwarp();
      if (rel) {
        RT_CHECK(nfree + __popc(rl & lt_mask) < cap);
        freeS[nfree + __popc(rl & lt_mask)] = static_cast<uint8_t>(top);
        top = prevS[top];
      }
      nfree += __popc(rl);
    } else {                                     // generic path (overflow in use)
      // allocate: shared entries first, then overflow entries
      const int rk = __popc(alc & lt_mask);
      const int gf = ws->gfree, gt = ws->gtop;
      __syncwarp();
      if (push) {
        int e;
        if (rk < nfree) {
          e = freeS[nfree - 1 - rk];
        } else {
          const int g = rk - nfree;             // g-th overflow entry of this round
          e = cap + (g < gf ? gfl()[gf - 1 - g] : gt + (g - gf));
          RT_CHECK(e - cap < P.gcap);
        }
#pragma unroll
        for (int q = 0; q < DIM; ++q) *fld(e, q) = static_cast<double>(y[q]);
        *fld(e, DIM) = tau;
        *fld(e, DIM + 1) = __longlong_as_double(static_cast<long long>(push_pk));
        if (e < cap) prevS[e] = static_cast<int16_t>(top);
        else gprev()[e - cap] = top;
        top = e;
      }
      const int ng = max(0, nalc - nfree);
      nfree = max(0, nfree - nalc);
      if (lane == 0) {
        const int from_list = min(ng, gf);
        ws->gfree = gf - from_list;
        ws->gtop = gt + (ng - from_list);
      }
      n_glob += ng;
      __syncwarp();
      bool last = false;
      if (has) {
#pragma unroll
        for (int q = 0; q < DIM; ++q) y[q] = static_cast<PT>(*fld(top, q));
        tau = *fld(top, DIM);
        double* const pkp = fld(top, DIM + 1);
        const uint64_t pk = static_cast<uint64_t>(__double_as_longlong(*pkp));
        label = pk & kLabelMask;
        last = (pk >> 56) == 1ull;
        if (!last) *pkp = __longlong_as_double(static_cast<long long>(pk + 1ull - (1ull << 56)));
      }
      const bool rel = has && last;
      const int freed = top;
      if (rel) top = prev_of(top);
      release_generic(rel, freed);
    }

    if constexpr (REC && !SH) {
      const uint32_t rel = tj - static_cast<uint32_t>(P.tree_offset);
      if (done && (rel & ((1u << P.rec_shift) - 1u)) == 0u) {
        TreeRec r;
        r.ne = ne; r.leaves = leaves; r.particles = parts; r.pruned = pruned ? 1 : 0;
        r.C = pruned ? 0.0 : tree_c(Pi, gexp, gden);
        P.recs[static_cast<int64_t>(iss_node) * P.n_rec + (rel >> P.rec_shift)] = r;
      }
    }

    // ---------------- record finished trees; assign new ones -----------------
    const unsigned fin = __ballot_sync(0xffffffffu, done);
    if (fin != 0u) {
      // a pruned tree aborts with groups still pending: return its entries
      bool drain = done && top >= 0;
      if (n_glob == 0) {                         // warp-uniform: shared entries only
        while (__any_sync(0xffffffffu, drain)) {
          const unsigned rs = __ballot_sync(0xffffffffu, drain);
          if (drain) {
            RT_CHECK(top >= 0 && top < cap && nfree + __popc(rs & lt_mask) < cap);
            freeS[nfree + __popc(rs & lt_mask)] = static_cast<uint8_t>(top);
            top = prevS[top];
          }
          nfree += __popc(rs);
          drain = drain && top >= 0;
        }
        __syncwarp();
      } else {
        while (__any_sync(0xffffffffu, drain)) {
          const int e = top;
          if (drain) top = prev_of(top);
          release_generic(drain, e);
          drain = drain && top >= 0;
        }
      }
      const int nfin = __popc(fin);
      const int rank = __popc(fin & lt_mask);
      if constexpr (SH) {
        // phase 1: the finished tree's summary (phase 2 evaluates the nodes)
        if (done) {
          TreeSum ts;
          ts.bin = pruned ? (P.K + 1) : ne;
          ts.nl = leaves; ts.ne = ne; ts.parts = parts;
          ts.W = pruned ? 0.0 : Pi;
          RT_CHECK(tj - static_cast<uint32_t>(P.tree_offset) < static_cast<uint32_t>(P.n_trees));
          P.tsum[tj - static_cast<uint32_t>(P.tree_offset)] = ts;
          if constexpr (sh_moments<GK>()) {
            // μ = Σδ/L, V = Σ|δ|² − Σδ·μ (≥ 0; its rounding is O(ε Σ|δ|²),
            // node-free — no cancellation against the node position)
            double* const o = P.leaves + static_cast<int64_t>(tj - static_cast<uint32_t>(P.tree_offset)) * (DIM + 1);
            const double il = leaves > 0 ? 1.0 / static_cast<double>(leaves) : 0.0;
            double v = m2;
#pragma unroll
            for (int k = 0; k < DIM; ++k) {
              const double mu = m1[k] * il;
              o[k] = mu;
              v = fma(-m1[k], mu, v);
            }
            o[DIM] = fmax(v, 0.0);
          }
        }
      } else {
        if constexpr (RING) {
          // record into the ring in lane-rank order: bin ne (= K+1, the
          // pruned bin, iff pruned), product, exponent sum; flush full groups
          if (done) {
            RT_CHECK(ne >= 0 && ne < P.nb && rn + nfin <= kRing);
            const int sl = (rhead + rn + rank) & (kRing - 1);
            rbin[sl] = static_cast<uint8_t>(ne);
            rval[sl] = Pi;
            rexp[sl] = gexp;
            if constexpr (RV == 2) rden[sl] = gden;
          }
          rn += nfin;
          if (rn >= 32) flush(32);
        } else if (done) {                          // bin ne (= K+1, the pruned bin, iff pruned)
          RT_CHECK(ne >= 0 && ne < P.nb);
          double* a = lacc() + ne * 96;
          red_add_keep(a, Pi, pol);
          red_add_keep(a + 32, Pi * Pi, pol);
          red_add_keep(a + 64, 1.0, pol);
        }
      }
      left -= nfin;
      const uint32_t avail = iss_end - iss_next;
      if (avail >= static_cast<uint32_t>(nfin)) {          // common: more trees of the task
        __syncwarp();
        if (done) start_tree(iss_next + static_cast<uint32_t>(rank));
        iss_next += static_cast<uint32_t>(nfin);
      } else if constexpr (SH) {
        // shared trees: a task carries no sums of its own (phase 1 stores
        // per-tree summaries), so lanes need no clean start — the lanes the
        // task cannot serve take the next task's trees at once instead of
        // idling until the task's longest tree ends
        __syncwarp();
        if (done && static_cast<uint32_t>(rank) < avail) start_tree(iss_next + static_cast<uint32_t>(rank));
        iss_next += avail;
        const uint32_t need = static_cast<uint32_t>(nfin) - avail;
        next_task();                                       // (warp-uniform)
        const uint32_t got = stream_end ? 0u : min(need, iss_end - iss_next);
        if (done && static_cast<uint32_t>(rank) >= avail) {
          const uint32_t r2 = static_cast<uint32_t>(rank) - avail;
          if (r2 < got) start_tree(iss_next + r2);
          else active = false;
        }
        iss_next += got;
      } else {                                             // the task's trees run out
        __syncwarp();
        if (done) {
          if (static_cast<uint32_t>(rank) < avail) start_tree(iss_next + static_cast<uint32_t>(rank));
          else active = false;
        }
        iss_next += avail;
        if (left == 0) close_and_next();                   // every tree recorded
      }
    }
  }
  if constexpr (SH) {                 // (streamed tasks: the leaf count is folded once)
    unsigned long long v1 = static_cast<unsigned long long>(c_leaf) * static_cast<unsigned long long>(P.n_points);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    if (lane == 0) atomicAdd(P.stats + 3, v1);
  }
  if (P.wtime != nullptr && lane == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    P.wtime[4 * gwarp + 1] = global_ns();
    P.wtime[4 * gwarp + 2] = smid;
    P.wtime[4 * gwarp + 3] = 0;   // (iteration count: not recorded)
  }
  // (trees, pruned trees and splits follow exactly from the bin counts and are
  // added by the task-reduction kernel; every task close folded c_leaf)
}

}  // namespace rtk
