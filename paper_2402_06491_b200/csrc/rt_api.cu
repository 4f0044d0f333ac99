// rt_api.cu — C ABI (include/rt.h) of the B200 random-tree Monte Carlo
// library: argument validation, equation normalisation (row a1), device
// scratch management, and the launches of the tree-walk, order-bin
// reduction, finalisation and batched Padé kernels (rows a3–a9).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/rt.h"
#include "philox.cuh"
#include "tree_walk.cuh"
#include "pdd.cuh"
#include "shared_eval.cuh"
#include "pade.cuh"

using rtk::WalkParams;

// ---------------------------------------------------------------------------
// errors
static thread_local std::string g_err;

static rt_status fail(rt_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define RT_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(e_ == cudaErrorMemoryAllocation ? RT_E_NOMEM : RT_E_CUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                  \
  } while (0)

extern "C" const char* rt_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------------------
// handle
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) cap = bytes;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct Norm {
  double lambda, inv_lambda, sigma;
  double a[9];
  int n_support;
  int support[9];
  uint64_t thresh[9];
  double w[9];
  int beta;
  uint32_t tq;     // Strategy B: leaf iff the 32-bit draw < tq (q̂ = tq / 2^32)
  double q_hat;
};

struct rt_handle {
  rt_eq_params p;
  Norm nz;
  cudaStream_t own_stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaStream_t last_stream = nullptr;
  bool have_timing = false;
  bool scratch_used = false;   // ev[2] marks the last use of the scratch on last_stream
  double host_total_ms = -1.0;
  DevBuf partials, segs, gpool, gaux, lacc, wtime, sh_tsum, sh_leaves, sh_sorted, sh_boff, pdd_pts, pdd_nodal, pdd_bc, pdd_field, pdd_c, pdd_u, pdd_spl, sums, stats, h_points, h_coeffs, h_stderr, h_aux, h_flags;
  int32_t grid_override = 0;
  int64_t tpt_override = 0;
  int32_t pool_override = 0;
  bool pdd_cluster = true;   // RT_PDD_CLUSTER=0: the single-CTA local solver (A/B tests)
  bool force_gen = false;    // RT_FORCE_GEN=1: the general tree-walk kernel everywhere (tests)
};

// ---------------------------------------------------------------------------
// row a1: normalisation.  f(u) = Σ b_k u^k = −λu + Σ a_k u^k with
// a_k = b_k + λ[k=1]; offspring k with probability p_k and
// weight a_k/(λ p̂_k); integer thresholds T_k =
// nearbyint(cum_k · 2^32), last = 2^32, p̂_k = (T_k − T_{k−1})/2^32
// (R2, R9).  λ default: −b_1 if b_1 < 0 else 1 (R3).
static rt_status normalize(const rt_eq_params& p, Norm& o) {
  std::memset(&o, 0, sizeof(o));
  const bool pot = p.strategy == RT_STRATEGY_POTENTIAL;
  double lam = p.lambda;
  // potential form: λ = −b_1 if b_1 < 0 else 1 (R3); the shift
  // u = v e^{t} of Strategy A uses rate 1 unless overridden
  if (!(lam > 0.0)) lam = (pot && p.b[1] < 0.0) ? -p.b[1] : 1.0;
  o.lambda = lam;
  o.inv_lambda = 1.0 / lam;
  o.sigma = std::sqrt(2.0 * p.D);
  int kmax = 0, ns = 0;
  for (int k = 0; k <= 8; ++k) {
    double a = (k <= p.degree) ? p.b[k] : 0.0;
    if (k == 1 && pot) a += lam;      // only the potential form moves −λu out of f
    o.a[k] = a;
    if (a != 0.0) {
      o.support[ns++] = k;
      kmax = k;
    }
  }
  o.n_support = ns;
  int beta = 1;
  while ((1 << beta) < kmax) ++beta;
  o.beta = beta;
  if (p.strategy == RT_STRATEGY_B) {
    const double tq = std::nearbyint(p.q * 4294967296.0);
    if (!(tq >= 1.0 && tq < 4294967296.0))
      return fail(RT_E_ARG, "Strategy B needs 0 < q < 1 with a nonzero 32-bit threshold");
    o.tq = static_cast<uint32_t>(tq);
    o.q_hat = tq / 4294967296.0;
  }
  if (ns == 0) return RT_OK;
  double prob[9];
  if (p.offspring == RT_OFFSPRING_UNIFORM) {
    for (int s = 0; s < ns; ++s) prob[s] = 1.0 / static_cast<double>(ns);
  } else {
    double tot = 0.0;
    for (int s = 0; s < ns; ++s) tot += std::fabs(o.a[o.support[s]]);
    for (int s = 0; s < ns; ++s) prob[s] = std::fabs(o.a[o.support[s]]) / tot;
  }
  const uint64_t two32 = 4294967296ull;
  double cum = 0.0;
  uint64_t prev = 0;
  for (int s = 0; s < ns; ++s) {
    cum += prob[s];
    uint64_t T = static_cast<uint64_t>(std::nearbyint(cum * 4294967296.0));
    if (T > two32 || s == ns - 1) T = two32;
    if (T <= prev)
      return fail(RT_E_ARG, "offspring k=%d has zero integer probability width", o.support[s]);
    o.thresh[s] = T;
    const double phat = static_cast<double>(T - prev) / 4294967296.0;
    // c'_α = c_α/p_α; Strategy B: c̃ = c/(1 − q)
    o.w[s] = o.a[o.support[s]] /
             ((p.strategy == RT_STRATEGY_B ? (1.0 - o.q_hat) : lam) * phat);
    prev = T;
  }
  return RT_OK;
}

static bool is_fin(double v) { return std::isfinite(v); }

extern "C" rt_status rt_create(const rt_eq_params* params, rt_handle** out) {
  if (!params || !out) return fail(RT_E_ARG, "null pointer");
  const rt_eq_params& p = *params;
  if (p.dim < 1 || p.dim > 3) return fail(RT_E_ARG, "dim must be 1, 2 or 3 (got %d)", p.dim);
  if (!(p.D > 0.0) || !is_fin(p.D)) return fail(RT_E_ARG, "D must be finite and > 0");
  if (p.degree < 0 || p.degree > 8) return fail(RT_E_ARG, "degree must be in [0, 8]");
  for (int k = 0; k <= p.degree; ++k)
    if (!is_fin(p.b[k])) return fail(RT_E_ARG, "b[%d] is not finite", k);
  if (!is_fin(p.lambda)) return fail(RT_E_ARG, "lambda is not finite");
  if (p.offspring != RT_OFFSPRING_ABS && p.offspring != RT_OFFSPRING_UNIFORM)
    return fail(RT_E_ARG, "unknown offspring rule %d", p.offspring);
  if (p.init_kind < RT_G_CONST || p.init_kind > RT_G_LORENTZ)
    return fail(RT_E_ARG, "unknown init_kind %d", p.init_kind);
  if (!is_fin(p.init_amp)) return fail(RT_E_ARG, "init_amp is not finite");
  if (!(p.init_scale > 0.0) || !is_fin(p.init_scale))
    return fail(RT_E_ARG, "init_scale must be finite and > 0");
  if (p.K < 0 || p.K > 30) return fail(RT_E_ARG, "K must be in [0, 30] (got %d)", p.K);
  if (p.precision != RT_PREC_FP64 && p.precision != RT_PREC_FP32_POS)
    return fail(RT_E_ARG, "unknown precision %d", p.precision);
  if (p.strategy < RT_STRATEGY_POTENTIAL || p.strategy > RT_STRATEGY_B)
    return fail(RT_E_ARG, "unknown strategy %d", p.strategy);
  if (p.precision == RT_PREC_FP32_POS && p.strategy != RT_STRATEGY_POTENTIAL)
    return fail(RT_E_ARG, "the FP32-position variant exists for RT_STRATEGY_POTENTIAL only");
  if (p.shared != 0 && p.shared != 1) return fail(RT_E_ARG, "shared must be 0 or 1");
  if (p.shared && p.precision != RT_PREC_FP64)
    return fail(RT_E_ARG, "shared trees are implemented in FP64 only");
  bool any_var = false;
  for (int k = 0; k <= 8; ++k) {
    if (p.coef_kind[k] != RT_COEF_CONST && p.coef_kind[k] != RT_COEF_GAUSS_RATIONAL)
      return fail(RT_E_ARG, "unknown coef_kind[%d] = %d", k, p.coef_kind[k]);
    any_var = any_var || p.coef_kind[k] == RT_COEF_GAUSS_RATIONAL;
  }
  if (any_var) {
    if (p.shared) return fail(RT_E_ARG, "shared trees need constant coefficients");
    if (p.strategy == RT_STRATEGY_POTENTIAL && p.coef_kind[1] != RT_COEF_CONST)
      return fail(RT_E_ARG, "a variable coefficient on k = 1 needs a strategy without the potential");
    if (!(p.coef_scale > 0.0) || !is_fin(p.coef_scale) || !(p.coef_t0 > 0.0) ||
        !is_fin(p.coef_t0) || p.coef_axis < 0 || p.coef_axis >= p.dim)
      return fail(RT_E_ARG, "variable coefficient needs scale > 0, t0 > 0, 0 <= axis < dim");
  }
  Norm nz;
  rt_status s = normalize(p, nz);
  if (s != RT_OK) return s;
  if (1 + p.K * nz.beta > 56)
    return fail(RT_E_ARG, "label width 1 + K*beta = %d exceeds 56 bits", 1 + p.K * nz.beta);
  rt_handle* h = new rt_handle();
  h->p = p;
  if (const char* e = std::getenv("RT_PDD_CLUSTER")) h->pdd_cluster = std::atoi(e) != 0;
  if (const char* e = std::getenv("RT_FORCE_GEN")) h->force_gen = std::atoi(e) != 0;
  h->nz = nz;
  cudaError_t e = cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking);
  for (int q = 0; q < 4 && e == cudaSuccess; ++q) e = cudaEventCreate(&h->ev[q]);
  if (e == cudaSuccess) e = h->stats.ensure(8 * sizeof(unsigned long long));
  if (e != cudaSuccess) {
    rt_destroy(h);
    return fail(RT_E_CUDA, "rt_create: %s", cudaGetErrorString(e));
  }
  *out = h;
  return RT_OK;
}

extern "C" rt_status rt_destroy(rt_handle* h) {
  if (!h) return RT_OK;
  if (h->own_stream) cudaStreamSynchronize(h->own_stream);
  if (h->last_stream) cudaStreamSynchronize(h->last_stream);
  for (DevBuf* b : {&h->partials, &h->segs, &h->gpool, &h->gaux, &h->lacc, &h->wtime, &h->sh_tsum, &h->sh_leaves, &h->sh_sorted, &h->sh_boff, &h->pdd_pts, &h->pdd_nodal,
                    &h->pdd_bc, &h->pdd_field, &h->pdd_c, &h->pdd_u, &h->pdd_spl, &h->sums, &h->stats, &h->h_points, &h->h_coeffs,
                    &h->h_stderr, &h->h_aux, &h->h_flags})
    b->release();
  for (int q = 0; q < 4; ++q)
    if (h->ev[q]) cudaEventDestroy(h->ev[q]);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
  return RT_OK;
}

extern "C" rt_status rt_set_launch(rt_handle* h, int32_t grid_ctas, int64_t trees_per_task) {
  if (!h) return fail(RT_E_ARG, "null handle");
  if (grid_ctas < 0 || trees_per_task < 0) return fail(RT_E_ARG, "negative launch override");
  h->grid_override = grid_ctas;
  h->tpt_override = trees_per_task;
  return RT_OK;
}

extern "C" rt_status rt_set_pool(rt_handle* h, int32_t pool_entries) {
  if (!h) return fail(RT_E_ARG, "null handle");
  if (pool_entries < 0) return fail(RT_E_ARG, "negative pool size");
  h->pool_override = pool_entries;
  return RT_OK;
}

// ---------------------------------------------------------------------------
// tree-walk launch (rows a3–a7)
using KernelFn = void (*)(WalkParams);

template <int DIM, int GK, bool REC, bool F32, bool SB, bool SH = false, bool GEN = true>
static KernelFn pick_kernel() {
  return rtk::tree_walk_kernel<DIM, GK, REC, F32, SB, SH, GEN>;
}

// The production (rec = false) kernel of one instantiation and, for rec,
// its record-emitting twin (launched on the production kernel's geometry),
// with the shared memory and stack-pool size of that instantiation's layout
// (rtk::RingVals decides whether it carries the finished-tree record ring).
template <int D, int G, bool F32, bool SB, bool SH, bool GEN>
static KernelFn pick(bool rec, KernelFn* prod, int* smem, int* pool_cap) {
  constexpr int rv = rtk::RingVals<G, F32, SH, GEN>();
  *smem = rtk::smem_bytes<D, rv>();
  *pool_cap = rtk::PoolCap<D, rv>::v;
  *prod = pick_kernel<D, G, false, F32, SB, SH, GEN>();
  return rec ? pick_kernel<D, G, true, F32, SB, SH, GEN>() : *prod;
}

// The kernel for (dim, g, rec, variant) and the production kernel whose
// occupancy fixes the launch geometry for both.
static KernelFn kernel_for(int dim, int gk, bool rec, bool f32, bool sb, bool sh, bool gen,
                           KernelFn* prod, int* smem, int* pool_cap) {
#define RT_K(D, G)                                                                      \
  if (dim == D && gk == G) {                                                            \
    if (sh && sb) return pick<D, G, false, true, true, true>(rec, prod, smem, pool_cap);   \
    if (sh) return pick<D, G, false, false, true, true>(rec, prod, smem, pool_cap);        \
    if (sb && !gen) return pick<D, G, false, true, false, false>(rec, prod, smem, pool_cap); \
    if (sb) return pick<D, G, false, true, false, true>(rec, prod, smem, pool_cap);        \
    if (f32 && !gen) return pick<D, G, true, false, false, false>(rec, prod, smem, pool_cap); \
    if (f32) return pick<D, G, true, false, false, true>(rec, prod, smem, pool_cap);       \
    if (!gen) return pick<D, G, false, false, false, false>(rec, prod, smem, pool_cap);    \
    return pick<D, G, false, false, false, true>(rec, prod, smem, pool_cap);               \
  }
  RT_K(1, 0) RT_K(1, 1) RT_K(1, 2) RT_K(1, 3)
  RT_K(2, 0) RT_K(2, 1) RT_K(2, 2) RT_K(2, 3)
  RT_K(3, 0) RT_K(3, 1) RT_K(3, 2) RT_K(3, 3)
#undef RT_K
  return nullptr;
}

struct Launch {
  int grid;
  int64_t T, tpn, n_tasks;
};

// Expected particles per tree of the equation at horizon t — used ONLY to
// size tasks (a function of the workload, never of the GPU).  Exponential
// clock at rate λ, offspring k with probability p̂_k, mean m̄ = Σ k p̂_k: the
// branching process has E[leaves](t) = e^{λ(m̄−1)t} and E[splits] =
// (E[leaves] − 1)/(m̄ − 1) (λt at m̄ = 1); Strategy B (leaf with probability
// q) has E[particles] = 1/(1 − (1−q) m̄).  Pruning at K caps it near
// 1 + K·k_max.
static double expected_particles(const rt_handle* h, double t) {
  const Norm& nz = h->nz;
  const rt_eq_params& p = h->p;
  if (nz.n_support == 0) return 1.5;
  double m = 0.0;
  int kmax = 0;
  uint64_t prev = 0;
  for (int s = 0; s < nz.n_support; ++s) {
    m += nz.support[s] * (static_cast<double>(nz.thresh[s] - prev) / 4294967296.0);
    prev = nz.thresh[s];
    kmax = std::max(kmax, nz.support[s]);
  }
  const double cap = 1.0 + static_cast<double>(p.K) * std::max(1, kmax);
  double e;
  if (p.strategy == RT_STRATEGY_B) {
    const double r = (1.0 - nz.q_hat) * m;
    e = r < 1.0 ? 1.0 / (1.0 - r) : cap;
  } else if (std::fabs(m - 1.0) < 1e-9) {
    e = 1.0 + nz.lambda * t;
  } else {
    const double leaves = std::exp(std::min(50.0, nz.lambda * (m - 1.0) * t));
    e = leaves + (leaves - 1.0) / (m - 1.0);
  }
  return std::max(1.0, std::min(e, cap));
}

static rt_status plan_launch(rt_handle* h, KernelFn fn, int smem, int64_t n_points,
                             int64_t n_trees, double t, Launch& L) {
  int dev = 0, nsm = 0, per_sm = 0;
  RT_CUDA(cudaGetDevice(&dev));
  RT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  RT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)fn, rtk::kThreads,
                                                        smem));
  if (per_sm < 1) return fail(RT_E_CUDA, "tree_walk kernel cannot be resident");
  int grid = nsm * per_sm;
  if (h->grid_override > 0) grid = h->grid_override;
  const int64_t total = n_points * n_trees;
  int64_t T = h->tpt_override;
  if (T <= 0) {
    // Warps fetch tasks dynamically and run each from a clean start, so a
    // task's sums depend on T alone; T is a function of the workload only
    // (not of the grid) so results are bitwise identical on any GPU size.
    // A task costs a fixed close (read-back, butterfly, partials) and a
    // clean-start tail; the launch ends with about half a task of
    // imbalance.  Balancing the two gives T ~ sqrt(c · trees / particles
    // per tree) (c = 0.6 fitted to task-size sweeps of cfg2, cfg3 and cfg5
    // at t = 0.25 and 2, profiles/r2/tsweep.md), and no fewer than ~16
    // tasks per warp of a 4096-warp grid's trees; >= 1024 trees keep the
    // per-task drain to a few percent; <= 32768 keeps the launch's end tail
    // short (cfg4, task sizes 2048 … 65536 measured: 32768 best).  Small
    // workloads (< 4096 x 1024 trees) are latency-bound: there the floor
    // drops so that every warp of a 4096-warp grid gets about one task (a
    // multiple of 32 trees, at least 128).
    const int64_t floor_T = std::min<int64_t>(
        1024, std::max<int64_t>(128, (total / 4096 + 31) / 32 * 32));
    T = total / (int64_t(4096) * 16);
    if (total >= int64_t(4096) * 1024) {
      const double tb = std::sqrt(0.6 * static_cast<double>(total) / expected_particles(h, t));
      T = std::max<int64_t>(T, (static_cast<int64_t>(tb) + 31) / 32 * 32);
    }
    T = std::max<int64_t>(T, floor_T);
    T = std::min<int64_t>(T, 32768);
  }
  T = std::min<int64_t>(T, n_trees);
  // task ids are 32-bit in the kernel: grow tasks until they number < 2^31
  // (n_points < 2^31, so T = n_trees — one task per node — always ends it)
  while (T < n_trees && n_points * ((n_trees + T - 1) / T) >= (int64_t(1) << 31))
    T = std::min<int64_t>(T * 2, n_trees);
  if (n_points * ((n_trees + T - 1) / T) >= (int64_t(1) << 31))
    return fail(RT_E_ARG, "too many tasks (n_points = %lld)", static_cast<long long>(n_points));
  L.T = T;
  L.tpn = (n_trees + T - 1) / T;
  L.n_tasks = n_points * L.tpn;
  const int64_t need_ctas = (L.n_tasks + rtk::kWarpsPerCta - 1) / rtk::kWarpsPerCta;
  L.grid = static_cast<int>(std::min<int64_t>(grid, need_ctas));
  return RT_OK;
}

constexpr int kReduceWarps = 8;
constexpr int64_t kReduceSeg = 512;   // tasks per segment (at least; see reduce_seg)

// Tasks per segment of the second pass: a function of the task count alone
// (never of the GPU), so the summation order — and the sums' bits — are fixed
// by the launch's task decomposition.
static inline int64_t reduce_seg(int64_t tpn) {
  return std::max<int64_t>(kReduceSeg, (tpn + 65534) / 65535);
}

// Adds (bin counts → trees, pruned trees, splits) of one node's finished sums
// to the event counters; lane = bin, all 32 lanes
__device__ __forceinline__ void fold_bin_counts(int b, int nb, double c, unsigned long long* stats) {
  unsigned long long trees = b < nb ? static_cast<unsigned long long>(c) : 0ull;
  unsigned long long splits = trees * static_cast<unsigned long long>(b);
  for (int o = 16; o > 0; o >>= 1) {
    trees += __shfl_xor_sync(0xffffffffu, trees, o);
    splits += __shfl_xor_sync(0xffffffffu, splits, o);
  }
  if (b == 0) {
    atomicAdd(stats + 0, trees);
    atomicAdd(stats + 4, splits);
  }
  if (b == nb - 1) atomicAdd(stats + 1, static_cast<unsigned long long>(c));
}

__global__ void __launch_bounds__(32 * kReduceWarps)
reduce_tasks_kernel(const double* __restrict__ partials, int64_t tpn, int nb, int64_t seg,
                    double* __restrict__ out, unsigned long long* __restrict__ stats) {
  // second pass, atomic-free and deterministic: CTA (i, s) sums node i's
  // tasks [s·seg, (s+1)·seg) with eight warps — warp w takes the segment's
  // tasks w, w+8, w+16, … in ascending order, lane = bin — and adds the eight
  // partial sums in warp order.  One segment: the node's sums, and the exact
  // bin counts also give trees, pruned trees and splits (a pruned tree
  // aborted at its (K+1)-th split).  Several: per-segment sums, combined in
  // segment order by reduce_segments_kernel (the segments give a node with
  // many tasks — shared trees, few nodes — enough CTAs to stream its partials).
  __shared__ double part[kReduceWarps][32][3];
  const int64_t i = blockIdx.x, sg = blockIdx.y, nseg = gridDim.y;
  const int b = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t q0 = sg * seg, q1 = min(tpn, q0 + seg);
  double s1 = 0.0, s2 = 0.0, c = 0.0;
  if (b < nb) {
    const int64_t st = static_cast<int64_t>(nb) * 3;
    const double* p = partials + (i * tpn * nb + b) * 3 + (q0 + w) * st;
    for (int64_t q = q0 + w; q < q1; q += kReduceWarps, p += kReduceWarps * st) {
      s1 += p[0];
      s2 += p[1];
      c += p[2];
    }
  }
  part[w][b][0] = s1;
  part[w][b][1] = s2;
  part[w][b][2] = c;
  __syncthreads();
  if (w != 0) return;
  s1 = s2 = c = 0.0;
#pragma unroll
  for (int v = 0; v < kReduceWarps; ++v) {
    s1 += part[v][b][0];
    s2 += part[v][b][1];
    c += part[v][b][2];
  }
  if (b < nb) {
    double* o = out + ((i * nseg + sg) * nb + b) * 3;
    o[0] = s1;
    o[1] = s2;
    o[2] = c;
  }
  if (nseg == 1) fold_bin_counts(b, nb, c, stats);
}

// Node i's segment sums added in segment order (one warp per node, lane = bin).
__global__ void __launch_bounds__(32)
reduce_segments_kernel(const double* __restrict__ segs, int64_t nseg, int nb,
                       double* __restrict__ sums, unsigned long long* __restrict__ stats) {
  const int64_t i = blockIdx.x;
  const int b = threadIdx.x;
  double s1 = 0.0, s2 = 0.0, c = 0.0;
  if (b < nb) {
    const double* p = segs + (i * nseg * nb + b) * 3;
    for (int64_t sg = 0; sg < nseg; ++sg, p += static_cast<int64_t>(nb) * 3) {
      s1 += p[0];
      s2 += p[1];
      c += p[2];
    }
    double* o = sums + (i * nb + b) * 3;
    o[0] = s1;
    o[1] = s2;
    o[2] = c;
  }
  fold_bin_counts(b, nb, c, stats);
}

// The second pass over partials[n_points][tpn][nb][3] into d_sums[n_points][nb][3].
static rt_status launch_reduce(rt_handle* h, int64_t n_points, int64_t tpn, int nb, double* d_sums,
                               cudaStream_t st) {
  const int64_t seg = reduce_seg(tpn), nseg = (tpn + seg - 1) / seg;
  auto* stats = static_cast<unsigned long long*>(h->stats.p);
  const auto* parts = static_cast<const double*>(h->partials.p);
  if (nseg <= 1) {
    reduce_tasks_kernel<<<dim3(static_cast<unsigned>(n_points), 1), 32 * kReduceWarps, 0, st>>>(
        parts, tpn, nb, seg, d_sums, stats);
    RT_CUDA(cudaGetLastError());
    return RT_OK;
  }
  RT_CUDA(h->segs.ensure(static_cast<size_t>(n_points) * nseg * nb * 3 * sizeof(double)));
  auto* segs = static_cast<double*>(h->segs.p);
  reduce_tasks_kernel<<<dim3(static_cast<unsigned>(n_points), static_cast<unsigned>(nseg)),
                        32 * kReduceWarps, 0, st>>>(parts, tpn, nb, seg, segs, stats);
  RT_CUDA(cudaGetLastError());
  reduce_segments_kernel<<<static_cast<unsigned>(n_points), 32, 0, st>>>(segs, nseg, nb, d_sums, stats);
  RT_CUDA(cudaGetLastError());
  return RT_OK;
}

__global__ void finalize_kernel(const double* __restrict__ sums, int K, double N,
                                double* __restrict__ coeffs, double* __restrict__ se,
                                double* __restrict__ u_sum, double* __restrict__ se_sum) {
  // c_n = ΣC_n/N, se_n = sqrt(max(0, ΣC_n²/N − c_n²)/(N−1)) (R4, R11)
  const int64_t i = blockIdx.x;
  const int b = threadIdx.x;
  const int nb = K + 2;
  double c = 0.0, s2 = 0.0;
  if (b <= K) {
    const double* s = sums + (i * nb + b) * 3;
    c = s[0] / N;
    s2 = s[1];
    const double v = s2 / N - c * c;
    if (coeffs) coeffs[i * (K + 1) + b] = c;
    if (se) se[i * (K + 1) + b] = sqrt((v > 0.0 ? v : 0.0) / (N - 1.0));
  }
  for (int o = 16; o > 0; o >>= 1) {
    c += __shfl_xor_sync(0xffffffffu, c, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (b == 0) {
    if (u_sum) u_sum[i] = c;
    if (se_sum) {
      const double v = s2 / N - c * c;
      se_sum[i] = sqrt((v > 0.0 ? v : 0.0) / (N - 1.0));
    }
  }
}

static rt_status check_run_args(const rt_handle* h, int64_t n_points, double t,
                                int64_t tree_offset, int64_t n_trees) {
  if (!h) return fail(RT_E_ARG, "null handle");
  if (n_points < 1) return fail(RT_E_ARG, "n_points must be >= 1");
  if (!(t > 0.0) || !is_fin(t)) return fail(RT_E_ARG, "t must be finite and > 0");
  if (n_trees < 2) return fail(RT_E_ARG, "n_trees must be >= 2");
  if (tree_offset < 0 || tree_offset + n_trees > (int64_t(1) << 32))
    return fail(RT_E_ARG, "tree range must lie in [0, 2^32)");
  if (n_trees >= (int64_t(1) << 31)) return fail(RT_E_ARG, "n_trees must be < 2^31 per call");
  if (n_points >= (int64_t(1) << 31)) return fail(RT_E_ARG, "n_points must be < 2^31");
  return RT_OK;
}

// Runs the tree walk + task reduction; d_sums receives [n][K+2][3].
static void fill_params(const rt_handle* h, WalkParams& P, double t, uint64_t seed) {
  const rt_eq_params& p = h->p;
  const Norm& nz = h->nz;
  std::memset(&P, 0, sizeof(P));
  P.rk = rtk::make_round_keys(seed);
  P.inv_lambda = nz.inv_lambda;
  P.two_d = 2.0 * p.D;
  P.amp = p.init_amp;
  P.inv_scale = 1.0 / p.init_scale;
  P.inv_scale2 = 1.0 / (p.init_scale * p.init_scale);
  P.t = t;
  // (no support — a purely linear f: every split draws entry 0, whose zero
  // weight makes the killed tree's product 0)
  for (int q = 0; q < 9; ++q) { P.thr[q] = 0xffffffffu; P.w[q] = 0.0; P.kval[q] = 0; }
  for (int q = 0; q < nz.n_support; ++q) {
    P.w[q] = nz.w[q];
    P.thr[q] = static_cast<uint32_t>(nz.thresh[q] - 1);
    P.kval[q] = nz.support[q];
  }
  P.n_support = nz.n_support;
  // f2/f3 weight factors
  P.var_s = 0u;
  for (int q = 0; q < nz.n_support; ++q)
    if (p.coef_kind[nz.support[q]] == RT_COEF_GAUSS_RATIONAL) P.var_s |= 1u << q;
  P.wmode = (P.var_s != 0u ? 1 : 0) | (p.strategy == RT_STRATEGY_A_SHIFT ? 2 : 0);
  P.lam = nz.lambda;
  P.root = p.strategy == RT_STRATEGY_A_SHIFT ? std::exp(nz.lambda * t) : 1.0;   // u = v e^{λt}
  P.coef_axis = p.coef_axis;
  P.coef_inv_s2 = 1.0 / (p.coef_scale * p.coef_scale);
  P.coef_t0 = p.coef_t0;
  P.tq = nz.tq;
  P.inv_q = p.strategy == RT_STRATEGY_B ? 1.0 / nz.q_hat : 1.0;
  P.beta = nz.beta;
  P.K = p.K;
  P.nb = p.K + 2;
}

// The handle's scratch (partials, lane-private sums, overflow stacks, task
// counter, PDD tables) is shared by every call: work on a stream other than
// the one that last used it waits for that work first (ev[2] is recorded
// after every call's last use of the scratch).  (a host call on
// the handle's own stream after an unsynchronised _dev call raced on it.)
// Work captured into a CUDA graph is ordered by the graph's user instead
// (a capture may not wait on uncaptured work), so captures neither wait nor
// leave a mark.
static bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

static rt_status order_after_last(rt_handle* h, cudaStream_t st) {
  if (h->scratch_used && h->last_stream != st && !capturing(st))
    RT_CUDA(cudaStreamWaitEvent(st, h->ev[2], 0));
  return RT_OK;
}

static void mark_scratch(rt_handle* h, cudaStream_t st) {
  h->last_stream = st;
  h->scratch_used = !capturing(st);
}

// Shared trees (NEXT row f4): phase 1 walks every tree once
// (tree_walk_kernel<…, SH>) writing tree summaries and leaf displacements in
// chunks that fit a memory budget; phase 2 (shared_eval_kernel) evaluates all
// nodes of every tree; the per-node task reduction is shared.
template <int DIM, int GK, bool REC>
static KernelFn eval_kernel(int npt) {
  return npt == 2 ? reinterpret_cast<KernelFn>(rtk::shared_eval_kernel<DIM, GK, REC, 2>)
                  : reinterpret_cast<KernelFn>(rtk::shared_eval_kernel<DIM, GK, REC, 1>);
}

static rt_status run_walk_shared(rt_handle* h, KernelFn prod, int smem, int pool_cap,
                                 const double* d_points, int64_t n_points, double t,
                                 int64_t tree_offset, int64_t n_trees, uint64_t seed, int rec_shift,
                                 rtk::TreeRec* d_recs, double* d_sums, cudaStream_t st, int grid) {
  const rt_eq_params& p = h->p;
  const Norm& nz = h->nz;
  const int nb = p.K + 2, nf = p.dim + 2, d = p.dim;
  int kmax = 0;
  for (int q = 0; q < nz.n_support; ++q) kmax = std::max(kmax, nz.support[q]);
  const int lmax = 1 + p.K * std::max(0, kmax - 1);           // leaves of a kept tree
  // per-tree slot: the leaf displacements, or μ and V for Gaussian data
  const int64_t slot = p.init_kind == RT_G_GAUSS ? d + 1 : static_cast<int64_t>(lmax) * d;
  const double per_tree = static_cast<double>(slot) * 8 + sizeof(rtk::TreeSum);
  int64_t M = std::max<int64_t>(1, std::min<int64_t>(n_trees, static_cast<int64_t>(4.0e9 / per_tree)));
  if (h->tpt_override > 0) M = std::min(M, h->tpt_override);   // (tests: force several chunks)
  const int64_t n_chunks = (n_trees + M - 1) / M;
  // phase 2 geometry: 64 or 128 nodes (1 or 2 per thread) x tpb trees per
  // CTA; about four waves of resident CTAs per chunk (the last wave's tail
  // is then a small share)
  const int npt = n_points >= 256 ? 2 : 1;
  const int npc = rtk::kEvalThreads * npt;
  const int tiles = static_cast<int>((n_points + npc - 1) / npc);
  KernelFn ev = nullptr, evr = nullptr;
#define RT_E(D, G) if (p.dim == D && p.init_kind == G) { ev = eval_kernel<D, G, false>(npt); evr = eval_kernel<D, G, true>(npt); }
  RT_E(1, 0) RT_E(1, 1) RT_E(1, 2) RT_E(1, 3) RT_E(2, 0) RT_E(2, 1) RT_E(2, 2) RT_E(2, 3)
  RT_E(3, 0) RT_E(3, 1) RT_E(3, 2) RT_E(3, 3)
#undef RT_E
  // (148 = B200's SM count as a constant, not the device's: the tree blocks
  // fix the summation order, which must not depend on the GPU it runs on)
  int ev_per_sm = 0;
  RT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ev_per_sm, (const void*)ev, rtk::kEvalThreads, 0));
  const int64_t want_blocks = std::max<int64_t>(1, (int64_t(4) * 148 * std::max(1, ev_per_sm) + tiles - 1) / tiles);
  int64_t tpb = (M + want_blocks - 1) / want_blocks;
  tpb = std::max<int64_t>(128, std::min<int64_t>(tpb, 8192));
  int64_t tpn_total = 0;
  for (int64_t c = 0; c < n_chunks; ++c) tpn_total += (std::min(M, n_trees - c * M) + tpb - 1) / tpb;
  RT_CUDA(h->partials.ensure(static_cast<size_t>(n_points) * tpn_total * nb * 3 * sizeof(double)));
  RT_CUDA(h->sh_tsum.ensure(static_cast<size_t>(M) * sizeof(rtk::TreeSum)));
  RT_CUDA(h->sh_leaves.ensure(static_cast<size_t>(M) * slot * sizeof(double)));
  RT_CUDA(h->sh_sorted.ensure(static_cast<size_t>(M) * sizeof(rtk::TreeSum)));
  RT_CUDA(h->sh_boff.ensure(static_cast<size_t>((M + tpb - 1) / tpb) * (nb + 1) * sizeof(int32_t)));
  const int gcap = 32 * (p.K + 1);
  const size_t nwarps = static_cast<size_t>(grid) * rtk::kWarpsPerCta;
  RT_CUDA(h->gpool.ensure(nwarps * gcap * nf * sizeof(double)));
  RT_CUDA(h->gaux.ensure(nwarps * 2 * gcap * sizeof(int32_t)));
  if (h->pool_override > 0) pool_cap = std::min(pool_cap, static_cast<int>(h->pool_override));

  WalkParams P;
  fill_params(h, P, t, seed);
  P.points = d_points;
  P.n_points = static_cast<int32_t>(n_points);
  P.pool_cap = pool_cap;
  P.gpool = static_cast<double*>(h->gpool.p);
  P.gaux = static_cast<int32_t*>(h->gaux.p);
  P.gcap = gcap;
  P.stats = static_cast<unsigned long long*>(h->stats.p);
  P.task_ctr = reinterpret_cast<unsigned int*>(P.stats + 5);
  P.tsum = static_cast<rtk::TreeSum*>(h->sh_tsum.p);
  P.leaves = static_cast<double*>(h->sh_leaves.p);
  P.lmax = lmax;
  rtk::EvalParams E;
  std::memset(&E, 0, sizeof(E));
  E.tsum = P.tsum; E.leaves = P.leaves; E.lmax = lmax; E.tpb = static_cast<int32_t>(tpb);
  E.points = d_points; E.n_points = static_cast<int32_t>(n_points); E.K = p.K; E.nb = nb;
  E.amp = P.amp; E.inv_scale = P.inv_scale; E.inv_scale2 = P.inv_scale2;
  E.partials = static_cast<double*>(h->partials.p); E.tpn_total = tpn_total;
  E.recs = d_recs; E.rec_shift = rec_shift;
  E.n_rec = (n_trees + (int64_t(1) << rec_shift) - 1) >> rec_shift;
  E.sorted = static_cast<rtk::TreeSum*>(h->sh_sorted.p);
  E.boff = static_cast<int32_t*>(h->sh_boff.p);

  RT_CUDA(cudaMemsetAsync(h->stats.p, 0, 6 * sizeof(unsigned long long), st));
  RT_CUDA(cudaEventRecord(h->ev[0], st));
  int64_t q0 = 0;
  for (int64_t c = 0; c < n_chunks; ++c) {
    const int64_t Mc = std::min(M, n_trees - c * M);
    // phase 1: tasks are tree ranges of one "unit"; ~8 tasks per warp
    const int64_t T1 = std::max<int64_t>(32, std::min<int64_t>(4096, Mc / static_cast<int64_t>(nwarps * 8)));
    P.n_trees = static_cast<int32_t>(Mc);
    P.tree_offset = static_cast<uint32_t>(tree_offset + c * M);
    P.T = static_cast<int32_t>(T1);
    P.tpn = static_cast<int32_t>((Mc + T1 - 1) / T1);
    P.n_tasks = P.tpn;
    RT_CUDA(cudaMemsetAsync(P.task_ctr, 0, sizeof(unsigned int), st));
    const int g1 = static_cast<int>(std::min<int64_t>(grid, (P.n_tasks + rtk::kWarpsPerCta - 1) / rtk::kWarpsPerCta));
    prod<<<g1, rtk::kThreads, smem, st>>>(P);
    RT_CUDA(cudaGetLastError());
    // phase 2: every node of every tree of the chunk
    E.M = Mc;
    E.q0 = q0;
    E.rel0 = static_cast<uint32_t>(c * M);
    const dim3 eg(static_cast<unsigned>(tiles), static_cast<unsigned>((Mc + tpb - 1) / tpb));
    rtk::bin_sort_kernel<<<eg.y, 32, 0, st>>>(E);
    RT_CUDA(cudaGetLastError());
    reinterpret_cast<void (*)(rtk::EvalParams)>(ev)<<<eg, rtk::kEvalThreads, 0, st>>>(E);
    RT_CUDA(cudaGetLastError());
    if (d_recs) {
      reinterpret_cast<void (*)(rtk::EvalParams)>(evr)<<<eg, rtk::kEvalThreads, 0, st>>>(E);
      RT_CUDA(cudaGetLastError());
    }
    q0 += eg.y;
  }
  RT_CUDA(cudaEventRecord(h->ev[1], st));
  {
    const rt_status o = launch_reduce(h, n_points, tpn_total, nb, d_sums, st);
    if (o != RT_OK) return o;
  }
  mark_scratch(h, st);
  h->have_timing = true;
  h->host_total_ms = -1.0;
  return RT_OK;
}

static rt_status run_walk(rt_handle* h, const double* d_points, int64_t n_points, double t,
                          int64_t tree_offset, int64_t n_trees, uint64_t seed, int rec_shift,
                          rtk::TreeRec* d_recs, double* d_sums, cudaStream_t st) {
  {
    const rt_status o = order_after_last(h, st);
    if (o != RT_OK) return o;
  }
  const rt_eq_params& p = h->p;
  const Norm& nz = h->nz;
  int smem = 0, pool_cap = 0;
  KernelFn prod = nullptr;
  const bool sh = p.shared != 0;
  bool var = false;
  for (int k = 0; k <= 8; ++k) var = var || p.coef_kind[k] != RT_COEF_CONST;
  // the general kernel only where f2 weight factors (the shift, variable
  // coefficients), > 3 offspring kinds or an empty support (purely linear f)
  // need it — Strategy B with constant coefficients has none of them
  const bool gen = h->force_gen || p.strategy == RT_STRATEGY_A_SHIFT || var || nz.n_support > 3 ||
                   nz.n_support == 0;
  KernelFn fn = kernel_for(p.dim, p.init_kind, d_recs != nullptr, p.precision == RT_PREC_FP32_POS,
                           p.strategy == RT_STRATEGY_B, sh, gen, &prod, &smem, &pool_cap);
  if (!fn) return fail(RT_E_ARG, "no kernel for dim=%d init_kind=%d", p.dim, p.init_kind);
  if (smem > 48 * 1024) {
    RT_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    RT_CUDA(cudaFuncSetAttribute((const void*)prod, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  Launch L;
  rt_status s = plan_launch(h, prod, smem, n_points, n_trees, t, L);   // same grid for the trace
  if (s != RT_OK) return s;
  if (sh) return run_walk_shared(h, prod, smem, pool_cap, d_points, n_points, t, tree_offset, n_trees,
                                 seed, rec_shift, d_recs, d_sums, st, L.grid);
  const int nb = p.K + 2;
  const int nf = p.dim + 2;
  // partials are per node in either mode: [n_points][tpn][nb][3]
  RT_CUDA(h->partials.ensure(static_cast<size_t>(n_points) * L.tpn * nb * 3 * sizeof(double)));
  // overflow stack entries once a warp's shared-memory pool is exhausted: a
  // lane's stack never exceeds K groups, so 32 (K+1) entries per warp always
  // suffice: [warps][gcap][nf] doubles and [warps][2][gcap] int32
  const int gcap = 32 * (p.K + 1);
  const size_t nwarps = static_cast<size_t>(L.grid) * rtk::kWarpsPerCta;
  RT_CUDA(h->gpool.ensure(nwarps * gcap * nf * sizeof(double)));
  RT_CUDA(h->gaux.ensure(nwarps * 2 * gcap * sizeof(int32_t)));
  // lane-private order-bin sums (RED targets): [warps][nb][ΣC, ΣC², n][32]
  RT_CUDA(h->lacc.ensure(nwarps * nb * 96 * sizeof(double)));
  if (h->pool_override > 0) pool_cap = std::min(pool_cap, static_cast<int>(h->pool_override));

  WalkParams P;
  fill_params(h, P, t, seed);
  P.n_points = static_cast<int32_t>(n_points);
  P.points = d_points;
  P.n_trees = static_cast<int32_t>(n_trees);
  P.tree_offset = static_cast<uint32_t>(tree_offset);
  P.T = static_cast<int32_t>(L.T);
  P.tpn = static_cast<int32_t>(L.tpn);
  P.n_tasks = static_cast<int32_t>(L.n_tasks);
  P.partials = static_cast<double*>(h->partials.p);
  P.pool_cap = pool_cap;
  P.gpool = static_cast<double*>(h->gpool.p);
  P.gaux = static_cast<int32_t*>(h->gaux.p);
  P.lacc = static_cast<double*>(h->lacc.p);
  P.gcap = gcap;
  P.recs = d_recs;
  P.rec_shift = rec_shift;
  P.n_rec = (n_trees + (int64_t(1) << rec_shift) - 1) >> rec_shift;
  P.stats = static_cast<unsigned long long*>(h->stats.p);
  P.task_ctr = reinterpret_cast<unsigned int*>(P.stats + 5);

  // debug: RT_WARP_TIMES=<file> appends one line per launch with every warp's
  // start/end %globaltimer (load-balance diagnostics; never set in production)
  const char* wt_path = std::getenv("RT_WARP_TIMES");
  if (wt_path != nullptr) {
    RT_CUDA(h->wtime.ensure(nwarps * 4 * sizeof(unsigned long long)));
    P.wtime = static_cast<unsigned long long*>(h->wtime.p);
  }
  RT_CUDA(cudaMemsetAsync(h->stats.p, 0, 6 * sizeof(unsigned long long), st));   // + task counter
  RT_CUDA(cudaEventRecord(h->ev[0], st));
  fn<<<L.grid, rtk::kThreads, smem, st>>>(P);
  RT_CUDA(cudaGetLastError());
  if (wt_path != nullptr) {
    std::vector<unsigned long long> wt(nwarps * 4);
    RT_CUDA(cudaMemcpyAsync(wt.data(), P.wtime, wt.size() * 8, cudaMemcpyDeviceToHost, st));
    RT_CUDA(cudaStreamSynchronize(st));
    if (FILE* f = std::fopen(wt_path, "a")) {
      for (size_t q = 0; q < wt.size(); ++q) std::fprintf(f, "%llu%c", wt[q], q + 1 < wt.size() ? ' ' : '\n');
      std::fclose(f);
    }
  }
  RT_CUDA(cudaEventRecord(h->ev[1], st));
  {
    const rt_status o = launch_reduce(h, n_points, L.tpn, nb, d_sums, st);
    if (o != RT_OK) return o;
  }
  mark_scratch(h, st);
  h->have_timing = true;
  h->host_total_ms = -1.0;
  return RT_OK;
}

extern "C" rt_status rt_sums_dev(rt_handle* h, const double* d_points, int64_t n_points,
                                 double t, int64_t tree_offset, int64_t n_trees, uint64_t seed,
                                 double* d_sums, void* stream) {
  rt_status s = check_run_args(h, n_points, t, tree_offset, n_trees);
  if (s != RT_OK) return s;
  if (!d_points || !d_sums) return fail(RT_E_ARG, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  s = run_walk(h, d_points, n_points, t, tree_offset, n_trees, seed, 0, nullptr, d_sums, st);
  if (s != RT_OK) return s;
  RT_CUDA(cudaEventRecord(h->ev[2], st));
  return RT_OK;
}

extern "C" rt_status rt_finalize_dev(const double* d_sums, int64_t n_points, int32_t K,
                                     int64_t N_total, double* d_coeffs, double* d_stderr,
                                     double* d_u_sum, double* d_se_sum, void* stream) {
  if (!d_sums) return fail(RT_E_ARG, "null sums");
  if (n_points < 1 || K < 0 || K > 30 || N_total < 2) return fail(RT_E_ARG, "bad sizes");
  finalize_kernel<<<static_cast<unsigned>(n_points), 32, 0, static_cast<cudaStream_t>(stream)>>>(
      d_sums, K, static_cast<double>(N_total), d_coeffs, d_stderr, d_u_sum, d_se_sum);
  RT_CUDA(cudaGetLastError());
  return RT_OK;
}

extern "C" rt_status rt_estimate_dev(rt_handle* h, const double* d_points, int64_t n_points,
                                     double t, int64_t n_trees, uint64_t seed,
                                     double* d_out_coeffs, double* d_out_stderr, void* stream) {
  rt_status s = check_run_args(h, n_points, t, 0, n_trees);
  if (s != RT_OK) return s;
  if (!d_points || !d_out_coeffs || !d_out_stderr) return fail(RT_E_ARG, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nb = h->p.K + 2;
  RT_CUDA(h->sums.ensure(static_cast<size_t>(n_points) * nb * 3 * sizeof(double)));
  double* sums = static_cast<double*>(h->sums.p);
  s = run_walk(h, d_points, n_points, t, 0, n_trees, seed, 0, nullptr, sums, st);
  if (s != RT_OK) return s;
  finalize_kernel<<<static_cast<unsigned>(n_points), 32, 0, st>>>(
      sums, h->p.K, static_cast<double>(n_trees), d_out_coeffs, d_out_stderr, nullptr, nullptr);
  RT_CUDA(cudaGetLastError());
  RT_CUDA(cudaEventRecord(h->ev[2], st));
  return RT_OK;
}

extern "C" rt_status rt_trace_dev(rt_handle* h, const double* d_points, int64_t n_points,
                                  double t, int64_t tree_offset, int64_t n_trees, uint64_t seed,
                                  int32_t rec_shift, rt_tree_rec* d_recs, double* d_sums,
                                  void* stream) {
  rt_status s = check_run_args(h, n_points, t, tree_offset, n_trees);
  if (s != RT_OK) return s;
  if (!d_points || !d_recs) return fail(RT_E_ARG, "null pointer");
  if (rec_shift < 0 || rec_shift > 31) return fail(RT_E_ARG, "rec_shift must be in [0, 31]");
  static_assert(sizeof(rt_tree_rec) == sizeof(rtk::TreeRec), "record layout");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nb = h->p.K + 2;
  double* sums = d_sums;
  if (!sums) {
    RT_CUDA(h->sums.ensure(static_cast<size_t>(n_points) * nb * 3 * sizeof(double)));
    sums = static_cast<double*>(h->sums.p);
  }
  s = run_walk(h, d_points, n_points, t, tree_offset, n_trees, seed, rec_shift,
               reinterpret_cast<rtk::TreeRec*>(d_recs), sums, st);
  if (s != RT_OK) return s;
  RT_CUDA(cudaEventRecord(h->ev[2], st));
  return RT_OK;
}

extern "C" rt_status rt_get_stats(const rt_handle* hc, rt_stats* out) {
  if (!hc || !out) return fail(RT_E_ARG, "null pointer");
  rt_handle* h = const_cast<rt_handle*>(hc);
  std::memset(out, 0, sizeof(*out));
  if (!h->have_timing) return RT_OK;
  RT_CUDA(cudaEventSynchronize(h->ev[2]));
  unsigned long long v[5];
  RT_CUDA(cudaMemcpy(v, h->stats.p, sizeof(v), cudaMemcpyDeviceToHost));
  out->trees = static_cast<int64_t>(v[0]);
  out->pruned = static_cast<int64_t>(v[1]);
  // every processed particle reaches its horizon (a leaf) or splits — the
  // aborting split of a pruned tree included (the kernel counts no particles)
  out->particles = static_cast<int64_t>(v[3]) + static_cast<int64_t>(v[4]);
  out->leaves = static_cast<int64_t>(v[3]);
  out->splits = static_cast<int64_t>(v[4]);
  float ms = 0.f;
  RT_CUDA(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
  out->kernel_ms = ms;
  if (h->host_total_ms >= 0.0) {
    out->total_ms = h->host_total_ms;
  } else {
    RT_CUDA(cudaEventElapsedTime(&ms, h->ev[0], h->ev[2]));
    out->total_ms = ms;
  }
  return RT_OK;
}

// ---------------------------------------------------------------------------
// host API
static rt_status check_points_host(const double* pts, int64_t n, int dim) {
  for (int64_t q = 0; q < n * dim; ++q)
    if (!is_fin(pts[q])) return fail(RT_E_ARG, "point coordinate %lld is not finite", (long long)q);
  return RT_OK;
}

extern "C" rt_status rt_estimate(rt_handle* h, const double* points, int64_t n_points, double t,
                                 int64_t n_trees, uint64_t seed, double* out_coeffs,
                                 double* out_stderr) {
  rt_status s = check_run_args(h, n_points, t, 0, n_trees);
  if (s != RT_OK) return s;
  if (!points || !out_coeffs || !out_stderr) return fail(RT_E_ARG, "null pointer");
  s = check_points_host(points, n_points, h->p.dim);
  if (s != RT_OK) return s;
  cudaStream_t st = h->own_stream;
  const size_t pb = static_cast<size_t>(n_points) * h->p.dim * sizeof(double);
  const size_t cb = static_cast<size_t>(n_points) * (h->p.K + 1) * sizeof(double);
  RT_CUDA(h->h_points.ensure(pb));
  RT_CUDA(h->h_coeffs.ensure(cb));
  RT_CUDA(h->h_stderr.ensure(cb));
  RT_CUDA(cudaEventRecord(h->ev[3], st));
  RT_CUDA(cudaMemcpyAsync(h->h_points.p, points, pb, cudaMemcpyHostToDevice, st));
  s = rt_estimate_dev(h, static_cast<double*>(h->h_points.p), n_points, t, n_trees, seed,
                      static_cast<double*>(h->h_coeffs.p), static_cast<double*>(h->h_stderr.p),
                      st);
  if (s != RT_OK) return s;
  RT_CUDA(cudaMemcpyAsync(out_coeffs, h->h_coeffs.p, cb, cudaMemcpyDeviceToHost, st));
  RT_CUDA(cudaMemcpyAsync(out_stderr, h->h_stderr.p, cb, cudaMemcpyDeviceToHost, st));
  RT_CUDA(cudaEventRecord(h->ev[2], st));
  RT_CUDA(cudaStreamSynchronize(st));
  float ms = 0.f;
  RT_CUDA(cudaEventElapsedTime(&ms, h->ev[3], h->ev[2]));
  h->host_total_ms = ms;
  return RT_OK;
}

// ---------------------------------------------------------------------------
// row a8: batched [L/M] Padé, one warp per node (pade.cuh)
static void launch_pade(const double* d_c, int64_t n, int K, int L, int M, const double* d_se_sum,
                        double* d_u, uint32_t* d_flags, cudaStream_t st) {
  const int per_cta = rtk::kPadeThreads / 32;
  rtk::pade_warp_kernel<<<static_cast<unsigned>((n + per_cta - 1) / per_cta), rtk::kPadeThreads, 0, st>>>(
      d_c, n, K, L, M, d_se_sum, d_u, d_flags);
}

static rt_status check_pade_args(int64_t n_points, int32_t K, int32_t L, int32_t M) {
  if (n_points < 1) return fail(RT_E_ARG, "n_points must be >= 1");
  if (L < 0 || M < 0 || M > 16 || L + M > K || K > 30)
    return fail(RT_E_ARG, "need 0 <= L, 0 <= M <= 16, L + M <= K <= 30 (L=%d M=%d K=%d)", L, M, K);
  return RT_OK;
}

extern "C" rt_status rt_pade_dev(const double* d_coeffs, int64_t n_points, int32_t K, int32_t L,
                                 int32_t M, const double* d_se_sum, double* d_u, uint32_t* d_flags,
                                 void* stream) {
  if (!d_coeffs || !d_u) return fail(RT_E_ARG, "null pointer");
  rt_status s = check_pade_args(n_points, K, L, M);
  if (s != RT_OK) return s;
  launch_pade(d_coeffs, n_points, K, L, M, d_se_sum, d_u, d_flags, static_cast<cudaStream_t>(stream));
  RT_CUDA(cudaGetLastError());
  return RT_OK;
}

extern "C" rt_status rt_pade(const double* coeffs, int64_t n_points, int32_t K, int32_t L,
                             int32_t M, const double* se_sum, double* out_u, uint32_t* out_flags) {
  if (!coeffs || !out_u) return fail(RT_E_ARG, "null pointer");
  rt_status s = check_pade_args(n_points, K, L, M);
  if (s != RT_OK) return s;
  const size_t cb = static_cast<size_t>(n_points) * (K + 1) * sizeof(double);
  double *dc = nullptr, *du = nullptr, *dse = nullptr;
  uint32_t* df = nullptr;
  RT_CUDA(cudaMalloc(&dc, cb));
  cudaError_t e = cudaMalloc(&du, n_points * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&df, n_points * sizeof(uint32_t));
  if (e == cudaSuccess && se_sum) e = cudaMalloc(&dse, n_points * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(dc, coeffs, cb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && se_sum)
    e = cudaMemcpy(dse, se_sum, n_points * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    launch_pade(dc, n_points, K, L, M, dse, du, df, nullptr);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out_u, du, n_points * sizeof(double), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && out_flags)
    e = cudaMemcpy(out_flags, df, n_points * sizeof(uint32_t), cudaMemcpyDeviceToHost);
  cudaFree(dc);
  cudaFree(du);
  cudaFree(df);
  cudaFree(dse);
  if (e != cudaSuccess) return fail(RT_E_CUDA, "rt_pade: %s", cudaGetErrorString(e));
  return RT_OK;
}

// ---------------------------------------------------------------------------
// row a9: interface nodes on planes (R14)
static double lin(double lo, double hi, int n, int j) {
  if (n == 1) return lo;
  return lo + (hi - lo) * (static_cast<double>(j) / static_cast<double>(n - 1));
}

static rt_status place_nodes(int dim, const rt_plane* planes, int32_t n_planes,
                             int64_t max_points, std::vector<double>& pts) {
  std::set<std::vector<double>> seen;
  pts.clear();
  int64_t count = 0;
  for (int32_t pl = 0; pl < n_planes && count < max_points; ++pl) {
    const rt_plane& P = planes[pl];
    if (P.axis < 0 || P.axis >= dim) return fail(RT_E_ARG, "plane %d: axis out of range", pl);
    if (P.n_per_dim < 1) return fail(RT_E_ARG, "plane %d: n_per_dim must be >= 1", pl);
    if (!is_fin(P.value) || !is_fin(P.lo) || !is_fin(P.hi))
      return fail(RT_E_ARG, "plane %d: non-finite bounds", pl);
    int free_ax[2] = {0, 0}, nfree = 0;
    for (int a = 0; a < dim; ++a)
      if (a != P.axis) free_ax[nfree++] = a;
    int64_t total = 1;
    for (int f = 0; f < nfree; ++f) total *= P.n_per_dim;
    for (int64_t idx = 0; idx < total && count < max_points; ++idx) {
      std::vector<double> x(dim, 0.0);
      x[P.axis] = P.value;
      int64_t rem = idx;
      for (int f = nfree - 1; f >= 0; --f) {   // row-major: last free axis fastest
        const int j = static_cast<int>(rem % P.n_per_dim);
        rem /= P.n_per_dim;
        x[free_ax[f]] = lin(P.lo, P.hi, P.n_per_dim, j);
      }
      if (!seen.insert(x).second) continue;
      pts.insert(pts.end(), x.begin(), x.end());
      ++count;
    }
  }
  return RT_OK;
}

extern "C" rt_status rt_interface_values(rt_handle* h, const rt_plane* planes, int32_t n_planes,
                                         int64_t max_points, double t, int64_t n_trees,
                                         uint64_t seed, int32_t L, int32_t M, double* out_points,
                                         double* out_u, double* out_stderr, uint32_t* out_flags,
                                         int64_t* out_n_points) {
  if (!h || !planes || !out_points || !out_u || !out_stderr || !out_n_points)
    return fail(RT_E_ARG, "null pointer");
  if (n_planes < 1 || max_points < 1) return fail(RT_E_ARG, "need n_planes >= 1, max_points >= 1");
  const int K = h->p.K;
  rt_status s = check_pade_args(1, K, L, M);
  if (s != RT_OK) return s;
  std::vector<double> pts;
  s = place_nodes(h->p.dim, planes, n_planes, max_points, pts);
  if (s != RT_OK) return s;
  const int64_t n = static_cast<int64_t>(pts.size()) / h->p.dim;
  if (n < 1) return fail(RT_E_ARG, "no nodes placed");
  s = check_run_args(h, n, t, 0, n_trees);
  if (s != RT_OK) return s;
  cudaStream_t st = h->own_stream;
  const int nb = K + 2;
  RT_CUDA(h->h_points.ensure(pts.size() * sizeof(double)));
  RT_CUDA(h->h_coeffs.ensure(static_cast<size_t>(n) * (K + 1) * sizeof(double)));
  RT_CUDA(h->h_stderr.ensure(static_cast<size_t>(n) * 2 * sizeof(double)));
  RT_CUDA(h->h_flags.ensure(static_cast<size_t>(n) * sizeof(uint32_t)));
  RT_CUDA(h->sums.ensure(static_cast<size_t>(n) * nb * 3 * sizeof(double)));
  double* d_pts = static_cast<double*>(h->h_points.p);
  double* d_c = static_cast<double*>(h->h_coeffs.p);
  double* d_u = static_cast<double*>(h->h_stderr.p);
  double* d_se = d_u + n;
  uint32_t* d_fl = static_cast<uint32_t*>(h->h_flags.p);
  double* d_sums = static_cast<double*>(h->sums.p);
  RT_CUDA(cudaEventRecord(h->ev[3], st));
  RT_CUDA(cudaMemcpyAsync(d_pts, pts.data(), pts.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  s = run_walk(h, d_pts, n, t, 0, n_trees, seed, 0, nullptr, d_sums, st);
  if (s != RT_OK) return s;
  finalize_kernel<<<static_cast<unsigned>(n), 32, 0, st>>>(d_sums, K, static_cast<double>(n_trees),
                                                            d_c, nullptr, nullptr, d_se);
  RT_CUDA(cudaGetLastError());
  launch_pade(d_c, n, K, L, M, d_se, d_u, d_fl, st);
  RT_CUDA(cudaGetLastError());
  RT_CUDA(cudaEventRecord(h->ev[2], st));
  RT_CUDA(cudaMemcpyAsync(out_points, d_pts, pts.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  RT_CUDA(cudaMemcpyAsync(out_u, d_u, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  RT_CUDA(cudaMemcpyAsync(out_stderr, d_se, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (out_flags)
    RT_CUDA(cudaMemcpyAsync(out_flags, d_fl, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  RT_CUDA(cudaStreamSynchronize(st));
  float ms = 0.f;
  RT_CUDA(cudaEventElapsedTime(&ms, h->ev[3], h->ev[2]));
  h->host_total_ms = ms;
  *out_n_points = n;
  return RT_OK;
}

// ---------------------------------------------------------------------------
// RNG parity hook
__global__ void philox_kernel(rtk::RoundKeys rk, const uint32_t* __restrict__ ctr, int64_t n,
                              uint32_t* __restrict__ out) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const uint4 r = rtk::philox4x32_10(ctr[4 * q], ctr[4 * q + 1], ctr[4 * q + 2], ctr[4 * q + 3], rk);
  out[4 * q] = r.x;
  out[4 * q + 1] = r.y;
  out[4 * q + 2] = r.z;
  out[4 * q + 3] = r.w;
}

extern "C" rt_status rt_philox_dev(uint64_t key, const uint32_t* d_ctr, int64_t n, uint32_t* d_out,
                                   void* stream) {
  if (!d_ctr || !d_out) return fail(RT_E_ARG, "null pointer");
  if (n < 1) return fail(RT_E_ARG, "n must be >= 1");
  philox_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      rtk::make_round_keys(key), d_ctr, n, d_out);
  RT_CUDA(cudaGetLastError());
  return RT_OK;
}

// ---------------------------------------------------------------------------
// NEXT row f1: PDD downstream (pdd.cuh)
static rt_status check_pdd(const rt_handle* h, const rt_pdd_cfg* c) {
  if (!c) return fail(RT_E_ARG, "null cfg");
  if (h) {
    if (h->p.dim != 2) return fail(RT_E_ARG, "PDD is implemented for dim = 2");
    if (h->p.strategy != RT_STRATEGY_POTENTIAL) return fail(RT_E_ARG, "PDD needs RT_STRATEGY_POTENTIAL");
    for (int k = 0; k <= 8; ++k)
      if (h->p.coef_kind[k] != RT_COEF_CONST) return fail(RT_E_ARG, "PDD needs constant coefficients");
  }
  if (!is_fin(c->lo) || !is_fin(c->hi) || !(c->hi > c->lo)) return fail(RT_E_ARG, "need lo < hi");
  if (!(c->T > 0.0) || !is_fin(c->T)) return fail(RT_E_ARG, "T must be > 0");
  if (c->n_cells < 4 || c->n_cells > 1020 || (c->n_cells & 1))
    return fail(RT_E_ARG, "n_cells must be even in [4, 1020]");
  if (c->n_steps < 1) return fail(RT_E_ARG, "n_steps must be >= 1");
  if (c->n_s < 4 || c->n_s > rtk::kPddMaxNodes || c->n_t < 4 || c->n_t > rtk::kPddMaxNodes)
    return fail(RT_E_ARG, "n_s and n_t must be in [4, %d]", rtk::kPddMaxNodes);
  if (c->boundary != 0 && c->boundary != 1) return fail(RT_E_ARG, "boundary must be 0 or 1");
  const int m = c->n_cells / 2;
  if (rtk::pdd_smem_bytes(m) > 227 * 1024) return fail(RT_E_ARG, "n_cells too large for shared memory");
  return RT_OK;
}

static rtk::PddGeom pdd_geom(const rt_pdd_cfg* c) {
  rtk::PddGeom G;
  G.lo = c->lo; G.hi = c->hi; G.n = c->n_cells; G.m = c->n_cells / 2;
  G.h = (c->hi - c->lo) / c->n_cells; G.T = c->T; G.n_steps = c->n_steps;
  G.dt = c->T / c->n_steps; G.ns = c->n_s; G.nt = c->n_t;
  return G;
}

static rtk::PddEq pdd_eq(const rt_eq_params& p) {
  rtk::PddEq E;
  for (int k = 0; k < 9; ++k) E.b[k] = (k <= p.degree) ? p.b[k] : 0.0;
  E.degree = p.degree; E.init_kind = p.init_kind; E.amp = p.init_amp;
  E.inv_scale = 1.0 / p.init_scale; E.inv_scale2 = 1.0 / (p.init_scale * p.init_scale); E.D = p.D;
  return E;
}

extern "C" rt_status rt_pdd_nodes(const rt_pdd_cfg* cfg, double* out) {
  rt_status s = check_pdd(nullptr, cfg);
  if (s != RT_OK) return s;
  if (!out) return fail(RT_E_ARG, "null pointer");
  const double mid = 0.5 * (cfg->lo + cfg->hi);
  for (int line = 0; line < 6; ++line)
    for (int j = 0; j < cfg->n_s; ++j) {
      const double sj = lin(cfg->lo, cfg->hi, cfg->n_s, j);
      double x = 0.0, y = 0.0;
      switch (line) {
        case 0: x = mid; y = sj; break;
        case 1: x = sj; y = mid; break;
        case 2: x = cfg->lo; y = sj; break;
        case 3: x = cfg->hi; y = sj; break;
        case 4: x = sj; y = cfg->lo; break;
        default: x = sj; y = cfg->hi; break;
      }
      out[(line * cfg->n_s + j) * 2 + 0] = x;
      out[(line * cfg->n_s + j) * 2 + 1] = y;
    }
  return RT_OK;
}

static rt_status pdd_downstream(rt_handle* h, const rt_pdd_cfg* cfg, const double* d_nodal,
                                double* d_field, double* d_bc, cudaStream_t st) {
  {
    const rt_status o = order_after_last(h, st);
    if (o != RT_OK) return o;
  }
  const rtk::PddGeom G = pdd_geom(cfg);
  double* bc = d_bc;
  if (!bc) {
    RT_CUDA(h->pdd_bc.ensure(static_cast<size_t>(6) * (G.n_steps + 1) * (G.n + 1) * sizeof(double)));
    bc = static_cast<double*>(h->pdd_bc.p);
  }
  // spline scratch: Ms [6][nt][ns], A and At [6][nt][n+1]
  RT_CUDA(h->pdd_spl.ensure((static_cast<size_t>(6) * G.nt * G.ns +
                             static_cast<size_t>(12) * G.nt * (G.n + 1)) * sizeof(double)));
  double* Ms = static_cast<double*>(h->pdd_spl.p);
  double* A = Ms + static_cast<size_t>(6) * G.nt * G.ns;
  double* At = A + static_cast<size_t>(6) * G.nt * (G.n + 1);
  rtk::pdd_spline_s_kernel<<<(6 * G.nt + 63) / 64, 64, 0, st>>>(d_nodal, Ms, G, 6);
  RT_CUDA(cudaGetLastError());
  const int nthr = 6 * (G.n + 1);
  rtk::pdd_spline_t_kernel<<<(nthr + 127) / 128, 128, 0, st>>>(d_nodal, Ms, A, At, bc, G, 6);
  RT_CUDA(cudaGetLastError());
  RT_CUDA(cudaEventRecord(h->ev[3], st));
  if (G.m - 1 <= 64 && h->pdd_cluster) {
    // a thread-block cluster of kPddCluster CTAs per subdomain (pdd.cuh)
    const int smem = rtk::pdd_cluster_smem_bytes(G.m);
    RT_CUDA(cudaFuncSetAttribute((const void*)rtk::pdd_adi_cluster_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(4 * rtk::kPddCluster);
    // (the four edges' W values are loaded one per thread: >= 4 (m+1) threads)
    lc.blockDim = dim3(std::max(256, (4 * (G.m + 1) + 31) / 32 * 32));
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = rtk::kPddCluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    RT_CUDA(cudaLaunchKernelEx(&lc, rtk::pdd_adi_cluster_kernel, static_cast<const double*>(bc), d_field,
                               G, pdd_eq(h->p)));
    return RT_OK;
  }
  const int smem = rtk::pdd_smem_bytes(G.m);
  RT_CUDA(cudaFuncSetAttribute((const void*)rtk::pdd_adi_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  // the pointwise reaction spreads over many threads; the line sweeps use m-1 of them
  // (at most 512: 1024 threads x 64 registers exceed the register file)
  const int threads = std::min(512, std::max(256, ((G.m + 1) * (G.m + 1) / 4 + 31) / 32 * 32));
  rtk::pdd_adi_kernel<<<4, threads, smem, st>>>(bc, d_field, G, pdd_eq(h->p));
  RT_CUDA(cudaGetLastError());
  return RT_OK;
}

extern "C" rt_status rt_pdd_downstream_dev(rt_handle* h, const rt_pdd_cfg* cfg,
                                           const double* d_nodal, double* d_field, double* d_bc,
                                           void* stream) {
  if (!h) return fail(RT_E_ARG, "null handle");
  rt_status s = check_pdd(h, cfg);
  if (s != RT_OK) return s;
  if (!d_nodal || !d_field) return fail(RT_E_ARG, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  s = pdd_downstream(h, cfg, d_nodal, d_field, d_bc, st);
  if (s != RT_OK) return s;
  RT_CUDA(cudaEventRecord(h->ev[2], st));
  mark_scratch(h, st);
  return RT_OK;
}

// t_0 nodal values: g at the nodal points (no Monte Carlo at t = 0)
__global__ void pdd_init_kernel(const double* __restrict__ pts, double* __restrict__ V, int ns,
                                int nt, rtk::PddEq E) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= 6 * ns) return;
  const int line = q / ns, j = q - line * ns;
  V[(static_cast<int64_t>(line) * nt + 0) * ns + j] = rtk::pdd_g(E, pts[2 * q], pts[2 * q + 1]);
}

extern "C" rt_status rt_pdd_solve(rt_handle* h, const rt_pdd_cfg* cfg, double* out_field,
                                  double* out_nodal, double* out_ms) {
  if (!h) return fail(RT_E_ARG, "null handle");
  rt_status s = check_pdd(h, cfg);
  if (s != RT_OK) return s;
  if (!out_field) return fail(RT_E_ARG, "null pointer");
  const int K = h->p.K;
  s = check_pade_args(1, K, cfg->L, cfg->M);
  if (s != RT_OK) return s;
  const int ns = cfg->n_s, nt = cfg->n_t, n1 = cfg->n_cells + 1;
  const int lines_mc = cfg->boundary ? 6 : 2;
  const int64_t npts = static_cast<int64_t>(lines_mc) * ns;
  s = check_run_args(h, npts, cfg->T, 0, cfg->n_trees);
  if (s != RT_OK) return s;
  cudaStream_t st = h->own_stream;
  std::vector<double> pts(6 * ns * 2);
  rt_pdd_nodes(cfg, pts.data());
  RT_CUDA(h->pdd_pts.ensure(pts.size() * sizeof(double)));
  RT_CUDA(h->pdd_nodal.ensure(static_cast<size_t>(6) * nt * ns * sizeof(double)));
  RT_CUDA(h->pdd_field.ensure(static_cast<size_t>(n1) * n1 * sizeof(double)));
  RT_CUDA(h->pdd_c.ensure(static_cast<size_t>(npts) * (K + 1) * sizeof(double)));
  RT_CUDA(h->pdd_u.ensure(static_cast<size_t>(npts) * sizeof(double)));
  RT_CUDA(h->sums.ensure(static_cast<size_t>(npts) * (K + 2) * 3 * sizeof(double)));
  double* d_pts = static_cast<double*>(h->pdd_pts.p);
  double* V = static_cast<double*>(h->pdd_nodal.p);
  double* dc = static_cast<double*>(h->pdd_c.p);
  double* du = static_cast<double*>(h->pdd_u.p);
  double* sums = static_cast<double*>(h->sums.p);
  RT_CUDA(cudaMemcpyAsync(d_pts, pts.data(), pts.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  RT_CUDA(cudaMemsetAsync(V, 0, static_cast<size_t>(6) * nt * ns * sizeof(double), st));
  // phase events, released on every exit path
  struct Events {
    cudaEvent_t e[2] = {nullptr, nullptr};
    ~Events() { for (cudaEvent_t x : e) if (x) cudaEventDestroy(x); }
  } ev;
  RT_CUDA(cudaEventCreate(&ev.e[0]));
  RT_CUDA(cudaEventCreate(&ev.e[1]));
  cudaEvent_t e0 = ev.e[0], e1 = ev.e[1];
  RT_CUDA(cudaEventRecord(e0, st));
  pdd_init_kernel<<<(6 * ns + 127) / 128, 128, 0, st>>>(d_pts, V, ns, nt, pdd_eq(h->p));
  RT_CUDA(cudaGetLastError());
  // probabilistic part: the interface (and edge) values at
  // every time level t_k > 0 by the tree walk, resummed by [L/M] Padé
  for (int k = 1; k < nt; ++k) {
    const double tk = cfg->T * (static_cast<double>(k) / (nt - 1));
    const uint64_t seed_k = cfg->seed + static_cast<uint64_t>(k) * 0x9E3779B97F4A7C15ull;
    s = run_walk(h, d_pts, npts, tk, 0, cfg->n_trees, seed_k, 0, nullptr, sums, st);
    if (s != RT_OK) return s;
    finalize_kernel<<<static_cast<unsigned>(npts), 32, 0, st>>>(
        sums, K, static_cast<double>(cfg->n_trees), dc, nullptr, nullptr, nullptr);
    // (a degenerate table — e.g. no tree reaching L splits at an early level —
    // falls back to the largest regular [L/M'], finite; pade.cuh bit0)
    launch_pade(dc, npts, K, cfg->L, cfg->M, nullptr, du, nullptr, st);
    RT_CUDA(cudaGetLastError());
    // du [line][j] -> V[line][k][j]
    RT_CUDA(cudaMemcpy2DAsync(V + static_cast<size_t>(k) * ns, static_cast<size_t>(nt) * ns * 8, du,
                              static_cast<size_t>(ns) * 8, static_cast<size_t>(ns) * 8, lines_mc,
                              cudaMemcpyDeviceToDevice, st));
  }
  RT_CUDA(cudaEventRecord(e1, st));
  // outer edges with zero Dirichlet data: lines 2..5 stay 0 at every level
  if (!cfg->boundary)
    RT_CUDA(cudaMemsetAsync(V + static_cast<size_t>(2) * nt * ns, 0,
                            static_cast<size_t>(4) * nt * ns * sizeof(double), st));
  double* F = static_cast<double*>(h->pdd_field.p);
  s = pdd_downstream(h, cfg, V, F, nullptr, st);
  if (s != RT_OK) return s;
  RT_CUDA(cudaEventRecord(h->ev[2], st));
  RT_CUDA(cudaMemcpyAsync(out_field, F, static_cast<size_t>(n1) * n1 * sizeof(double),
                          cudaMemcpyDeviceToHost, st));
  std::vector<double> nodal(static_cast<size_t>(6) * nt * ns);
  RT_CUDA(cudaMemcpyAsync(nodal.data(), V, nodal.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  RT_CUDA(cudaStreamSynchronize(st));
  if (out_nodal) std::memcpy(out_nodal, nodal.data(), nodal.size() * sizeof(double));
  // the spline and the subdomain solves would spread a non-finite nodal
  // value over the whole field: refuse it
  for (size_t q = 0; q < nodal.size(); ++q)
    if (!is_fin(nodal[q]))
      return fail(RT_E_NUMERIC, "rt_pdd_solve: nodal value %zu (line %zu, level %zu) is not finite",
                  q, q / (static_cast<size_t>(nt) * ns), (q / ns) % nt);
  if (out_ms) {
    float a = 0.f, b = 0.f, c = 0.f;
    RT_CUDA(cudaEventElapsedTime(&a, e0, e1));
    RT_CUDA(cudaEventElapsedTime(&b, e1, h->ev[3]));
    RT_CUDA(cudaEventElapsedTime(&c, h->ev[3], h->ev[2]));
    out_ms[0] = a; out_ms[1] = b; out_ms[2] = c;
  }
  return RT_OK;
}

// ---------------------------------------------------------------------------
// K0: measured FP64 FMA throughput of this GPU — the measured
// companion of the nominal FP64 roofline (148 SMs x 64 lanes x clock).  Every
// thread runs 8 independent DFMA chains (enough ILP to saturate the pipe at
// full occupancy); one DFMA = one FP64 lane-op, the unit of bench.py's roofline.
__global__ void __launch_bounds__(256) fp64_peak_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1.0, x2 = x0 + 2.0, x3 = x0 + 3.0;
  double x4 = x0 + 4.0, x5 = x0 + 5.0, x6 = x0 + 6.0, x7 = x0 + 7.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == 1.2345) out[0] = s;   // keep the chains alive
}

extern "C" rt_status rt_fp64_peak(double* out_lane_ops_per_s, double* out_ms) {
  if (!out_lane_ops_per_s) return fail(RT_E_ARG, "null pointer");
  int dev = 0, nsm = 0;
  RT_CUDA(cudaGetDevice(&dev));
  RT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  double* d = nullptr;
  RT_CUDA(cudaMalloc(&d, sizeof(double)));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
    cudaFree(d);
    return fail(RT_E_CUDA, "rt_fp64_peak: event creation failed");
  }
  const int blocks = nsm * 8, threads = 256, iters = 4096;
  fp64_peak_kernel<<<blocks, threads>>>(d, 64, 0.999999, 1e-7);   // warm-up
  cudaEventRecord(e0);
  fp64_peak_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (e != cudaSuccess) return fail(RT_E_CUDA, "rt_fp64_peak: %s", cudaGetErrorString(e));
  const double ops = static_cast<double>(blocks) * threads * iters * 16.0 * 8.0;
  *out_lane_ops_per_s = ops / (ms * 1e-3);
  if (out_ms) *out_ms = ms;
  return RT_OK;
}
