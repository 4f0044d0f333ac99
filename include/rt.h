/* rt.h — C ABI of the B200 (sm_100a) random-tree Monte Carlo library.
 *
 * The library estimates u(x,t) for the semilinear parabolic Cauchy problem
 *
 *     u_t = D Δu + f(u),  x ∈ R^d,  u(x,0) = g(x),  f(u) = Σ_{k=0}^{m} b_k u^k
 *
 * (arXiv:2402.06491, Eq. nonlinear_new, constant-coefficient
 * case) at a set of nodes, e.g. the interface nodes of a probabilistic domain
 * decomposition.  Each Monte Carlo sample is a generalized
 * random tree (Strategy A): particles live for exponential
 * times, branch into k offspring with weight a_k/(λ p_k), move by Brownian
 * increments, and the tree contributes the product of g over its leaves times
 * its weights (Eq. rep_strategyB), binned by its number of
 * splitting events Ne (Eq. recursion).  The per-order series
 * is resummed per node by an [L/M] Padé approximant at z = 1
 * (PAPER.md:295-301, 744-780).  The numerical contract (RNG layout, order
 * bins, prune rule, standard errors, Padé flags) is DESIGN.md §2.
 *
 * Conventions for every entry point:
 *   - Return value: rt_status; RT_OK = 0.  On failure rt_last_error() returns
 *     a thread-local, NUL-terminated message (valid until the next call on the
 *     same thread).  Output buffers are unspecified after a failure.
 *   - The caller owns every input and output buffer.  rt_create copies the
 *     parameters; the handle owns its device scratch (grown lazily, freed by
 *     rt_destroy).  A handle must not be used from two threads at once, and
 *     its "_dev" calls share that scratch (task partials, lane-private bin
 *     sums, overflow stacks): calls on different streams must be ordered by
 *     the caller — use one handle per concurrently running stream.
 *   - "host" pointers are ordinary CPU memory; such calls are synchronous.
 *     "_dev" entry points take device pointers and a cudaStream_t (as void*;
 *     NULL = legacy default stream), are stream-ordered and do not
 *     synchronize.
 *   - Layouts are row-major, FP64 unless stated: points [n_points × dim];
 *     coefficients / standard errors [n_points × (K+1)].
 *   - Results are a pure function of (parameters, points, t, tree range,
 *     seed) and the launch geometry; with a fixed geometry they are bitwise
 *     reproducible run to run, and tree j of node i is the same tree whatever
 *     range or geometry computes it (counter-based RNG).
 *   - Diagnostic environment switches (tests only; none changes a result):
 *     RT_FORCE_GEN=1 (read by rt_create) selects the general tree-walk kernel
 *     where the specialised one would run; RT_PDD_CLUSTER=0 (rt_create) the
 *     single-CTA PDD local solver; RT_WARP_TIMES=<file> appends per-warp
 *     start/end times of every tree-walk launch to <file>.
 */
#ifndef RT_H
#define RT_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RT_OK = 0,
  RT_E_ARG = 1,     /* invalid argument (null pointer, out-of-range value) */
  RT_E_CUDA = 2,    /* CUDA runtime error (message in rt_last_error)        */
  RT_E_NOMEM = 3,   /* device allocation failed                            */
  RT_E_STATE = 4,   /* handle state error                                  */
  RT_E_NUMERIC = 5  /* a result is not finite (rt_pdd_solve's nodal values) */
} rt_status;

/* Offspring law for the branching power α. */
typedef enum {
  RT_OFFSPRING_ABS = 0,     /* p_k ∝ |a_k| on the support (R2, default) */
  RT_OFFSPRING_UNIFORM = 1  /* uniform on the support, the paper's rule P:222     */
} rt_offspring;

/* Initial data g (u(x,0) = g(x)). */
typedef enum {
  RT_G_CONST = 0,      /* g = amp                                   */
  RT_G_TANH_STEP = 1,  /* g = amp * 0.5 * (1 + tanh(x_1 / scale))   */
  RT_G_GAUSS = 2,      /* g = amp * exp(-|x|^2 / scale^2)           */
  RT_G_LORENTZ = 3     /* g = amp / (1 + |x|^2 / scale^2)           */
} rt_init;

/* How a tree samples the Duhamel form of the PDE:
 *  RT_STRATEGY_POTENTIAL: f = −λu + Σ a_k u^k, exponential clock of rate λ,
 *    weights a_k/(λ p_k) (the hot path's default);
 *  RT_STRATEGY_A_SHIFT:   Strategy A with u = v e^{λt}:
 *    weights b_k e^{(k−1)λτ_c}/(λ p_k) at a split whose children have
 *    horizon τ_c, e^{λt} per tree;
 *  RT_STRATEGY_B:         Strategy B: a particle is a leaf
 *    with probability q (weight g/q), else splits after the uniform fraction S
 *    of its horizon τ with weight τ b_k/((1−q) p_k), children horizon τ(1−S). */
typedef enum { RT_STRATEGY_POTENTIAL = 0, RT_STRATEGY_A_SHIFT = 1, RT_STRATEGY_B = 2 } rt_strategy;

/* Coefficient of u^k: constant b_k, or b_k e^{−x_a²/s²}/(t + t0) evaluated at
 * the split position and the children's time argument τ_c (Example 5,
 * PAPER.md:1084-1088).  Not allowed on k = 1 with RT_STRATEGY_POTENTIAL. */
typedef enum { RT_COEF_CONST = 0, RT_COEF_GAUSS_RATIONAL = 1 } rt_coef;

typedef enum {
  RT_PREC_FP64 = 0,       /* everything FP64                                     */
  RT_PREC_FP32_POS = 1    /* FP32 positions, increments and g; FP64 clock, weights,
                             tree product and sums (cfg5 variant) */
} rt_precision;

typedef struct {
  int32_t dim;          /* d ∈ {1,2,3}                                             */
  double  D;            /* diffusion > 0; Brownian σ = sqrt(2D) (R5)     */
  int32_t degree;       /* m ∈ [0, 8]                                              */
  double  b[9];         /* f(u) = Σ_{k=0}^{m} b[k] u^k; b[k>m] ignored             */
  double  lambda;       /* clock rate λ; <= 0 selects -b[1] if b[1] < 0, else 1    */
  int32_t offspring;    /* rt_offspring                                            */
  int32_t init_kind;    /* rt_init                                                 */
  double  init_amp;     /* amp of g                                                */
  double  init_scale;   /* scale of g (> 0)                                        */
  int32_t K;            /* orders 0..K are kept; trees with Ne > K are pruned.     */
                        /* 0 <= K <= 30 and 1 + K*β <= 56 (β = child-digit bits)   */
  int32_t precision;    /* rt_precision                                            */
  /* --- NEXT rows f2 / f3; zero-initialised = the default path --- */
  int32_t strategy;     /* rt_strategy                                             */
  double  q;            /* RT_STRATEGY_B: P(leaf) = P(ξ = 0), 0 < q < 1             */
  int32_t coef_kind[9]; /* per power k: rt_coef (variable c_k(x,t))  */
  int32_t coef_axis;    /* a: the coordinate of the variable factor                */
  double  coef_scale;   /* s > 0                                                   */
  double  coef_t0;      /* t0 > 0                                                  */
  int32_t shared;       /* 1: shared trees (NEXT row f4): the random  */
                        /* numbers omit the node index, every node sees the same   */
                        /* trees, leaves evaluated at x_i + δ; unbiased per node,  */
                        /* correlated across nodes; constant coefficients, FP64    */
} rt_eq_params;

typedef struct {
  int64_t trees;        /* trees sampled (kept + pruned)                 */
  int64_t pruned;       /* trees with Ne > K                             */
  int64_t particles;    /* particle lifetimes simulated (= leaves + splits) */
  int64_t leaves;       /* g evaluations                                 */
  int64_t splits;       /* splitting events (incl. the aborting one)     */
  double  kernel_ms;    /* tree-walk kernel time of the last estimate    */
  double  total_ms;     /* whole call (host API) or all kernels (_dev)   */
} rt_stats;

/* A plane x_axis = value carrying an n_per_dim^(d-1) grid over [lo, hi] in
 * every free axis (PDD artificial interfaces). */
typedef struct {
  int32_t axis;
  double  value;
  double  lo, hi;
  int32_t n_per_dim;
} rt_plane;

/* Per-tree record (debug / parity): structure and contribution of one tree. */
typedef struct {
  int32_t ne;          /* splitting events (order bin); > K if pruned   */
  int32_t leaves;      /* g evaluations                                 */
  int32_t particles;   /* particles simulated                           */
  int32_t pruned;      /* 1 if Ne > K                                   */
  double  C;           /* Π weights × Π g (0 if pruned)                 */
} rt_tree_rec;

typedef struct rt_handle rt_handle;

/* Validate and normalise the equation (row a1: λ, a_k, support, integer
 * thresholds, weights) and allocate a handle.
 * RT_E_ARG on: null pointers, dim ∉ {1,2,3}, D <= 0 or non-finite, degree ∉
 * [0,8], non-finite b/λ/amp/scale, scale <= 0, K ∉ [0,30], label width
 * 1 + K*β > 56, a support category of zero integer width, an unknown enum,
 * an unknown precision, RT_STRATEGY_B with q ∉ (0,1) (or a zero-width integer
 * threshold), a variable coefficient with s <= 0, t0 <= 0, an axis outside
 * [0, dim), or on k = 1 under RT_STRATEGY_POTENTIAL, RT_PREC_FP32_POS with a
 * strategy other than RT_STRATEGY_POTENTIAL, shared ∉ {0, 1}, shared trees
 * with variable coefficients or RT_PREC_FP32_POS.  An empty support (purely linear f) is legal. */
rt_status rt_create(const rt_eq_params* params, rt_handle** out);

/* Free the handle and its device scratch.  NULL is a no-op. */
rt_status rt_destroy(rt_handle* h);

/* Host API (synchronous): copies points to the device, samples n_trees trees
 * per node, and copies back the per-order coefficients c_n = ΣC_n / N and
 * standard errors se_n = sqrt(max(0, ΣC_n²/N − c_n²)/(N−1)), n = 0..K, where
 * N = n_trees counts pruned trees (R4, R11).
 * RT_E_ARG on: null pointers, n_points < 1 or >= 2^31, t <= 0 or non-finite,
 * n_trees < 2 or >= 2^31 (per call; larger counts are split over calls with
 * rt_sums_dev's tree_offset), non-finite points.  Times the copies inside
 * rt_stats.total_ms.
 * Tree j of node i draws Philox4x32-10 blocks keyed by (seed; j, i, particle
 * label, call), mapped to its clock and Gaussian increments as DESIGN.md R29
 * (Strategy A: one Gamma variate split into the clock and the Box-Muller
 * radii) or R8 (Strategy B) specify: results are reproducible bit for bit
 * across runs and launch grids. */
rt_status rt_estimate(rt_handle* h, const double* points, int64_t n_points, double t,
                      int64_t n_trees, uint64_t seed,
                      double* out_coeffs, double* out_stderr);

/* Device API of rt_estimate: d_points [n_points × dim] device, outputs device
 * [n_points × (K+1)]; stream-ordered on `stream`. */
rt_status rt_estimate_dev(rt_handle* h, const double* d_points, int64_t n_points, double t,
                          int64_t n_trees, uint64_t seed,
                          double* d_out_coeffs, double* d_out_stderr, void* stream);

/* Raw order-binned sums for trees j ∈ [tree_offset, tree_offset + n_trees):
 * d_sums [n_points × (K+2) × 3] = (ΣC, ΣC², count) per order n = 0..K, and at
 * n = K+1 the count of pruned trees.  Sums of disjoint tree ranges add, which
 * is how ranks / calls are merged.  tree_offset + n_trees <= 2^32. */
rt_status rt_sums_dev(rt_handle* h, const double* d_points, int64_t n_points, double t,
                      int64_t tree_offset, int64_t n_trees, uint64_t seed,
                      double* d_sums, void* stream);

/* c_n, se_n (as rt_estimate) and the partial sum u_sum = Σ_n c_n with its
 * standard error se_sum from d_sums of N_total trees.  Any output may be NULL. */
rt_status rt_finalize_dev(const double* d_sums, int64_t n_points, int32_t K, int64_t N_total,
                          double* d_coeffs, double* d_stderr, double* d_u_sum,
                          double* d_se_sum, void* stream);

/* [L/M] Padé at z = 1 of each node's c_0..c_{L+M} (row stride K+1):
 * Q(0) = 1, deg P <= L, deg Q <= M, Q Σc_n z^n − P = O(z^{L+M+1}), denominator
 * by Gaussian elimination with partial pivoting.
 * out_u [n_points]; out_flags [n_points] (may be NULL):
 *   bit0  exact zero pivot in [L/M] (degenerate table): u is the value of the
 *         largest regular [L/M'], M' < M — [L/0] = c_0+…+c_L always is —
 *         SPEC.md:403's fallback; M' is stored in bits 8..15;
 *   bit1  |Q(1)| <= 1e-14 |P(1)|;
 *   bit2  Q has a sign change on (0, 1] (256 equispaced points);
 *   bit3  |u − Σ_{n=0}^{K} c_n| > 10 se_sum[i] — the resummed value and the
 *         partial sum disagree beyond the statistics;
 *         only when se_sum [n_points] (the standard error of the partial sum,
 *         rt_finalize_dev's d_se_sum) is given, else never set.
 * u is NaN only for non-finite coefficients.  One warp per node, all in
 * registers.  RT_E_ARG: null coeffs/out_u, n_points < 1, L < 0, M < 0,
 * M > 16, L + M > K, K > 30.  Host variant synchronous; _dev stream-ordered. */
rt_status rt_pade(const double* coeffs, int64_t n_points, int32_t K, int32_t L, int32_t M,
                  const double* se_sum, double* out_u, uint32_t* out_flags);
rt_status rt_pade_dev(const double* d_coeffs, int64_t n_points, int32_t K, int32_t L,
                      int32_t M, const double* d_se_sum, double* d_u, uint32_t* d_flags,
                      void* stream);

/* Row a9: place nodes on planes (plane-major; free axes row-major ascending;
 * linspace(lo, hi, n) = lo + (hi−lo)·(j/(n−1)); exact duplicates of earlier
 * points skipped; at most max_points kept), then estimate and resum them.
 * Host buffers: out_points [max_points × dim], out_u, out_stderr (se of the
 * partial sum, R11), out_flags [max_points]; *out_n_points = count. */
rt_status rt_interface_values(rt_handle* h, const rt_plane* planes, int32_t n_planes,
                              int64_t max_points, double t, int64_t n_trees, uint64_t seed,
                              int32_t L, int32_t M, double* out_points, double* out_u,
                              double* out_stderr, uint32_t* out_flags,
                              int64_t* out_n_points);

/* Per-tree records of the production kernel (parity / debugging): for trees
 * j = tree_offset + s·2^rec_shift (s = 0, 1, …) within [tree_offset,
 * tree_offset + n_trees) of every node, d_recs[i * n_rec + s] with
 * n_rec = ceil(n_trees / 2^rec_shift).  The sampled launch is otherwise the
 * estimate launch; d_sums (may be NULL) receives its sums. */
rt_status rt_trace_dev(rt_handle* h, const double* d_points, int64_t n_points, double t,
                       int64_t tree_offset, int64_t n_trees, uint64_t seed, int32_t rec_shift,
                       rt_tree_rec* d_recs, double* d_sums, void* stream);

/* Counters of the last estimate / sums / trace on this handle. */
rt_status rt_get_stats(const rt_handle* h, rt_stats* out);

/* Launch geometry override (0 = automatic): CTAs of the tree-walk kernel
 * and trees per task; in shared-tree mode (rt_eq_params.shared) the second
 * value instead caps the trees per chunk (one phase-1 + phase-2 pass each,
 * DESIGN.md §12).  Changes only summation order. */
rt_status rt_set_launch(rt_handle* h, int32_t grid_ctas, int64_t trees_per_task);

/* Stack-pool override (0 = automatic): at most pool_entries pending sibling
 * groups per warp are kept in shared memory, the rest in the global overflow
 * area.  Changes neither results nor summation order; tests use
 * it to exercise the overflow path.  RT_E_ARG: null handle, pool_entries < 0. */
rt_status rt_set_pool(rt_handle* h, int32_t pool_entries);

/* The library's Philox4x32-10 block function on device buffers:
 * d_out[4q..4q+3] = philox(key, d_ctr[4q..4q+3]), q < n (RNG parity tests). */
rt_status rt_philox_dev(uint64_t key, const uint32_t* d_ctr, int64_t n, uint32_t* d_out,
                        void* stream);

/* ------------------------------------------------------------------------
 * NEXT row f1 — probabilistic domain decomposition downstream (PAPER.md:936-950,
 * 1007-1012), d = 2 with constant coefficients: the square
 * [lo, hi]² is cut by the artificial interfaces x = mid and y = mid
 * (mid = (lo+hi)/2) into four subdomains.  Six lines carry nodal points s_j =
 * lo + j (hi−lo)/(n_s−1) at time levels t_k = k T/(n_t−1): 0 interface x = mid
 * (points (mid, s_j)), 1 interface y = mid ((s_j, mid)), 2 edge x = lo,
 * 3 edge x = hi ((lo|hi, s_j)), 4 edge y = lo, 5 edge y = hi ((s_j, lo|hi)).
 * Their values (t_0: g; t_k > 0: the tree walk + Padé) are interpolated by
 * not-a-knot tensor splines in (s, t) and used as Dirichlet data of four
 * decoupled Crank–Nicolson (Peaceman–Rachford ADI, Strang-split RK4 reaction)
 * solves on the grid x_i = lo + i h, h = (hi−lo)/n_cells.  Fields are
 * [(n_cells+1)²] row-major in x: F[i (n_cells+1) + j] = u(x_i, y_j, T). */
typedef struct {
  double   lo, hi;      /* square domain [lo, hi]²                                 */
  double   T;           /* final time > 0                                          */
  int32_t  n_cells;     /* grid cells per side, even, 4 <= n_cells <= 1020          */
  int32_t  n_steps;     /* time steps, Δt = T / n_steps                            */
  int32_t  n_s, n_t;    /* nodal points per line / time levels, 4 <= n <= 64        */
  int32_t  boundary;    /* 0: zero Dirichlet on the outer edges; 1: probabilistic   */
                        /* values there too                    */
  int32_t  L, M;        /* Padé order of the nodal values (L + M <= K)             */
  int64_t  n_trees;     /* trees per nodal point and time level                    */
  uint64_t seed;        /* time level k uses seed + k·0x9E3779B97F4A7C15           */
} rt_pdd_cfg;

/* Nodal point coordinates [6][n_s][2] (host buffer) of the layout above. */
rt_status rt_pdd_nodes(const rt_pdd_cfg* cfg, double* out_points);

/* Downstream only, stream-ordered on device buffers: d_nodal [6][n_t][n_s]
 * nodal values → d_field [(n_cells+1)²].  d_bc (may be NULL) receives the
 * boundary tables [6][n_steps+1][n_cells+1] (spline values at (x_i, t_n)).
 * RT_E_ARG: bad geometry (see rt_pdd_cfg), dim != 2, a strategy other than
 * RT_STRATEGY_POTENTIAL or variable coefficients, null pointers. */
rt_status rt_pdd_downstream_dev(rt_handle* h, const rt_pdd_cfg* cfg, const double* d_nodal,
                                double* d_field, double* d_bc, void* stream);

/* The whole PDD (synchronous, host buffers): nodal values by the tree walk,
 * splines, subdomain solves.  out_nodal [6][n_t][n_s] and out_ms[3] = {T_MC,
 * T_INT, T_LOCAL} (device time, ms) may be NULL.  A degenerate Padé table at
 * a nodal point falls back to a lower order (rt_pade bit0); RT_E_NUMERIC if a
 * nodal value is still not finite (the field is then not computed). */
rt_status rt_pdd_solve(rt_handle* h, const rt_pdd_cfg* cfg, double* out_field, double* out_nodal,
                       double* out_ms);

/* Measured FP64 FMA throughput of the current GPU (FP64 lane-ops/s; one
 * DFMA = one lane-op): 8 CTAs of 256 threads per SM, 8 independent DFMA
 * chains per thread, CUDA events around one launch.  The measured companion
 * of the nominal FP64 roofline.  out_ms may be NULL. */
rt_status rt_fp64_peak(double* out_lane_ops_per_s, double* out_ms);

/* Thread-local message of the last failure on this thread ("" if none). */
const char* rt_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* RT_H */
