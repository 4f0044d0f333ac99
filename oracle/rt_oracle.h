/* rt_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU oracle of the random-tree Monte Carlo
 * estimator of arXiv:2402.06491 (Acebrón & Rodríguez-Rozas), Strategy A
 * (PAPER.md:159-301), with order binning and [L/M] Padé resummation
 * (PAPER.md:295-301, 744-780).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * code, header, table or constant generator with the CUDA product
 * (paper_2402_06491_b200/), and the product never loads it.
 *
 * Every function states the passage it follows; the numerical contract
 * (the readings of the paper where it is silent) is DESIGN.md §2.
 */
#ifndef RT_ORACLE_H
#define RT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t dim;          /* 1..3 */
  double  D;            /* u_t = D Δu + f(u) */
  int32_t degree;       /* m */
  double  b[9];         /* f(u) = Σ_k b[k] u^k */
  double  lambda;       /* clock rate; <= 0 -> default */
  int32_t offspring;    /* 0: p_k ∝ |a_k|, 1: uniform on the support */
  int32_t init_kind;    /* 0 const, 1 tanh step, 2 gauss, 3 lorentz */
  double  init_amp;
  double  init_scale;
  int32_t K;            /* orders 0..K kept */
  int32_t precision;    /* ignored by the oracle (FP64 throughout) */
  /* --- NEXT rows f2/f3 --------------------------------- */
  int32_t strategy;     /* 0: exponential clock with the potential -λu (default);
                           1: Strategy A with the shift u = v e^{λt};
                           2: Strategy B, Bernoulli leaves + uniform split times
                               */
  double  q;            /* Strategy B: P(ξ = 0) = probability a particle is a leaf */
  int32_t coef_kind[9]; /* per power k: 0 b_k constant; 1 b_k e^{-x_a²/s²}/(t + t0)
                           (Example 5) */
  int32_t coef_axis;    /* a */
  double  coef_scale;   /* s > 0 */
  double  coef_t0;      /* t0 > 0 */
  int32_t shared;       /* 1: shared trees (NEXT row f4): the random numbers omit
                           the node index, every node sees the same trees, node
                           i's leaves are evaluated at x_i + δ (δ the leaf's
                           displacement from the root); constant coefficients */
  int32_t sampling;     /* Strategy A only.  0: the contract (R29: one
                           Gamma(m+1) variate split by uniform spacings into the
                           clock and the Box–Muller radii, 32-bit uniforms).
                           1: TEXTBOOK sampling, a pin of R29 in law only
                           (tests/test_oracle_sampling.py): S = -ln(u)/λ with
                           u = unif53(call-0 w1:w0), Box–Muller r = sqrt(-2 ln v1),
                           angle 2π v2 from the unif53 pair of call 1 (call 2
                           for the third normal, d = 3) — SURVEY.md §8(c)'s
                           original definition.  Never the product's contract. */
} or_params;

typedef struct {
  double   lambda, inv_lambda, sigma;
  double   a[9];
  int32_t  n_support;
  int32_t  support[9];     /* k values, ascending */
  uint64_t thresh[9];      /* integer thresholds T_k (last = 2^32) */
  double   p_hat[9];       /* effective probabilities */
  double   w[9];           /* weights a_k / (λ p̂_k); Strategy B: a_k / ((1 - q̂) p̂_k) */
  int32_t  beta;           /* bits per child digit in labels */
  uint64_t tq;             /* Strategy B: leaf iff 32-bit draw < tq (q̂ = tq / 2^32) */
  double   q_hat;          /* Strategy B: effective leaf probability */
} or_norm;

typedef struct {
  int32_t ne;         /* splitting events (order bin) */
  int32_t leaves;     /* g evaluations */
  int32_t particles;  /* particles processed */
  int32_t pruned;     /* 1 if Ne > K (aborted) */
  double  C;          /* tree contribution (0 if pruned) */
} or_tree_rec;

typedef struct { int64_t trees, pruned, particles, leaves, splits; } or_stats;

/* Philox4x32-10 block: out = philox(key, ctr). */
void or_philox(const uint32_t key[2], const uint32_t ctr[4], uint32_t out[4]);
/* (2*(x>>12)+1) * 2^-53 */
double or_unif53(uint32_t lo, uint32_t hi);
/* (2w+1) * 2^-33 */
double or_unif32(uint32_t w);

int or_normalize(const or_params* p, or_norm* out);   /* 0 ok, else error */

/* One tree at node x (node index i), tree index j. */
int or_tree(const or_params* p, const double* x, int64_t i, int64_t j, double t,
            uint64_t seed, or_tree_rec* rec);

/* Records for trees j in [j0, j0+n_trees) of every node: rec[i*n_trees + (j-j0)]. */
int or_trees(const or_params* p, const double* points, int64_t n_points, double t,
             int64_t j0, int64_t n_trees, uint64_t seed, or_tree_rec* rec);

int or_trees_at(const or_params* p, const double* points, int64_t n_points, double t,
                const int64_t* js, int64_t n_js, uint64_t seed, or_tree_rec* rec);

/* Order-binned sums sums[(i*(K+2)+n)*3 + {0:ΣC, 1:ΣC², 2:count}] for n = 0..K+1
 * (n = K+1 counts pruned trees), over trees j in [j0, j0+n_trees). */
int or_sums(const or_params* p, const double* points, int64_t n_points, double t,
            int64_t j0, int64_t n_trees, uint64_t seed, double* sums, or_stats* st);

/* Per-order coefficients and standard errors from sums (N = total trees). */
void or_finalize(const double* sums, int64_t n_points, int32_t K, int64_t N,
                 double* coeffs, double* stderr_n, double* u_sum, double* se_sum);

/* [L/M] Padé of c[0..L+M] evaluated at z = 1; flags bit0 zero pivot in
 * [L/M] (the value is then [L/M'], M' < M the largest regular order, M' in
 * bits 8..15), bit1 |Q(1)| <= 1e-14 |P(1)|, bit2 Q changes sign on (0,1]. */
int or_pade(const double* c, int32_t L, int32_t M, double* u, uint32_t* flags,
            double* p_out, double* q_out);
/* or_pade plus bit3: |u - (c_0 + ... + c_K)| > 10 se_sum. */
int or_pade_node(const double* c, int32_t K, int32_t L, int32_t M, double se_sum,
                 double* u, uint32_t* flags);

#ifdef __cplusplus
}
#endif
#endif
