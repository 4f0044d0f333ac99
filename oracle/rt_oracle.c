/* rt_oracle.c — TEST INFRASTRUCTURE ONLY (see rt_oracle.h).
 *
 * A plain, slow, single-threaded, obviously-correct CPU implementation of the
 * generalized random-tree representation of arXiv:2402.06491, Strategy A,
 * written from PAPER.md and the readings of DESIGN.md §2.  FP64 throughout,
 * compiled without fast-math and without FMA contraction.  The tree is walked
 * RECURSIVELY, exactly as the recursive expansion of Eq. (probexp2) is written
 * (PAPER.md:217-239): a particle either survives to the horizon and evaluates
 * g, or splits at its clock ring into α children whose values multiply.
 *
 * Parity pins (tests/test_oracle_pins.py) tie every function here to something
 * other than itself: Philox known-answer vectors and torch's philox engine,
 * the ODE closed form for spatially constant data, the exact per-order ODE
 * series, the heat kernel for linear f, the Poisson law of a k = 1 offspring,
 * the Yule law of Ne, finite differences in 1-D, SPEC's Padé fixtures and an
 * mpmath Padé.
 */
#include "rt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Random numbers.  The paper names no generator (PAPER.md is silent; DESIGN.md
 * reading R1): Philox4x32-10 (Salmon et al., SC'11), key = seed, counter =
 * (tree j, node i, particle label lo32, label hi24 | call << 24).           */
void or_philox(const uint32_t key[2], const uint32_t ctr[4], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Uniform in (0,1) from 64 random bits: (2*(x>>12)+1) * 2^-53 (exact). */
double or_unif53(uint32_t lo, uint32_t hi) {
  uint64_t x = ((uint64_t)hi << 32) | (uint64_t)lo;
  uint64_t m = 2u * (x >> 12) + 1u;
  return (double)m * 0x1.0p-53;
}

/* Uniform in (0,1) from 32 random bits: (2w+1) * 2^-33 (exact). */
double or_unif32(uint32_t w) {
  return (2.0 * (double)w + 1.0) * 0x1.0p-33;
}

static void draw(uint64_t seed, int64_t i, int64_t j, uint64_t label, uint32_t call,
                 uint32_t out[4]) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t ctr[4] = {(uint32_t)j, (uint32_t)i, (uint32_t)label,
                     (uint32_t)((label >> 32) & 0xFFFFFFu) | (call << 24)};
  or_philox(key, ctr, out);
}

/* ------------------------------------------------------------------------ */
/* Equation normalisation (row a1).  PAPER.md:90-101 (Eq. nonlinear_prev: a
 * potential term -c u with exponential clock density c e^{-cS}) and
 * PAPER.md:212-222 (Eq. probexp2: a random power α with probability p_α and the
 * compensating coefficient c'_α = c_α / p_α).  Writing f(u) = Σ b_k u^k as
 * -λu + Σ a_k u^k with a_k = b_k + λ[k = 1] puts the equation in the form of
 * Eq. nonlinear_prev with arbitrary-sign coefficients.
 * The weight of an α-split is a_α / (λ p_α) (reading R2/R3).      */
int or_normalize(const or_params* p, or_norm* o) {
  memset(o, 0, sizeof(*o));
  if (p->degree < 0 || p->degree > 8) return 1;
  if (p->strategy < 0 || p->strategy > 2) return 3;
  if (p->sampling != 0 && p->sampling != 1) return 7;
  if (p->sampling == 1 && p->strategy == 2) return 7;   /* Strategy B keeps R8 */
  double lam = p->lambda;
  /* strategy 0: λ = -b_1 if b_1 < 0 else 1 (R3); Strategy A's shift
   * u = v e^{t} uses rate 1 unless overridden            */
  if (!(lam > 0.0)) lam = (p->strategy == 0 && p->b[1] < 0.0) ? -p->b[1] : 1.0;
  o->lambda = lam;
  o->inv_lambda = 1.0 / lam;
  o->sigma = sqrt(2.0 * p->D);  /* generator D Δ = ½σ² Δ  (R5) */
  for (int k = 0; k <= 8; ++k) {
    o->a[k] = (k <= p->degree) ? p->b[k] : 0.0;
    /* only the potential form moves -λu out of f; the shift (Eq. totalduhamel)
     * and Strategy B (Eq. totalduhamel_B) sample every term of f, the linear
     * one as a one-child "split"                                            */
    if (k == 1 && p->strategy == 0) o->a[k] += lam;
    if (p->coef_kind[k] != 0 && p->coef_kind[k] != 1) return 4;
  }
  /* shared trees (f4) need node-independent weights: constant coefficients */
  if (p->shared != 0 && p->shared != 1) return 6;
  if (p->shared)
    for (int k = 0; k <= 8; ++k)
      if (p->coef_kind[k] != 0) return 6;
  /* a variable coefficient cannot ride on the potential's k = 1 term */
  if (p->strategy == 0 && p->coef_kind[1] != 0) return 4;
  for (int k = 0; k <= 8; ++k)
    if (p->coef_kind[k] == 1 && !(p->coef_scale > 0.0 && p->coef_t0 > 0.0 &&
                                  p->coef_axis >= 0 && p->coef_axis < p->dim)) return 4;
  if (p->strategy == 2) {
    /* ξ = 0 (leaf) iff a 32-bit draw is below tq: q̂ = tq / 2^32 exactly */
    if (!(p->q > 0.0 && p->q < 1.0)) return 5;
    uint64_t tq = (uint64_t)nearbyint(p->q * 4294967296.0);
    if (tq == 0 || tq >= 4294967296ull) return 5;
    o->tq = tq;
    o->q_hat = (double)tq / 4294967296.0;
  }
  int ns = 0, kmax = 0;
  for (int k = 0; k <= 8; ++k)
    if (o->a[k] != 0.0) { o->support[ns++] = k; kmax = k; }
  o->n_support = ns;
  /* child-digit width: smallest β >= 1 with 2^β >= kmax */
  int beta = 1;
  while ((1 << beta) < kmax) ++beta;
  o->beta = beta;
  if (ns == 0) return 0;
  double prob[9];
  if (p->offspring == 1) {
    for (int s = 0; s < ns; ++s) prob[s] = 1.0 / (double)ns;   /* paper's rule P:222 */
  } else {
    double tot = 0.0;
    for (int s = 0; s < ns; ++s) tot += fabs(o->a[o->support[s]]);
    for (int s = 0; s < ns; ++s) prob[s] = fabs(o->a[o->support[s]]) / tot;
  }
  double cum = 0.0;
  uint64_t prev = 0;
  for (int s = 0; s < ns; ++s) {
    cum += prob[s];
    uint64_t T = (uint64_t)nearbyint(cum * 4294967296.0);
    if (T > 4294967296ull) T = 4294967296ull;
    if (s == ns - 1) T = 4294967296ull;
    if (T <= prev) return 2;            /* zero-width category: infinite weight */
    o->thresh[s] = T;
    o->p_hat[s] = (double)(T - prev) / 4294967296.0;
    /* c'_α = c_α / p_α; Strategy B's c̃ = c / (1 - q)
     * replaces the clock's 1/λ                              */
    if (p->strategy == 2)
      o->w[s] = o->a[o->support[s]] / ((1.0 - o->q_hat) * o->p_hat[s]);
    else
      o->w[s] = o->a[o->support[s]] / (lam * o->p_hat[s]);
    prev = T;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Initial data g (u(x,0) = g(x)); the four shapes of the
 * BASELINE.json configs.                                                   */
static double g_eval(const or_params* p, const double* x) {
  double r2 = 0.0;
  for (int k = 0; k < p->dim; ++k) r2 += x[k] * x[k];
  double s2 = p->init_scale * p->init_scale;
  switch (p->init_kind) {
    case 0: return p->init_amp;
    case 1: return p->init_amp * 0.5 * (1.0 + tanh(x[0] / p->init_scale));
    case 2: return p->init_amp * exp(-r2 / s2);
    case 3: return p->init_amp / (1.0 + r2 / s2);
    default: return NAN;
  }
}

/* Spatio-temporal factor of a variable coefficient c_k(x, t) = b_k φ(x, t),
 * φ = e^{-x_a²/s²} / (t + t0) (Example 5: e^{-x²}/(t+0.1)),
 * evaluated at the split position and the time argument of the children's
 * sub-problem, c_α(y, t - s) (PAPER.md:237 h^{(α)}; PAPER.md:326 for B).     */
static double coef_factor(const or_params* p, int k, const double* y, double tc) {
  if (p->coef_kind[k] == 0) return 1.0;
  double xa = y[p->coef_axis];
  return exp(-(xa * xa) / (p->coef_scale * p->coef_scale)) / (tc + p->coef_t0);
}

/* ------------------------------------------------------------------------ */
/* One tree (the generation procedure; Eq. recursion
 * PAPER.md:224-239; Eq. rep_strategyB).                   */
typedef struct {
  const or_params* p;
  const or_norm* nz;
  uint64_t seed;
  int64_t i, j;
  int32_t ne, leaves, particles;
  int stop;          /* 1 pruned (Ne > K), 2 killed (empty support) */
  const double* node;  /* shared trees (f4): the node x_i, the walk carries δ */
} tree_ctx;

/* Value of the sub-tree rooted at the particle with ancestry label `label`
 * that starts at y with remaining horizon tau.                             */
static double particle(tree_ctx* c, const double* y, double tau, uint64_t label) {
  const or_params* p = c->p;
  const or_norm* nz = c->nz;
  uint32_t r0[4], r1[4], r2[4];
  c->particles++;
  draw(c->seed, c->i, c->j, label, 0, r0);
  draw(c->seed, c->i, c->j, label, 1, r1);
  const int strat_b = (p->strategy == 2);

  /* The particle's fate.  Strategy A (both forms): exponential clock S with
   * density λ e^{-λS}; leaf iff S > τ (1{S > t}).
   * Strategy B: ξ with P(ξ = 0) = q decides
   * leaf / split; a split happens after the uniform fraction S of the
   * horizon, the children inherit τ(1 - S).                                */
  int is_leaf;
  double h, tc;
  double e1 = 0.0, e2 = 0.0;         /* Strategy A: the radii's Exp(1) variates */
  if (strat_b) {
    is_leaf = (uint64_t)r0[3] < nz->tq;                /* ξ = 0 */
    double Sf = or_unif53(r0[0], r0[1]);               /* S ~ U(0,1) */
    h = is_leaf ? tau : tau * Sf;
    tc = tau * (1.0 - Sf);
  } else if (p->sampling == 1) {
    /* textbook sampling (pin of R29 in law, see rt_oracle.h): the clock by
     * inversion, S = -ln(u)/λ; the normals below by
     * Box–Muller with r = sqrt(-2 ln v)                                    */
    double S = -log(or_unif53(r0[0], r0[1])) * nz->inv_lambda;
    is_leaf = S > tau;
    h = is_leaf ? tau : S;
    tc = tau - S;
  } else {
    /* DESIGN.md R29: G = -log(U_1 ... U_{m+1}) ~ Gamma(m+1) split by the
     * spacings of m sorted uniforms into m+1 iid Exp(1) variates: e0 for the
     * clock, e1 (e2) for the Box-Muller radii r = sqrt(2e).               */
    double u12 = or_unif32(r0[0]) * or_unif32(r0[1]);
    double e0;
    if (p->dim <= 2) {
      double v = or_unif32(r0[3]);
      double G = -log(u12);
      e0 = G * v;
      e1 = G * (1.0 - v);
    } else {
      uint32_t lo = r1[1] < r1[2] ? r1[1] : r1[2], hi = r1[1] < r1[2] ? r1[2] : r1[1];
      double v1 = or_unif32(lo), v2 = or_unif32(hi);
      double G = -log(u12 * or_unif32(r1[0]));
      e0 = G * v1;
      e1 = G * (v2 - v1);
      e2 = G * (1.0 - v2);
    }
    double S = e0 * nz->inv_lambda;                    /* S ~ λ e^{-λS} */
    is_leaf = S > tau;
    h = is_leaf ? tau : S;
    tc = tau - S;
  }

  /* Brownian increment over the particle's lifetime (Eqs. green, SDE,
   * PAPER.md:174-191): Box–Muller normals r·(cos, sin)(2πa).  Strategy A
   * (R29): r = sqrt(2e) with e the Exp(1) variates split off the clock's
   * Gamma variate, 32-bit angles.  Strategy B (R8): textbook r = sqrt(-2 log
   * u) — d <= 2: one pair from block 1 (u = w1:w0, angle w3:w2); d = 3:
   * radii from block-1 (w1:w0), (w3:w2), angles from block 2 (w0, w1), its
   * block-0 word 3 being ξ.                                               */
  double xi[3];
  if (!strat_b && p->sampling == 1) {
    double v1 = or_unif53(r1[0], r1[1]), v2 = or_unif53(r1[2], r1[3]);
    double rr = sqrt(-2.0 * log(v1));
    xi[0] = rr * cos(2.0 * M_PI * v2);
    xi[1] = rr * sin(2.0 * M_PI * v2);
    if (p->dim == 3) {
      draw(c->seed, c->i, c->j, label, 2, r2);
      double v3 = or_unif53(r2[0], r2[1]), v4 = or_unif53(r2[2], r2[3]);
      xi[2] = sqrt(-2.0 * log(v3)) * cos(2.0 * M_PI * v4);
    }
  } else if (strat_b) {
    if (p->dim <= 2) {
      double v1 = or_unif53(r1[0], r1[1]), v2 = or_unif53(r1[2], r1[3]);
      double rr = sqrt(-2.0 * log(v1));
      xi[0] = rr * cos(2.0 * M_PI * v2);
      xi[1] = rr * sin(2.0 * M_PI * v2);
    } else {
      double v1 = or_unif53(r1[0], r1[1]), v3 = or_unif53(r1[2], r1[3]);
      draw(c->seed, c->i, c->j, label, 2, r2);
      double v2 = or_unif32(r2[0]), v4 = or_unif32(r2[1]);
      double rr = sqrt(-2.0 * log(v1));
      xi[0] = rr * cos(2.0 * M_PI * v2);
      xi[1] = rr * sin(2.0 * M_PI * v2);
      xi[2] = sqrt(-2.0 * log(v3)) * cos(2.0 * M_PI * v4);
    }
  } else {
    /* angles 2π·unif32: block-1 word 0 (d <= 2); block-0 word 3 and
     * block-1 word 3 (d = 3) */
    double rr = sqrt(2.0 * e1);
    double a1 = or_unif32(p->dim <= 2 ? r1[0] : r0[3]);
    xi[0] = rr * cos(2.0 * M_PI * a1);
    xi[1] = rr * sin(2.0 * M_PI * a1);
    if (p->dim == 3) xi[2] = sqrt(2.0 * e2) * cos(2.0 * M_PI * or_unif32(r1[3]));
  }
  double step = nz->sigma * sqrt(h);
  double x[3];
  for (int k = 0; k < p->dim; ++k) x[k] = y[k] + step * xi[k];

  if (is_leaf) {                       /* the branch reaches the horizon */
    c->leaves++;
    double gv;
    if (c->node) {                     /* shared trees: g(x_i + δ) */
      double xe[3];
      for (int k = 0; k < p->dim; ++k) xe[k] = c->node[k] + x[k];
      gv = g_eval(p, xe);
    } else {
      gv = g_eval(p, x);               /* g at the leaf */
    }
    return strat_b ? gv / nz->q_hat : gv;   /* g̃ = g / q */
  }
  /* splitting event */
  c->ne++;
  if (c->ne > p->K) { c->stop = 1; return 0.0; }   /* prune */
  if (nz->n_support == 0) { c->stop = 2; return 0.0; }
  uint32_t u = r0[2];
  int s = 0;
  while (!((uint64_t)u < nz->thresh[s])) ++s;
  int k = nz->support[s];
  /* h^(α)(y, s) = c'_α(y, t - s) e^{(t-s)(α-1)} (the factor
   * e^{(α-1)τ_c} only with the shift, the child horizon τ_c = t - s, DESIGN.md
   * reading C18); Strategy B: η(τ) c̃'_α(y, τ(1 - S)) with η(τ) = τ
   *                                                      */
  double val = nz->w[s] * coef_factor(p, k, x, tc);
  if (p->strategy == 1) val *= exp((double)(k - 1) * nz->lambda * tc);
  if (strat_b) val *= tau;
  for (int ch = 0; ch < k; ++ch) {
    uint64_t child = (label << nz->beta) | (uint64_t)ch;
    val *= particle(c, x, tc, child);
    if (c->stop) return 0.0;
  }
  return val;
}

static const double ZERO3[3] = {0.0, 0.0, 0.0};

/* Root factor: Strategy A's shift estimates v, and u = v e^{λt}. */
static double root_factor(const or_params* p, const or_norm* nz, double t) {
  return p->strategy == 1 ? exp(nz->lambda * t) : 1.0;
}

int or_tree(const or_params* p, const double* x, int64_t i, int64_t j, double t,
            uint64_t seed, or_tree_rec* rec) {
  or_norm nz;
  int e = or_normalize(p, &nz);
  if (e) return e;
  tree_ctx c = {p, &nz, seed, p->shared ? 0 : i, j, 0, 0, 0, 0, p->shared ? x : NULL};
  double C = root_factor(p, &nz, t) * particle(&c, p->shared ? ZERO3 : x, t, 1u);
  rec->ne = c.ne;
  rec->leaves = c.leaves;
  rec->particles = c.particles;
  rec->pruned = (c.stop == 1);
  rec->C = (c.stop == 1) ? 0.0 : C;
  return 0;
}

int or_trees(const or_params* p, const double* points, int64_t n_points, double t,
             int64_t j0, int64_t n_trees, uint64_t seed, or_tree_rec* rec) {
  or_norm nz;
  int e = or_normalize(p, &nz);
  if (e) return e;
  for (int64_t i = 0; i < n_points; ++i)
    for (int64_t q = 0; q < n_trees; ++q) {
      tree_ctx c = {p, &nz, seed, p->shared ? 0 : i, j0 + q, 0, 0, 0, 0,
                    p->shared ? points + i * p->dim : NULL};
      double C = root_factor(p, &nz, t) * particle(&c, p->shared ? ZERO3 : points + i * p->dim, t, 1u);
      or_tree_rec* r = rec + i * n_trees + q;
      r->ne = c.ne; r->leaves = c.leaves; r->particles = c.particles;
      r->pruned = (c.stop == 1);
      r->C = (c.stop == 1) ? 0.0 : C;
    }
  return 0;
}

/* Records for an explicit list of tree indices js[0..n_js) of every node:
 * rec[i*n_js + q] is tree js[q] of node i (sampled parity at full size). */
int or_trees_at(const or_params* p, const double* points, int64_t n_points, double t,
                const int64_t* js, int64_t n_js, uint64_t seed, or_tree_rec* rec) {
  or_norm nz;
  int e = or_normalize(p, &nz);
  if (e) return e;
  for (int64_t i = 0; i < n_points; ++i)
    for (int64_t q = 0; q < n_js; ++q) {
      tree_ctx c = {p, &nz, seed, p->shared ? 0 : i, js[q], 0, 0, 0, 0,
                    p->shared ? points + i * p->dim : NULL};
      double C = root_factor(p, &nz, t) * particle(&c, p->shared ? ZERO3 : points + i * p->dim, t, 1u);
      or_tree_rec* r = rec + i * n_js + q;
      r->ne = c.ne; r->leaves = c.leaves; r->particles = c.particles;
      r->pruned = (c.stop == 1);
      r->C = (c.stop == 1) ? 0.0 : C;
    }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Order-binned Monte Carlo sums (Eq. simplecase_discrete:
 * u ≈ (1/N) Σ_j f(β_j); grouping by the number of splitting events,
 * PAPER.md:224-239).                                                       */
int or_sums(const or_params* p, const double* points, int64_t n_points, double t,
            int64_t j0, int64_t n_trees, uint64_t seed, double* sums, or_stats* st) {
  or_norm nz;
  int e = or_normalize(p, &nz);
  if (e) return e;
  const int nb = p->K + 2;
  memset(sums, 0, sizeof(double) * (size_t)(n_points * nb * 3));
  or_stats s = {0, 0, 0, 0, 0};
  for (int64_t i = 0; i < n_points; ++i) {
    double* row = sums + i * nb * 3;
    for (int64_t q = 0; q < n_trees; ++q) {
      tree_ctx c = {p, &nz, seed, p->shared ? 0 : i, j0 + q, 0, 0, 0, 0,
                    p->shared ? points + i * p->dim : NULL};
      double C = root_factor(p, &nz, t) * particle(&c, p->shared ? ZERO3 : points + i * p->dim, t, 1u);
      s.trees++;
      s.particles += c.particles;
      s.leaves += c.leaves;
      s.splits += c.ne;
      if (c.stop == 1) {
        s.pruned++;
        row[(p->K + 1) * 3 + 2] += 1.0;
      } else {
        row[c.ne * 3 + 0] += C;
        row[c.ne * 3 + 1] += C * C;
        row[c.ne * 3 + 2] += 1.0;
      }
    }
  }
  if (st) *st = s;
  return 0;
}

/* c_n = ΣC_n / N (N counts pruned trees); se_n = sqrt(max(0, ΣC_n²/N - c_n²)/(N-1)).
 * u_sum = Σ_n c_n; se_sum from the disjoint-bin total (R11).      */
void or_finalize(const double* sums, int64_t n_points, int32_t K, int64_t N,
                 double* coeffs, double* se, double* u_sum, double* se_sum) {
  const int nb = K + 2;
  double Nd = (double)N;
  for (int64_t i = 0; i < n_points; ++i) {
    const double* row = sums + i * nb * 3;
    double us = 0.0, s2 = 0.0;
    for (int n = 0; n <= K; ++n) {
      double c = row[n * 3 + 0] / Nd;
      double v = row[n * 3 + 1] / Nd - c * c;
      if (coeffs) coeffs[i * (K + 1) + n] = c;
      if (se) se[i * (K + 1) + n] = sqrt((v > 0.0 ? v : 0.0) / (Nd - 1.0));
      us += c;
      s2 += row[n * 3 + 1];
    }
    if (u_sum) u_sum[i] = us;
    if (se_sum) {
      double v = s2 / Nd - us * us;
      se_sum[i] = sqrt((v > 0.0 ? v : 0.0) / (Nd - 1.0));
    }
  }
}

/* ------------------------------------------------------------------------ */
/* [L/M] Padé approximant: P/Q with deg P <= L,
 * deg Q <= M, Q(0) = 1 and Q(z) Σ c_n z^n - P(z) = O(z^{L+M+1}).  The
 * denominator solves Σ_{j=1..M} q_j c_{L+i-j} = -c_{L+i}, i = 1..M (c_{<0} = 0),
 * by Gaussian elimination with partial pivoting; p_i = Σ_{j<=min(i,M)} q_j c_{i-j}.
 * Evaluated at z = 1 (the series variable counts splitting events; R4).
 *
 * Degenerate table ("falls back to highest non-degenerate order,
 * flagged"; R12): if the [L/M] system has an exact zero pivot, the
 * value is that of [L/M'] for the largest M' < M whose system is regular —
 * [L/0], the partial sum c_0 + … + c_L, always is — bit0 is set and M' is
 * stored in flag bits 8..15.                                                */
static int pade_denominator(const double* c, int32_t L, int32_t M, double* q) {
  double A[16][17];
  q[0] = 1.0;
  for (int i = 1; i <= M; ++i) {
    for (int j = 1; j <= M; ++j) {
      int idx = L + i - j;
      A[i - 1][j - 1] = (idx >= 0) ? c[idx] : 0.0;
    }
    A[i - 1][M] = -c[L + i];
  }
  /* forward elimination with partial pivoting (first max |.| on ties) */
  for (int col = 0; col < M; ++col) {
    int piv = col;
    for (int r = col + 1; r < M; ++r)
      if (fabs(A[r][col]) > fabs(A[piv][col])) piv = r;
    if (A[piv][col] == 0.0) return 1;                   /* exact zero pivot */
    if (piv != col)
      for (int k = 0; k <= M; ++k) { double tmp = A[col][k]; A[col][k] = A[piv][k]; A[piv][k] = tmp; }
    for (int r = col + 1; r < M; ++r) {
      double f = A[r][col] / A[col][col];
      for (int k = col; k <= M; ++k) A[r][k] -= f * A[col][k];
    }
  }
  /* back substitution */
  for (int r = M - 1; r >= 0; --r) {
    double s = A[r][M];
    for (int k = r + 1; k < M; ++k) s -= A[r][k] * q[k + 1];
    q[r + 1] = s / A[r][r];
  }
  return 0;
}

int or_pade(const double* c, int32_t L, int32_t M, double* u, uint32_t* flags,
            double* p_out, double* q_out) {
  double q[17], pc[17];
  uint32_t fl = 0;
  if (L < 0 || M < 0 || M > 16 || L > 16) return 1;
  int Mu = M;
  while (Mu > 0 && pade_denominator(c, L, Mu, q)) --Mu;   /* degenerate: lower M */
  if (Mu == 0) q[0] = 1.0;
  if (Mu < M) fl |= 1u | ((uint32_t)Mu << 8);
  for (int j = Mu + 1; j <= M; ++j) q[j] = 0.0;
  for (int i = 0; i <= L; ++i) {
    double s = 0.0;
    for (int j = 0; j <= (i < Mu ? i : Mu); ++j) s += q[j] * c[i - j];
    pc[i] = s;
  }
  double P1 = 0.0, Q1 = 0.0;
  for (int i = 0; i <= L; ++i) P1 += pc[i];
  for (int j = 0; j <= Mu; ++j) Q1 += q[j];
  *u = P1 / Q1;
  if (fabs(Q1) <= 1e-14 * fabs(P1)) fl |= 2u;
  /* sign change of Q on (0, 1]: Q(0) = 1; sample 256 equispaced points */
  for (int s = 1; s <= 256; ++s) {
    double z = (double)s / 256.0, Qz = 0.0, zp = 1.0;
    for (int j = 0; j <= Mu; ++j) { Qz += q[j] * zp; zp *= z; }
    if (!(Qz > 0.0)) { fl |= 4u; break; }
  }
  if (flags) *flags = fl;
  if (p_out) for (int i = 0; i <= L; ++i) p_out[i] = pc[i];
  if (q_out) for (int j = 0; j <= M; ++j) q_out[j] = q[j];
  return 0;
}

/* Per-node resummation with the divergence diagnostic (
 * PAPER.md:295-301 the partial sums of a divergent series, 766-769 artificial
 * poles): or_pade of c[0..L+M], plus bit3 when the Padé value and the partial
 * sum u_sum = c_0 + … + c_K (the estimate whose standard error is se_sum)
 * differ by more than 10 se_sum.                                            */
int or_pade_node(const double* c, int32_t K, int32_t L, int32_t M, double se_sum,
                 double* u, uint32_t* flags) {
  uint32_t fl = 0;
  int e = or_pade(c, L, M, u, &fl, NULL, NULL);
  if (e) return e;
  double us = 0.0;
  for (int n = 0; n <= K; ++n) us += c[n];
  if (fabs(*u - us) > 10.0 * se_sum) fl |= 8u;
  if (flags) *flags = fl;
  return 0;
}
