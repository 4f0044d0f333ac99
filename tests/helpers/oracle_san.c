/* Drives the oracle (oracle/rt_oracle.c) through every entry point on small
 * cases of each strategy, dimension and data shape; built with
 * -fsanitize=address,undefined by tests/test_oracle_sanitize.py (host
 * sanitizers: the GPU pool does not offer compute-sanitizer). */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "rt_oracle.h"

static or_params base(int dim, int strategy, int kind, int shared) {
  or_params p;
  memset(&p, 0, sizeof(p));
  p.dim = dim; p.D = 1.0; p.degree = 4;
  double b[5] = {0.0, -1.0, 0.5, 0.8, -0.3};
  for (int k = 0; k < 5; ++k) p.b[k] = b[k];
  p.init_kind = kind; p.init_amp = 0.4; p.init_scale = 1.0; p.K = 12;
  p.strategy = strategy; p.q = 0.7; p.shared = shared;
  p.coef_scale = 1.0; p.coef_t0 = 0.1;
  if (strategy != 0 && !shared) p.coef_kind[2] = 1;
  return p;
}

int main(void) {
  double pts[3 * 4] = {0.0, 0.1, -0.2, 0.5, 1.0, -1.5, -0.7, 0.3, 2.0, 1.1, -0.4, 0.25};
  int nb = 14, bad = 0;
  double* sums = malloc(sizeof(double) * 4 * nb * 3);
  or_tree_rec* rec = malloc(sizeof(or_tree_rec) * 4 * 50);
  for (int dim = 1; dim <= 3; ++dim)
    for (int strategy = 0; strategy <= 2; ++strategy)
      for (int kind = 0; kind <= 3; ++kind)
        for (int shared = 0; shared <= 1; ++shared)
        for (int sampling = 0; sampling <= (strategy == 2 ? 0 : 1); ++sampling) {
          or_params p = base(dim, strategy, kind, shared);
          p.sampling = sampling;   /* 1: the textbook sampler (pin of R29 in law) */
          or_stats st;
          if (or_sums(&p, pts, 4, 1.0, 7, 200, 3, sums, &st)) bad++;
          if (or_trees(&p, pts, 4, 0.5, 0, 50, 11, rec)) bad++;
          double c[13 * 4], se[13 * 4], us[4], ses[4];
          or_finalize(sums, 4, 12, 200, c, se, us, ses);
          for (int i = 0; i < 4; ++i) {
            double u, pp[8], qq[8];
            uint32_t fl;
            if (or_pade(c + 13 * i, 5, 5, &u, &fl, pp, qq)) bad++;
            if (or_pade_node(c + 13 * i, 12, 5, 5, ses[i], &u, &fl)) bad++;
          }
        }
  printf("sanitized oracle run done, %d errors\n", bad);
  free(sums);
  free(rec);
  return bad != 0;
}
