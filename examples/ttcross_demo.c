/*
 * ttcross_demo.c -- the C-ABI without Python: D_5 of BASELINE.json configs[1] (the (4/5!)
 * t-form Ising integral on a 257-point trapezoid grid over [-20, 20], u = e^t nodes), solved
 * by tt_cross_init -> tt_cross_sweep -> tt_integrate (include/ttcross.h).
 *
 *   build: gcc -O2 -o examples/ttcross_demo examples/ttcross_demo.c -Iinclude \
 *              -Lpaper_1903_11554_b200 -lttcross -Wl,-rpath,$PWD/paper_1903_11554_b200 -lm
 *   run  : examples/ttcross_demo            (prints the integral, ranks and evaluations)
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "ttcross.h"

#define D 5
#define N 257

int main(void) {
  static double u[D * N], w[D * N];
  const double L = 20.0, h = 2.0 * L / (N - 1);
  for (int m = 0; m < D; ++m)
    for (int a = 0; a < N; ++a) {
      u[m * N + a] = exp(-L + h * a);
      w[m * N + a] = (a == 0 || a == N - 1) ? h / 2 : h;
    }
  ttc_config cfg = {0};
  cfg.family = TTC_FAMILY_D;
  cfg.d = D;
  cfg.n = N;
  cfg.rank_cap = 16;
  cfg.n_samples = 32;
  cfg.rook_iters = 4;
  cfg.tol = 1e-11;
  cfg.seed = 20190327ULL;
  cfg.rank = 0;
  cfg.world = 1;
  cfg.fold_weights = 0;
  ttc_ctx* ctx = NULL;
  if (tt_cross_init(&ctx, &cfg, u, w, TTC_MEM_HOST, NULL) != TTC_OK) {
    fprintf(stderr, "tt_cross_init: %s\n", tt_last_error());
    return 1;
  }
  if (tt_cross_sweep(ctx, 16) != TTC_OK) {
    fprintf(stderr, "tt_cross_sweep: %s\n", tt_last_error());
    return 1;
  }
  double value = 0, log10_abs = 0;
  int32_t sign = 0;
  if (tt_integrate(ctx, &value, &log10_abs, &sign) != TTC_OK) {
    fprintf(stderr, "tt_integrate: %s\n", tt_last_error());
    return 1;
  }
  int32_t ranks[D - 1];
  tt_cross_get_state(ctx, ranks, NULL, NULL);
  ttc_stats st;
  tt_cross_get_stats(ctx, &st);
  printf("D_5 = %.17g  log10 %.6f  sign %d  ranks", value, log10_abs, sign);
  for (int k = 0; k < D - 1; ++k) printf(" %d", ranks[k]);
  printf("  evals %lld  launches %lld  (%s)\n", (long long)st.evals, (long long)st.launches, tt_build_info());
  tt_cross_destroy(ctx);
  return 0;
}
