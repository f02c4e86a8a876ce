/* Host cost of fk_step_plan on the headline forest (host-only pool: the
 * planning work without the upload).  cc -O2 profiles/plan_bench.c
 * -Iinclude -Lpaper_2405_19888_b200 -lforkattn -o /tmp/plan_bench */
#include <stdio.h>
#include <stdlib.h>
#include <time.h>
#include "forkattn.h"

static double now_us(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e6 + ts.tv_nsec / 1e3;
}

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 64, S = argc > 2 ? atoi(argv[2]) : 256, P = 6000;
  fk_pool_desc d = {40, 40, 128, 16, 1 << 22, 0, -1, 0};
  fk_pool* p;
  if (fk_pool_create(&d, &p)) return 1;
  int64_t ids[4096], n;
  fk_ctx_create(p, 0, -1);
  fk_ctx_grow(p, 0, P, ids, 4096, &n);
  int64_t leaves[1024];
  for (int r = 0; r < B; ++r) {
    fk_ctx_create(p, 1 + r, 0);
    fk_ctx_grow(p, 1 + r, S + (r * 7) % 16, ids, 4096, &n);
    leaves[r] = 1 + r;
  }
  fk_plan_info info;
  int64_t pos[1024], nid[1024];
  double t_plan = 0, t_grow = 0;
  const int iters = 400;
  for (int i = 0; i < iters; ++i) {
    double t0 = now_us();
    if (fk_step_plan(p, leaves, B, 1, NULL, &info)) { printf("plan failed: %s\n", fk_last_error()); return 1; }
    double t1 = now_us();
    fk_step_grow(p, pos, nid, NULL);
    t_plan += t1 - t0;
    t_grow += now_us() - t1;
  }
  printf("B=%d S=%d: plan %.1f us, grow %.1f us per step (batch_tokens %lld)\n", B, S, t_plan / iters,
         t_grow / iters, (long long)info.batch_tokens);
  fk_pool_destroy(p);
  return 0;
}
