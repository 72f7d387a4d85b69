/* abi_smoke.c — the C ABI (include/gv.h) called from plain C, no Python:
 * create -> load_edges -> push_sample_pool -> train_episode -> get_* ->
 * destroy on a 4-cycle plus chords, with the pool drawn from the library's
 * own host augmentation (gv_augment, Alg. 2). Exit code 0 = every call
 * returned GV_OK and the statistics / embeddings are consistent:
 *   - samples_global == pool size, n_ranks == 1, ms_device_max == ms_total;
 *   - isolated node 7 keeps context row 0 and its initial vertex row;
 *   - every embedding is finite.
 * Built and run by tests/test_abi.py (compile + link on CPU) and
 * tests/test_gpu_abi_c.py (run on the GPU). */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "gv.h"

#define CHECK(call)                                                              \
  do {                                                                           \
    gv_status s_ = (call);                                                       \
    if (s_ != GV_OK) {                                                           \
      fprintf(stderr, "%s -> %s: %s\n", #call, gv_status_string(s_),             \
              gv_last_error(ctx));                                               \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

int main(void) {
  gv_ctx* ctx = NULL;
  const uint32_t nv = 8, dim = 16, K = 1;
  const uint32_t src[] = {0, 1, 2, 3, 0, 1, 4, 5, 6};
  const uint32_t dst[] = {1, 2, 3, 0, 2, 3, 5, 6, 4};
  const uint64_t ne = sizeof(src) / sizeof(src[0]);
  const uint64_t pool = 50000;
  if (gv_abi_version() != GV_ABI_VERSION) return 2;
  gv_lr_schedule lr = {GV_LR_LINEAR, 1e-4, pool};
  gv_options opt;
  gv_default_options(&opt);
  CHECK(gv_create(nv, dim, 2, K, 0.025f, &lr, &opt, &ctx));
  CHECK(gv_load_edges(ctx, src, dst, NULL, ne));
  float* v0 = malloc(sizeof(float) * nv * dim);
  float* v1 = malloc(sizeof(float) * nv * dim);
  float* c1 = malloc(sizeof(float) * nv * dim);
  uint32_t* pairs = malloc(sizeof(uint32_t) * 2 * pool);
  if (!v0 || !v1 || !c1 || !pairs) return 3;
  CHECK(gv_get_vertex_embeddings(ctx, v0, (uint64_t)nv * dim));
  CHECK(gv_augment(ctx, 40, 2, 4, pool, 7, pairs));
  CHECK(gv_push_sample_pool(ctx, pairs, pool));
  gv_episode_stats st;
  CHECK(gv_train_episode(ctx, &st));
  CHECK(gv_get_vertex_embeddings(ctx, v1, (uint64_t)nv * dim));
  CHECK(gv_get_context_embeddings(ctx, c1, (uint64_t)nv * dim));
  int bad = 0;
  bad |= st.samples_global != pool;
  bad |= st.n_ranks != 1;
  bad |= st.ms_device_max != st.ms_total_rank[0];
  bad |= !(st.ms_device_max > 0.0);
  for (uint64_t k = 0; k < (uint64_t)nv * dim; ++k) bad |= !isfinite(v1[k]) || !isfinite(c1[k]);
  for (uint32_t k = 0; k < dim; ++k) bad |= c1[7 * dim + k] != 0.0f || v1[7 * dim + k] != v0[7 * dim + k];
  double moved = 0;
  for (uint32_t k = 0; k < dim; ++k) moved += fabs(v1[k] - v0[k]);
  bad |= !(moved > 0.0);
  printf("abi_smoke: samples %llu, loss %.6f, ms_device_max %.3f -> %s\n",
         (unsigned long long)st.samples_global, st.loss_sum, st.ms_device_max, bad ? "FAIL" : "ok");
  gv_destroy(ctx);
  free(v0); free(v1); free(c1); free(pairs);
  return bad ? 4 : 0;
}
