/* A native C consumer of include/dg.h, linked against libdg.so (no Python,
 * no torch) -- what a C/C++ caller of the reference's topology.hpp API sees.
 * tests/test_c_abi.py compiles it with gcc and checks its output:
 *
 *   c_abi_main layout          sizeof / offsetof of every public struct
 *                              (compared with the ctypes mirror in __init__.py)
 *   c_abi_main schedules       name, info and every round's neighbour lists of
 *                              the built-in topologies (compared with the oracle)
 *   c_abi_main engine OUT      8 nodes, one-peer ring, DAdam then AccumAdam s=4,
 *                              12 fused engine steps on cuda:0; x, m, v (and acc)
 *                              written to OUT (compared bit-exactly with the
 *                              oracle's fp32 mirror; needs a GPU)
 */
#include <stddef.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "dg.h"

#define CHECK(call)                                                                 \
  do {                                                                              \
    int rc_ = (call);                                                               \
    if (rc_ != DG_OK) {                                                             \
      fprintf(stderr, "%s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #call, rc_,     \
              dg_last_error());                                                     \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

#define FIELD(S, F) printf("field %s %s %zu %zu\n", #S, #F, offsetof(S, F), sizeof(((S*)0)->F))
#define SIZE(S) printf("sizeof %s %zu\n", #S, sizeof(S))

static void layout(void) {
  SIZE(dg_adam_cfg);
  FIELD(dg_adam_cfg, alpha); FIELD(dg_adam_cfg, beta1); FIELD(dg_adam_cfg, beta2);
  FIELD(dg_adam_cfg, eps); FIELD(dg_adam_cfg, s); FIELD(dg_adam_cfg, paper_literal);
  SIZE(dg_validation);
  FIELD(dg_validation, symmetric); FIELD(dg_validation, nonnegative);
  FIELD(dg_validation, rows_stochastic); FIELD(dg_validation, cols_stochastic);
  FIELD(dg_validation, eigenvalues_in_range); FIELD(dg_validation, max_asymmetry);
  FIELD(dg_validation, min_entry); FIELD(dg_validation, max_row_error);
  FIELD(dg_validation, max_col_error); FIELD(dg_validation, min_eigenvalue);
  FIELD(dg_validation, max_eigenvalue);
  SIZE(dg_engine_config);
  FIELD(dg_engine_config, schedule); FIELD(dg_engine_config, world_size);
  FIELD(dg_engine_config, rank); FIELD(dg_engine_config, device);
  FIELD(dg_engine_config, nccl_id); FIELD(dg_engine_config, d); FIELD(dg_engine_config, chunk);
  FIELD(dg_engine_config, algo); FIELD(dg_engine_config, adam);
  FIELD(dg_engine_config, total_steps); FIELD(dg_engine_config, transport);
  FIELD(dg_engine_config, flags);
  SIZE(dg_engine_stats);
  FIELD(dg_engine_stats, local_nodes); FIELD(dg_engine_stats, first_node);
  FIELD(dg_engine_stats, nodes); FIELD(dg_engine_stats, world_size); FIELD(dg_engine_stats, rank);
  FIELD(dg_engine_stats, d); FIELD(dg_engine_stats, chunk);
  FIELD(dg_engine_stats, kernel_launches); FIELD(dg_engine_stats, steps);
  FIELD(dg_engine_stats, bytes_sent); FIELD(dg_engine_stats, bytes_received);
  FIELD(dg_engine_stats, hbm_bytes); FIELD(dg_engine_stats, nccl_version);
  FIELD(dg_engine_stats, kernel_ms); FIELD(dg_engine_stats, timed_launches);
  FIELD(dg_engine_stats, timed_hbm_bytes); FIELD(dg_engine_stats, transport);
  FIELD(dg_engine_stats, barriers); FIELD(dg_engine_stats, remote_kernel_ms);
  FIELD(dg_engine_stats, remote_bytes);
  SIZE(dg_rm_params);
  FIELD(dg_rm_params, N); FIELD(dg_rm_params, b); FIELD(dg_rm_params, theta);
  FIELD(dg_rm_params, gamma); FIELD(dg_rm_params, omega); FIELD(dg_rm_params, sigma2);
  FIELD(dg_rm_params, workers_per_node); FIELD(dg_rm_params, normalized);
  FIELD(dg_rm_params, allow_omega_above_one);
}

static void dump_schedule(const char* label, dg_schedule* s) {
  int n, period, wpn, is_static;
  char name[64];
  size_t len = 0;
  CHECK(dg_schedule_info(s, &n, &period, &wpn, &is_static));
  CHECK(dg_schedule_name(s, name, sizeof name, &len));
  printf("schedule %s name=%s n=%d period=%d wpn=%d static=%d\n", label, name, n, period, wpn, is_static);
  int* idx = malloc(sizeof(int) * (size_t)n);
  double* w = malloc(sizeof(double) * (size_t)n);
  for (long r = 1; r <= period; ++r)
    for (int i = 0; i < n; ++i) {
      int cnt = 0;
      CHECK(dg_schedule_neighbors(s, r, i, idx, w, n, &cnt));
      printf("round %ld worker %d:", r, i);
      for (int k = 0; k < cnt; ++k) printf(" %d:%.17g", idx[k], w[k]);
      printf("\n");
    }
  /* validate() of round 1 through the C ABI */
  double* m = malloc(sizeof(double) * (size_t)n * (size_t)n);
  dg_validation v;
  char desc[512];
  CHECK(dg_schedule_matrix(s, 1, m));
  CHECK(dg_validate(m, n, &v));
  CHECK(dg_validation_describe(&v, desc, sizeof desc, &len));
  printf("validate %s pass=%d\n", label, dg_validation_pass(&v));
  free(m);
  free(idx);
  free(w);
  dg_schedule_free(s);
}

static void schedules(void) {
  dg_schedule* s;
  CHECK(dg_make_complete(8, &s));
  dump_schedule("complete8", s);
  CHECK(dg_make_one_peer_ring(8, &s));
  dump_schedule("one_peer_ring8", s);
  CHECK(dg_make_one_peer_exponential(8, &s));
  dump_schedule("one_peer_exponential8", s);
  CHECK(dg_make_one_peer_exponential(16, &s));
  dump_schedule("one_peer_exponential16", s);
  CHECK(dg_make_aer(8, 2, &s));
  dump_schedule("aer8_2", s);
  CHECK(dg_make_static_exponential(8, &s));
  dump_schedule("static_exponential8", s);
  /* errors.hpp taxonomy through the ABI: one_peer_exponential needs a power of two */
  int rc = dg_make_one_peer_exponential(6, &s);
  printf("error one_peer_exponential6 rc=%d\n", rc);
}

static int engine(const char* out_path) {
  enum { N = 8, T = 12 };
  const size_t d = 4099; /* not a multiple of 4: exercises the scalar tail */
  const unsigned long long seed = 2410;
  FILE* f = fopen(out_path, "wb");
  if (!f) return 1;
  float* host = malloc(sizeof(float) * d);
  for (int algo = DG_ALGO_DADAM; algo <= DG_ALGO_ACCUM; ++algo) {
    dg_schedule* s;
    CHECK(dg_make_one_peer_ring(N, &s));
    dg_engine_config cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.schedule = s;
    cfg.world_size = 1;
    cfg.d = d;
    cfg.algo = algo;
    if (algo == DG_ALGO_DADAM) {
      dg_adam_cfg a = {2e-3, 0.974, 0.999, 1e-8, 1, 0};
      cfg.adam = a;
    } else {
      dg_adam_cfg a = {8e-4, 0.9, 0.999, 1e-8, 4, 0};
      cfg.adam = a;
    }
    cfg.total_steps = T;
    cfg.transport = DG_TRANSPORT_AUTO;
    dg_engine* e;
    CHECK(dg_engine_create(&cfg, &e));
    dg_schedule_free(s); /* borrowed during create only */
    CHECK(dg_engine_fill_synthetic(e, DG_BUF_X, seed, 6 /* ConsensusInit (rng.hpp:9-16) */, 1, 0));
    for (long t = 1; t <= T; ++t) {
      CHECK(dg_engine_fill_synthetic(e, DG_BUF_G, seed, 2 /* Minibatch */, 1, (uint64_t)t));
      CHECK(dg_engine_step(e, t));
    }
    CHECK(dg_engine_sync(e));
    dg_engine_stats st;
    CHECK(dg_engine_get_stats(e, &st));
    printf("engine algo=%d nodes=%d steps=%ld launches=%ld\n", algo, st.local_nodes, st.steps,
           st.kernel_launches);
    const int kinds = algo == DG_ALGO_ACCUM ? 4 : 3;
    const int which[4] = {DG_BUF_X, DG_BUF_M, DG_BUF_V, DG_BUF_ACC};
    for (int k = 0; k < kinds; ++k)
      for (int i = 0; i < N; ++i) {
        CHECK(dg_engine_download(e, i, which[k], host, 0, d));
        fwrite(host, sizeof(float), d, f);
      }
    dg_engine_destroy(e);
  }
  free(host);
  fclose(f);
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    fprintf(stderr, "usage: %s layout|schedules|engine OUT\n", argv[0]);
    return 2;
  }
  printf("dg_version %d\n", dg_version());
  if (!strcmp(argv[1], "layout")) layout();
  else if (!strcmp(argv[1], "schedules")) schedules();
  else if (!strcmp(argv[1], "engine") && argc > 2) return engine(argv[2]);
  else return 2;
  return 0;
}
