/*
 * oracle.h -- CPU ORACLE (TEST INFRASTRUCTURE ONLY).
 *
 * This library is the checker for the B200 gossip + decentralized-Adam path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load it. The product path (libdg.so) never links or calls it.
 *
 * It restates, in plain C++20 with an extern "C" surface for ctypes:
 *   - the keyed SplitMix64 stream generator        (reference proj/src/rng.cpp:11-42)
 *   - the topology module (schedules, validation,   (reference proj/include/declab/topology.hpp:12-100,
 *     spectral/effective lambda, gossip_consensus)   SPEC.md:77-188; topology.cpp does not exist upstream)
 *   - dadam_step / accum_adam_step                   (Alg. 1,
 *                                                     PAPER.md:2139-2158 Alg. 3)
 *     in fp64 (reference semantics, vec.cpp op order) and as an fp32 "mirror"
 *     with the exact per-element op order of SURVEY.md Appendix A, which the
 *     CUDA kernel must reproduce bit for bit.
 *
 * Parity pinning: the RNG and the vec primitives are pinned against the
 * reference's own vec.cpp / rng.cpp compiled from /root/reference into
 * oracle/_ref (see oracle/ref_shim.cpp, oracle/Makefile) and against committed
 * golden vectors in tests/golden/ generated from that build.  The topology
 * restatement is pinned by the SPEC's [TRIVIAL]/[DERIVED]/[PAPER] examples
 * (the reference ships no topology.cpp and no Eigen, so there is nothing else
 * to pin it against).
 */
#pragma once
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror errors.hpp (ConfigError=2, DivergenceError=3, InvariantError=4) */
enum { OR_OK = 0, OR_CONFIG_ERROR = 2, OR_DIVERGENCE = 3, OR_INVARIANT = 4 };
const char* or_last_error(void);
long or_last_divergence_iteration(void);

/* ---------------- rng (rng.cpp:14-42) ---------------- */
/* draws first..first+n-1 (0-based draw index) of StreamRng(seed,purpose,worker,iteration) */
void or_rng_u64(uint64_t seed, uint32_t purpose, uint64_t worker, uint64_t iteration,
                uint64_t first, size_t n, uint64_t* out);
void or_rng_unit(uint64_t seed, uint32_t purpose, uint64_t worker, uint64_t iteration,
                 uint64_t first, size_t n, double* out);
/* synthetic bucket value: (float)(2u-1), u = draw e of the stream */
void or_fill_f32(uint64_t seed, uint32_t purpose, uint64_t worker, uint64_t iteration,
                 size_t n, float* out);

/* ---------------- topology (topology.hpp:40-100) ---------------- */
enum { OR_COMPLETE = 0, OR_ONE_PEER_RING = 1, OR_ONE_PEER_EXP = 2, OR_AER = 3, OR_STATIC_EXP = 4 };
typedef struct or_sched or_sched;
int or_make(int kind, int n, int workers_per_node, or_sched** out);
/* from_matrices (topology.hpp:44-45): rows-major P x n x n */
int or_from_matrices(const double* w, int n, int period, int workers_per_node, or_sched** out);
void or_free(or_sched* s);
int or_info(const or_sched* s, int* workers, int* period, int* wpn, int* is_static);
int or_matrix(const or_sched* s, long round, double* w_rowmajor);
int or_neighbors(const or_sched* s, long round, int worker, int* idx, double* w, int cap,
                 int* count);

typedef struct {
  int symmetric, nonnegative, rows_stochastic, cols_stochastic, eigenvalues_in_range;
  double max_asymmetry, min_entry, max_row_error, max_col_error, min_eigenvalue,
      max_eigenvalue;
} or_validation;
int or_validate(const double* w, int n, or_validation* out);
int or_spectral_lambda(const double* w, int n, double* out);
int or_effective_lambda(const or_sched* s, double* out);
/* x0: n x d row-major; err_out: rounds+1 */
int or_gossip_consensus(const or_sched* s, const double* x0, int n, size_t d, int rounds,
                        int threads, double* err_out);

/* ---------------- optim ---------------- */
typedef struct {
  double alpha, beta1, beta2, eps;
  int s;             /* accumulation length (Alg. 3) */
  int paper_literal; /* Alg. 3 line 12 uses beta1 as printed */
} or_adam_cfg;

int or_dadam_step_f64(double* x, const double* g, double* m, double* v, const double* mixed,
                      size_t d, const or_adam_cfg* cfg, long t);
int or_dadam_step_f32(float* x, const float* g, float* m, float* v, const float* mixed,
                      size_t d, const or_adam_cfg* cfg, long t);
int or_accum_adam_step_f64(double* x, const double* g, double* m_hat, double* v_hat,
                           double* b, const double* mixed, size_t d, const or_adam_cfg* cfg,
                           long t, long T);
int or_accum_adam_step_f32(float* x, const float* g, float* m_hat, float* v_hat, float* b,
                           const float* mixed, size_t d, const or_adam_cfg* cfg, long t,
                           long T);

/* Multi-node driver (trainsim run_training loop restricted to the hot path,
 * SPEC.md:350-357): steps t_begin..t_end inclusive over all n nodes, Jacobi
 * snapshot of x^(t-1), gradients g_i^(t)[e] = (float)(2u-1) from
 * StreamRng(seed, Minibatch=2, i, t).  algo: 0 = DAdam, 1 = AccumAdam.
 * States are n x d row-major.  b may be NULL for DAdam.  */
enum { OR_DADAM = 0, OR_ACCUM = 1, OR_ALLREDUCE = 2 /* Alg. 2 */ };
int or_run_f64(const or_sched* s, int algo, const or_adam_cfg* cfg, uint64_t seed, size_t d,
               long t_begin, long t_end, long T, int threads, double* x, double* m, double* v,
               double* b);
int or_run_f32(const or_sched* s, int algo, const or_adam_cfg* cfg, uint64_t seed, size_t d,
               long t_begin, long t_end, long T, int threads, float* x, float* m, float* v,
               float* b);
/* One step for all n nodes with caller-provided gradients g (n x d), fp64.
 * Used as the CPU baseline ("port"): no gradient generation inside. */
int or_step_all_f64(const or_sched* s, int algo, const or_adam_cfg* cfg, size_t d, long t,
                    long T, int threads, const double* g, double* x, double* x_prev, double* m,
                    double* v, double* b);
/* fp32 mirror of one step with a caller-supplied gradient (e.g. g held fixed
 * across steps, as the CUDA-graph step ranges of the engine replay it). */
int or_step_all_f32(const or_sched* s, int algo, const or_adam_cfg* cfg, size_t d, long t,
                    long T, int threads, const float* g, float* x, float* x_prev, float* m,
                    float* v, float* b);
int or_max_threads(void);

/* Column-sampled run: every parameter column evolves independently of the
 * others (mixing and Adam are elementwise), so the trajectory of the columns
 * cols[0..ncols) of a d-parameter bucket can be replayed exactly without the
 * rest of the bucket.  x0 and g_i^(t) are drawn at the columns' own draw
 * indices (x0: ConsensusInit per node if dispersed, else the shared InitModel
 * stream).  Outputs are n x ncols row-major, fp32 mirror (_f32) or fp64 with
 * the same fp32 inputs (_f64).  Used to check full-size (125M .. 1.3B) buckets. */
int or_run_cols_f32(const or_sched* s, int algo, const or_adam_cfg* cfg, uint64_t seed,
                    const uint64_t* cols, size_t ncols, int dispersed, long t_begin, long t_end,
                    long T, int threads, float* x, float* m, float* v, float* b);
int or_run_cols_f64(const or_sched* s, int algo, const or_adam_cfg* cfg, uint64_t seed,
                    const uint64_t* cols, size_t ncols, int dispersed, long t_begin, long t_end,
                    long T, int threads, double* x, double* m, double* v, double* b);

#ifdef __cplusplus
}
#endif
