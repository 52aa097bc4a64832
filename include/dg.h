/*
 * dg.h -- C ABI of the B200-native decentralized gossip + Adam step
 *         (arXiv 2410.11998, Alg. 1 DAdam and Alg. 3 AccumAdam).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference is
 * an in-process C++20 API (namespace declab); every entry point below names
 * the reference symbol it replaces.  Plain C types only: no CUDA, NCCL or torch
 * types appear in any signature (streams are passed as void* = cudaStream_t).
 *
 * Status codes mirror the reference error taxonomy (errors.hpp:8-26, exit
 * codes SPEC.md:550): ConfigError -> DG_CONFIG_ERROR (2), DivergenceError ->
 * DG_DIVERGENCE (3, iteration via dg_last_divergence_iteration), InvariantError
 * -> DG_INVARIANT (4).  CUDA / NCCL failures add codes 5 / 6.
 *
 * Threading (topology.hpp:39): schedules are immutable and
 * safe for concurrent reads; an engine is driven by one host thread; all
 * device work is stream-ordered and asynchronous; errors are sticky per engine.
 */
#ifndef DG_H_
#define DG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum dg_status {
  DG_OK = 0,
  DG_CONFIG_ERROR = 2, /* declab::ConfigError     (errors.hpp:10-12) */
  DG_DIVERGENCE = 3,   /* declab::DivergenceError (errors.hpp:16-20) */
  DG_INVARIANT = 4,    /* declab::InvariantError  (errors.hpp:24-26) */
  DG_CUDA_ERROR = 5,
  DG_NCCL_ERROR = 6
};

/* Thread-local message of the last failing call on this thread. */
const char* dg_last_error(void);
/* DivergenceError::iteration (errors.hpp:17) of the last DG_DIVERGENCE. */
long dg_last_divergence_iteration(void);
int dg_version(void);

/* ======================================================================
 * Topology -- replaces declab::MixingSchedule and the make_* builders
 * (proj/include/declab/topology.hpp:36-100).
 * ====================================================================== */
typedef struct dg_schedule dg_schedule;

/* make_complete(n)                     topology.hpp:65-66 */
int dg_make_complete(int n, dg_schedule** out);
/* make_one_peer_ring(n), n even        topology.hpp:67-69 */
int dg_make_one_peer_ring(int n, dg_schedule** out);
/* make_one_peer_exponential(n), 2^k    topology.hpp:70-72 */
int dg_make_one_peer_exponential(int n, dg_schedule** out);
/* make_aer(n, workers_per_node)        topology.hpp:73-78 */
int dg_make_aer(int n, int workers_per_node, dg_schedule** out);
/* NEW (not in the reference; north_star "static exponential"): undirected
 * circulant i +/- 2^k, weight 1/(deg+1), period 1. */
int dg_make_static_exponential(int n, dg_schedule** out);
/* MixingSchedule::from_matrices(name, wpn, rounds)   topology.hpp:44-45
 * w: period x n x n row-major; validates every round + union connectivity */
int dg_schedule_from_matrices(const double* w, int n, int period, int workers_per_node,
                              dg_schedule** out);
/* from_matrices with the schedule's name (topology.hpp:44-45; the unnamed form
 * above names it "custom") */
int dg_schedule_from_matrices_named(const char* name, const double* w, int n, int period,
                                    int workers_per_node, dg_schedule** out);
/* name()  topology.hpp:50 -- "complete", "one_peer_ring", "one_peer_exponential",
 * "aer", "static_exponential" for the builders.  Copies a NUL-terminated string
 * into buf (cap bytes; DG_CONFIG_ERROR if too small); *len = strlen(name). */
int dg_schedule_name(const dg_schedule* s, char* buf, size_t cap, size_t* len);
/* workers() / period() / workers_per_node() / is_static()   topology.hpp:47-51 */
int dg_schedule_info(const dg_schedule* s, int* workers, int* period, int* workers_per_node,
                     int* is_static);
/* neighbors_at(round)[worker] (1-based periodic round; ascending; self included)
 * with the matching w_ij.  topology.hpp:54-55.  *count is set even when cap is
 * too small (then DG_CONFIG_ERROR). */
int dg_schedule_neighbors(const dg_schedule* s, long round, int worker, int* idx, double* w,
                          int cap, int* count);
/* matrix_at(round) as n x n row-major doubles.  topology.hpp:53 */
int dg_schedule_matrix(const dg_schedule* s, long round, double* w_rowmajor);
void dg_schedule_free(dg_schedule* s);

/* MixingValidation (topology.hpp:16-34) */
typedef struct dg_validation {
  int symmetric, nonnegative, rows_stochastic, cols_stochastic, eigenvalues_in_range;
  double max_asymmetry, min_entry, max_row_error, max_col_error, min_eigenvalue, max_eigenvalue;
} dg_validation;
/* MixingValidation::pass() (topology.hpp:29-32): 1 if every check passed */
int dg_validation_pass(const dg_validation* v);
/* MixingValidation::describe() (topology.hpp:33): one-line human-readable
 * report; same buffer contract as dg_schedule_name */
int dg_validation_describe(const dg_validation* v, char* buf, size_t cap, size_t* len);
/* validate(W)                 topology.hpp:80 */
int dg_validate(const double* w, int n, dg_validation* out);
/* spectral_lambda(W)          topology.hpp:82-84 (DG_CONFIG_ERROR if not symmetric) */
int dg_spectral_lambda(const double* w, int n, double* out);
/* effective_lambda(schedule)  topology.hpp:86-88 */
int dg_effective_lambda(const dg_schedule* s, double* out);

/* ======================================================================
 * Per-node semantic step -- replaces declab::dadam_step / accum_adam_step
 * (SPEC.md:272-298).  The reference returns a new WorkerState; here the
 * fp32 device buffers are updated in place (x, m, v[, acc]).  All pointers
 * are device pointers of length d; `mixed` is the caller-formed
 * Sigma_j w_ij x_j^(t-1).  Stream-ordered on `stream`
 * (cudaStream_t, NULL = legacy default).  Non-finite results are reported by
 * dg_step_check_divergence().
 * ====================================================================== */
typedef struct dg_adam_cfg {
  double alpha, beta1, beta2, eps; /* OptimizerConfig */
  int s;                           /* accumulation length (Alg. 3), >= 1 */
  int paper_literal;               /* Alg. 3 line 12 with beta1 as printed */
} dg_adam_cfg;

/* mixed = sum_k w[k] * xs[k] in the given order (ascending j, self included);
 * xs is a HOST array of `count` device pointers.  The mixing half of the step
 * (gossip_consensus inner loop topology.hpp:98-100). */
int dg_gossip_mix_f32(float* mixed, const float* const* xs, const double* w, int count, size_t d,
                      void* stream);
/* dadam_step(state, g, mixed, cfg, t)          SPEC.md:272-280 (t >= 1) */
int dg_dadam_step_f32(float* x, const float* g, float* m, float* v, const float* mixed, size_t d,
                      const dg_adam_cfg* cfg, long t, void* stream);
/* accum_adam_step(state, g, mixed, cfg, t)     SPEC.md:290-298 (T mod s == 0, t <= T);
 * m_hat/v_hat/acc are WorkerState::m_hat/v_hat/b_acc */
int dg_accum_adam_step_f32(float* x, const float* g, float* m_hat, float* v_hat, float* acc,
                           const float* mixed, size_t d, const dg_adam_cfg* cfg, long t, long T,
                           void* stream);
/* Synchronises `stream` and returns DG_DIVERGENCE (iteration = first t with a
 * non-finite x/m/v, errors.hpp:16-20) if any semantic step since the last
 * call produced one; clears the flag. */
int dg_step_check_divergence(void* stream);

/* Synthetic bucket values on the device: out[e] = (float)(2u-1), u = draw e of
 * StreamRng(seed, purpose, worker, iteration) (rng.cpp:26-42), bit-identical
 * to the CPU generator. */
int dg_fill_synthetic_f32(float* out, size_t n, uint64_t seed, uint32_t purpose, uint64_t worker,
                          uint64_t iteration, void* stream);

/* ======================================================================
 * Fused engine -- one per GPU.  Owns the flat fp32 buckets of the nodes
 * resident on this GPU (nodes block-partitioned: node i -> rank
 * floor(i*G/N)), the NCCL communicator and two streams.  One call to
 * dg_engine_step(t) performs, for every resident node i, Alg. 1 lines 4-6
 * (or Alg. 3 lines 4-14) with x_i <- sum_j w_ij^(t) x_j^(t-1), exchanging
 * remote neighbours' buckets chunk by chunk over NVLink (ncclSend/ncclRecv on
 * the comm stream, double-buffered, overlapped with the fused kernel on the
 * previous chunk).  Replaces the trainsim inner loop
 * for the hot path.
 * ====================================================================== */
typedef struct dg_engine dg_engine;
/* DG_ALGO_ALLREDUCE: All-Reduce Adam (Alg. 2),
 * the comparison baseline: gbar = mean of all N nodes'
 * gradients (fp64 column sums, NCCL all-reduce across ranks), every node applies
 * Adam with gbar and no mixing; nodes must stay identical (|x_i - x_0| <= 1e-12,
 * else dg_engine_sync returns DG_INVARIANT).  The schedule only fixes N. */
enum { DG_ALGO_DADAM = 0, DG_ALGO_ACCUM = 1, DG_ALGO_ALLREDUCE = 2 };
enum { DG_BUF_X = 0, DG_BUF_G = 1, DG_BUF_M = 2, DG_BUF_V = 3, DG_BUF_ACC = 4 };

typedef struct dg_engine_config {
  const dg_schedule* schedule; /* borrowed during create; N = workers() */
  int world_size;              /* GPUs (ranks) */
  int rank;                    /* this engine's rank */
  int device;                  /* CUDA device ordinal */
  const void* nccl_id;         /* 128-byte ncclUniqueId from rank 0 (world_size > 1) */
  size_t d;                    /* parameters per node (flat fp32 bucket) */
  size_t chunk;                /* elements per gossip chunk; 0 = 6,553,600 (25 MiB) */
  int algo;                    /* DG_ALGO_DADAM | DG_ALGO_ACCUM */
  dg_adam_cfg adam;
  long total_steps;            /* T (AccumAdam requires T mod s == 0) */
  int transport;               /* DG_TRANSPORT_*: how remote neighbour buckets move (world_size > 1) */
  int flags;                   /* DG_ENGINE_* */
} dg_engine_config;

/* DG_ENGINE_IN_PLACE: x is never double-buffered (the DG_BUF_X pointer is
 * stable for the engine's lifetime, e.g. framework parameters are views of
 * it); forces the NCCL transport when world_size > 1.  Required for
 * dg_engine_step_range. */
enum { DG_ENGINE_IN_PLACE = 1 };

/* DG_TRANSPORT_P2P (default): the fused kernel reads remote neighbours'
 * x^(t-1) directly from peer HBM over NVLink (CUDA IPC mappings; x is
 * double-buffered in exchange rounds, a stream-ordered 1-element NCCL
 * all-reduce is the cross-GPU step barrier).  DG_TRANSPORT_NCCL: chunked
 * ncclSend/ncclRecv into double-buffered recv slots on a side stream,
 * overlapped with the fused kernel on the previous chunk. */
enum { DG_TRANSPORT_AUTO = 0, DG_TRANSPORT_NCCL = 1, DG_TRANSPORT_P2P = 2 };

typedef struct dg_engine_stats {
  int local_nodes, first_node, nodes, world_size, rank;
  size_t d, chunk;
  long kernel_launches;     /* fused kernels launched since create */
  long steps;               /* dg_engine_step calls */
  double bytes_sent;        /* NVLink payload sent since create */
  double bytes_received;
  double hbm_bytes;         /* algorithmic HBM bytes of the fused kernels since create */
  long nccl_version;
  double kernel_ms;         /* summed CUDA-event durations of timed fused launches */
  long timed_launches;      /* launches covered by kernel_ms / timed_hbm_bytes */
  double timed_hbm_bytes;   /* algorithmic HBM bytes of those launches */
  int transport;            /* DG_TRANSPORT_NCCL | DG_TRANSPORT_P2P (1-GPU engines report P2P) */
  long barriers;            /* cross-GPU step barriers issued */
  double remote_kernel_ms;  /* timed fused launches that read remote buckets in-kernel (P2P) */
  double remote_bytes;      /* NVLink bytes those launches read */
} dg_engine_stats;

/* ncclGetUniqueId (call on rank 0, broadcast the 128 bytes to all ranks) */
int dg_nccl_unique_id(void* out128);
int dg_engine_create(const dg_engine_config* cfg, dg_engine** out);
/* Borrowed device pointer of buffer `which` of resident node `local_node`.
 * Valid until the next dg_engine_step: rounds with large mixing components
 * keep x double-buffered, so the DG_BUF_X pointer can alternate between steps. */
int dg_engine_buffer(dg_engine* e, int local_node, int which, float** dev_ptr);
/* Host <-> device copies of a node's buffer slice, ordered on the compute
 * stream.  upload is asynchronous (host memory must stay valid until the next
 * dg_engine_sync; pinned memory gives a true async copy); download synchronises. */
int dg_engine_upload(dg_engine* e, int local_node, int which, const float* host, size_t offset,
                     size_t count);
int dg_engine_download(dg_engine* e, int local_node, int which, float* host, size_t offset,
                       size_t count);
/* out[k] = buffer `which` of resident node `local_node` at element idx[k]
 * (host index array, n entries; synchronous).  Sampled checkpoints / parity
 * checks of full-size buckets without copying them whole. */
int dg_engine_gather(dg_engine* e, int local_node, int which, const uint64_t* idx, size_t n,
                     float* out);
/* Fill buffer `which` of every resident node with synthetic values of
 * StreamRng(seed, purpose, worker, iteration): worker = global node id when
 * per_node != 0, else 0 (shared x^(0), Alg. 1 line 1). */
int dg_engine_fill_synthetic(dg_engine* e, int which, uint64_t seed, uint32_t purpose,
                             int per_node, uint64_t iteration);
/* Consensus error of the current models over ALL nodes (collective: every rank
 * calls it; synchronous).  *dispersion = sum_i ||x_i - xbar||^2 with
 * xbar = (1/N) sum_i x_i (fp64 column sums, NCCL all-reduce across ranks);
 * *mean_sq = ||xbar||^2.  gossip_consensus's error[t] (topology.hpp:90-96) is
 * dispersion_t / dispersion_0. */
int dg_engine_consensus(dg_engine* e, double* dispersion, double* mean_sq);
/* Fixes xbar for every later dg_engine_consensus call to the CURRENT column
 * mean (collective, synchronous): gossip_consensus measures dispersion around
 * the preserved initial mean xbar^(0) (topology.hpp:90-94). */
int dg_engine_consensus_fix_mean(dg_engine* e);
/* One fused gossip + Adam step for iteration t (>= 1); asynchronous. */
int dg_engine_step(dg_engine* e, long t);
/* Steps t_first..t_last in order (the trainsim hot loop).
 * flags & DG_RUN_GRAPH: the range is captured once into a CUDA graph (cached
 * per (t_first, t_last) and starting x buffer) and replayed as one graph
 * launch -- for small buckets whose steps are launch-bound (BASELINE config
 * 1); DG_RUN_CAPTURE_ONLY: capture (no execution) so a later call replays.
 * Results are identical to calling dg_engine_step for each t. */
enum { DG_RUN_GRAPH = 1, DG_RUN_CAPTURE_ONLY = 2 };
int dg_engine_run_steps(dg_engine* e, long t_first, long t_last, int flags);
/* Bucketed step (the paper's per-bucket update U_k, PAPER.md:302-304 and
 * 1089-1095).  Updates elements [off, off+len) of every
 * resident node for iteration t -- mixing with round-t peers, Adam -- after
 * the round-t exchange of that range (pre-posted by the same range's call at
 * t-1, else posted now) has landed, then immediately posts the round-(t+1)
 * exchange of the updated range on the comm stream so it overlaps whatever
 * the caller does next (the rest of backward, the next forward).  Every rank
 * must call the same ranges in the same order; off must be a multiple of 64;
 * the ranges of one iteration must tile [0, d).  Requires DG_ENGINE_IN_PLACE. */
int dg_engine_step_range(dg_engine* e, long t, size_t off, size_t len);
/* Stream joins with a caller stream (cudaStream_t): wait_stream makes the
 * engine's streams wait for work already queued on `stream` (e.g. backward
 * producing g); join makes `stream` wait for the engine's queued updates
 * (e.g. the next forward reading x). */
int dg_engine_wait_stream(dg_engine* e, void* stream);
int dg_engine_join(dg_engine* e, void* stream);
/* Waits for all queued work; DG_DIVERGENCE (with iteration) if any step
 * produced a non-finite state; DG_NCCL_ERROR on an asynchronous NCCL error. */
int dg_engine_sync(dg_engine* e);
/* The engine's streams (cudaStream_t) for event timing by the caller. */
int dg_engine_streams(dg_engine* e, void** compute_stream, void** comm_stream);
int dg_engine_get_stats(const dg_engine* e, dg_engine_stats* out);
/* on != 0: bracket every fused launch with CUDA events on the compute stream;
 * durations are harvested into kernel_ms at dg_engine_sync.  on == 0 stops
 * and also resets kernel_ms / timed_launches / timed_hbm_bytes. */
int dg_engine_set_timing(dg_engine* e, int on);
/* Frees the engine.  COLLECTIVE for multi-GPU engines on the P2P transport:
 * every rank calls it (a final stream-ordered barrier keeps this rank's
 * exported x buffers mapped until every peer's last kernel has read them). */
void dg_engine_destroy(dg_engine* e);

/* ======================================================================
 * Runtime model: the discrete-event
 * per-iteration runtime recurrences of PAPER.md Appendix A.5 (All-Reduce and
 * decentralized) and A.8.1 (SGP variant), evaluated
 * verbatim; host only.  Unit time = one worker's forward pass with the global
 * batch; forward 1/N (All-Reduce: b/N unless `normalized`), backward 2/N per
 * bucket, theta per bucket update, gamma per bucket All-Reduce, omega*gamma per
 * decentralized round, p^(i,t) ~ N(1, sigma2) truncated to [0.5, 1.5] drawn
 * from StreamRng(seed, SpeedNoise, i, t) (rng.cpp:64-73).
 * ====================================================================== */
typedef struct dg_rm_params {
  int N, b;                  /* workers, buckets */
  double theta, gamma, omega, sigma2;
  int workers_per_node;      /* SGP variant grouping (divides N) */
  int normalized;            /* All-Reduce forward p/N instead of the paper-literal p*b/N */
  int allow_omega_above_one;
} dg_rm_params;
enum { DG_RM_ALLREDUCE = 0, DG_RM_DECENTRALIZED = 1, DG_RM_SGP = 2 };
/* runtimes[t-1] = max_i T_U^(i,t) - max_i T_U^(i,t-1) for t = 1..T.  schedule:
 * neighbour sets N_i^(t) for DECENTRALIZED / SGP (NULL = complete).  timeline
 * (optional): T x N x (1 + 3b) completion times F, B_1..B_b, U_1..U_b, C_1..C_b
 * (All-Reduce stores its single U in U_1). */
int dg_rm_simulate(int mode, const dg_rm_params* p, const dg_schedule* schedule, long T, uint64_t seed,
                   double* runtimes, double* timeline);
/* Eq. (3) best possible speedup */
int dg_rm_closed_form_speedup(double gamma, int N, int b, double theta, double* out);
/* p^(i,t) (rng.cpp:64-73 on StreamRng(seed, SpeedNoise, worker, iteration)) */
int dg_rm_speed_multiplier(uint64_t seed, uint64_t worker, uint64_t iteration, double sigma2, double* out);

/* ======================================================================
 * Host-only plan inspection (no GPU needed): the gossip exchange of one
 * round for one rank, as the engine issues it.  sends: (peer rank, global
 * node id whose bucket is sent); recvs: (peer rank, global node id received),
 * both ordered by (peer, node) so that NCCL's in-order per-peer matching pairs
 * them.  *nsend / *nrecv are set even when cap is too small.
 * ====================================================================== */
int dg_plan_exchange(const dg_schedule* s, int world_size, int rank, long round, int* send_peer,
                     int* send_node, int* nsend, int* recv_peer, int* recv_node, int* nrecv,
                     int cap);

#ifdef __cplusplus
}
#endif
#endif /* DG_H_ */
