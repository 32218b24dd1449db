/*
 * lsp_b200.h -- C-ABI of the B200-native LSP (d,r)-sparse projector path.
 *
 * This is the drop-in boundary for the hot path of the reference library
 * (lspkit `lsp_core`, /root/reference/proj).  Each entry point names the
 * reference interface it replaces (file:line under /root/reference).  Plain C
 * types only: host pointers where the reference takes lsp::Matrix /
 * lsp::SparseProjector by value, device pointers (and a caller-owned
 * cudaStream_t passed as void*) for the device-resident hot path.
 *
 * Naming follows the reference: `d` is the subspace width and `r` the number
 * of nonzeros per projector row (BASELINE.json calls them r and d).
 *
 * Conventions
 *  - Status: every function returns lsp_status; LSP_OK == 0.  The reference's
 *    exception taxonomy maps as  std::invalid_argument -> LSP_EINVAL,
 *    lsp::NumericError -> LSP_ENUMERIC, lsp::IoError -> LSP_EIO
 *    (proj/include/lsp/common.hpp:13-31).  lsp_last_error() returns the
 *    message of the last failure on the calling host thread.
 *  - Ownership: device buffers passed in are caller-owned; handles are
 *    library-owned and released with the matching *_destroy.  A pair keeps
 *    pointers to its two projectors (they must outlive it).
 *  - Asynchrony: functions taking a stream enqueue work on it and return
 *    without synchronising, unless documented as synchronous.
 *  - Threading: handles may be used from any host thread, but not
 *    concurrently on the same handle (one handle per layer).
 *  - Layout: dense matrices are row-major with an explicit leading dimension
 *    in ELEMENTS.  s x s subspace matrices (S, delta, Adam moments) may be
 *    passed in the reference layout (LSP_LAYOUT_ROW: X[a][b] at a*d+b) or
 *    transposed (LSP_LAYOUT_T: X[a][b] at b*d+a), the layout the fused device
 *    path uses internally.
 */
#ifndef LSP_B200_H_
#define LSP_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSP_B200_VERSION 1

typedef enum {
  LSP_OK = 0,
  LSP_EINVAL = 1,   /* std::invalid_argument */
  LSP_ENUMERIC = 2, /* lsp::NumericError */
  LSP_EIO = 3,      /* lsp::IoError */
  LSP_ECUDA = 4,    /* CUDA runtime failure (incl. no device) */
  LSP_ENOMEM = 5,
  LSP_ENCCL = 6     /* NCCL missing or failed (lsp_comm_*, *_allreduce) */
} lsp_status;

typedef enum { LSP_F64 = 0, LSP_F32 = 1, LSP_BF16 = 2 } lsp_dtype;
typedef enum { LSP_LAYOUT_ROW = 0, LSP_LAYOUT_T = 1 } lsp_layout;
/* proj/include/lsp/projector.hpp:38-41 */
typedef enum { LSP_REG_SQUARED = 0, LSP_REG_UNSQUARED = 1 } lsp_reg_kind;
/* proj/include/lsp/subspace_opt.hpp:39-42 */
typedef enum { LSP_TRANSFER_ENTRYWISE = 0, LSP_TRANSFER_MATRIX = 1 } lsp_transfer_kind;

typedef struct lsp_projector_s* lsp_projector_t; /* device SparseProjector (CSR + CSC) */
typedef struct lsp_pair_s* lsp_pair_t;           /* ProjectorPair + device workspace   */
typedef struct lsp_adam_s* lsp_adam_t;           /* device SubspaceOptState            */
typedef struct lsp_layer_s* lsp_layer_t;         /* per-layer schedule unit            */
typedef void* lsp_stream_t;                      /* cudaStream_t (NULL = legacy stream) */

/* proj/include/lsp/projector.hpp:43-51 */
typedef struct {
  double alpha;
  double reg_beta;
  double step_size;
  int max_steps;
  int timeout_steps;
  uint64_t seed;
  int reg_kind; /* lsp_reg_kind */
} lsp_fit_config;

/* proj/include/lsp/projector.hpp:53-60 (loss_curve returned separately) */
typedef struct {
  double final_rel_bias;
  int success;
  int timed_out;
  int stalled;
  int steps;
  int n_loss; /* total entries of the loss curve (may exceed max_curve) */
} lsp_fit_report;

/* ----------------------------------------------------------------------------
 * Library / device
 * -------------------------------------------------------------------------- */
const char* lsp_last_error(void);
int lsp_version(void);
/* Synchronous: number of usable CUDA devices (0 without a GPU). */
int lsp_device_count(int* count);
/* Number of kernels this library has launched in this process (all handles);
 * used by bench.py to report gpu_launches. */
uint64_t lsp_launch_count(void);
/* Process-wide cap on the SMs the persistent kernels of each phase size their
 * grids for (0 = all SMs): compress_sms for stage 1 of compress, update_sms
 * for the decompress-and-apply stream.  Lets a caller run the compress of one
 * layer and the update of another concurrently on two streams (schedule.py,
 * concurrent mode) without one persistent grid starving the other.  No
 * reference counterpart (the reference runs these serially on the CPU). */
int lsp_set_sm_budget(int compress_sms, int update_sms);
/* Default values of lsp_fit_config (projector.hpp:43-51). */
lsp_fit_config lsp_fit_config_default(void);

/* ----------------------------------------------------------------------------
 * Host-side projector construction and text I/O (no GPU needed)
 * -------------------------------------------------------------------------- */
/* proj/include/lsp/common.hpp:42-45 */
uint64_t lsp_derive_seed(uint64_t master, uint64_t tag, uint64_t index);
/* proj/src/projector.cpp:66-85 -- bit-exact positions and values (mt19937_64,
 * partial Fisher-Yates, Box-Muller).  pos/val hold n_rows*r entries. */
int lsp_init_sparse(int n_rows, int d, int r, uint64_t seed, int32_t* pos, double* val);
/* proj/src/projector.cpp:87-96 (d = n_rows, r = 1, value 1) */
int lsp_identity_pattern(int n_rows, int32_t* pos, double* val);
/* proj/src/projector.cpp:317-327.  Writes up to cap bytes (NUL-terminated) and
 * returns, via *needed, the full size including the NUL. */
int lsp_save_projector(int n_rows, int d, int r, const int32_t* pos, const double* val,
                       char* buf, int64_t cap, int64_t* needed);
/* proj/src/projector.cpp:329-354.  Two calls: with pos == NULL only the header
 * is parsed into *n_rows, *d, *r; then again with arrays of n_rows*r entries.
 * Malformed input -> LSP_EIO with the reference's messages. */
int lsp_load_projector(const char* text, int64_t len, int* n_rows, int* d, int* r,
                       int32_t* pos, double* val);
/* proj/src/trainer.cpp:60-72 */
int lsp_subsample_size(double gamma_bound, double chernoff_beta, int m, int n,
                       int total_steps, double delta, int64_t* out);

/* ----------------------------------------------------------------------------
 * Device projectors and pairs
 * -------------------------------------------------------------------------- */
/* Uploads a SparseProjector (proj/include/lsp/projector.hpp:18-30): validates
 * it like load_projector (positions in [0,d), strictly ascending per row,
 * finite values) and builds the CSR and CSC device arrays.  compute = LSP_F32
 * or LSP_F64 selects the value/accumulator precision of every kernel that
 * uses this projector. Synchronous. */
int lsp_projector_create(int n_rows, int d, int r, const int32_t* pos, const double* val,
                         lsp_dtype compute, lsp_projector_t* out);
/* Replace the values (positions are frozen, as in fit). Synchronous. */
int lsp_projector_set_values(lsp_projector_t p, const double* val);
/* Download positions and values (either may be NULL). Synchronous. */
int lsp_projector_get(lsp_projector_t p, int32_t* pos, double* val);
int lsp_projector_shape(lsp_projector_t p, int* n_rows, int* d, int* r);
int lsp_projector_destroy(lsp_projector_t p);

/* ProjectorPair (projector.hpp:32-36); P has m rows, Q has n rows.
 * P.d != Q.d -> LSP_EINVAL ("projector pair: P.d != Q.d", projector.cpp:20-23). */
int lsp_pair_create(lsp_projector_t p, lsp_projector_t q, lsp_pair_t* out);
int lsp_pair_destroy(lsp_pair_t pair);

/* Generic sparse products with one projector P (n_rows x d when densified),
 * proj/src/projector.cpp:105-161.  x and out are device matrices in the
 * projector's compute dtype:
 *   LSP_LEFT     out (n_rows x cols) = P   x (d x cols)        left_mul
 *   LSP_LEFT_T   out (d x cols)      = P^T x (n_rows x cols)   leftT_mul
 *   LSP_RIGHT    out (rows x d)      = x (rows x n_rows) P     right_mul
 *   LSP_RIGHT_T  out (rows x n_rows) = x (rows x d) P^T        rightT_mul
 * `rows`/`cols` give the free dimension of x (cols for LEFT*, rows for RIGHT*). */
typedef enum { LSP_LEFT = 0, LSP_LEFT_T = 1, LSP_RIGHT = 2, LSP_RIGHT_T = 3 } lsp_mul_op;
int lsp_projector_mul(lsp_projector_t p, int op, int free_dim, const void* x, int64_t ldx,
                      void* out, int64_t ldo, lsp_stream_t stream);

/* ----------------------------------------------------------------------------
 * Hot path (device pointers, asynchronous on `stream`)
 * -------------------------------------------------------------------------- */
/* compress: S = P^T G Q  (projector.cpp:163-168).  g is m x n (ldg elements)
 * of g_dtype; s is d x d in the pair's compute dtype and the given layout. */
int lsp_compress(lsp_pair_t pair, const void* g, int64_t ldg, lsp_dtype g_dtype, void* s,
                 lsp_layout s_layout, lsp_stream_t stream);
/* decompress: out = P S Q^T  (projector.cpp:170-175); out is m x n of out_dtype. */
int lsp_decompress(lsp_pair_t pair, const void* s, lsp_layout s_layout, void* out,
                   int64_t ldo, lsp_dtype out_dtype, lsp_stream_t stream);
/* Fused decompress-and-apply: w -= lr * P delta Q^T in one read-modify-write
 * pass over w (the apply of proj/src/trainer.cpp:190). */
int lsp_decompress_apply(lsp_pair_t pair, const void* delta, lsp_layout delta_layout,
                         double lr, void* w, int64_t ldw, lsp_dtype w_dtype,
                         lsp_stream_t stream);
/* estimation_bias: out = P P^T sigma Q Q^T - sigma  (projector.cpp:177-181). */
int lsp_estimation_bias(lsp_pair_t pair, const void* sigma, int64_t lds, lsp_dtype dtype,
                        void* out, int64_t ldo, lsp_stream_t stream);
/* relative_bias: |b(sigma)|_F / |sigma|_F (projector.cpp:183-187).
 * SYNCHRONOUS (returns a host double). Zero sigma -> LSP_EINVAL. */
int lsp_relative_bias(lsp_pair_t pair, const void* sigma, int64_t lds, lsp_dtype dtype,
                      double* out, lsp_stream_t stream);

/* ----------------------------------------------------------------------------
 * Subspace Adam (proj/include/lsp/subspace_opt.hpp:17-37)
 * -------------------------------------------------------------------------- */
/* make_opt_state(rows, cols, beta1, beta2, eps) (subspace_opt.cpp:17-33);
 * moments zero-initialised on the device in the given compute dtype and
 * stored in `layout` (the fused path, lsp_step/lsp_update, needs LSP_LAYOUT_T). */
int lsp_adam_create(int rows, int cols, double beta1, double beta2, double eps,
                    lsp_dtype compute, lsp_layout layout, lsp_adam_t* out);
int lsp_adam_destroy(lsp_adam_t st);
/* adam_step (subspace_opt.cpp:35-57): grad (device, rows x cols, compute dtype,
 * same layout as the stored moments) -> moments updated in place, delta
 * (bias-corrected M/(sqrt(V)+eps), no learning rate) written to `delta`.
 * A non-finite gradient leaves M, V and delta untouched and latches a device
 * flag that lsp_adam_check reports as LSP_ENUMERIC (reference semantics:
 * NumericError before any state change). */
int lsp_adam_step(lsp_adam_t st, const void* grad, void* delta, lsp_stream_t stream);
/* SYNCHRONOUS: LSP_ENUMERIC if a non-finite gradient was seen since the last
 * check (and clears the flag), else LSP_OK. */
int lsp_adam_check(lsp_adam_t st, lsp_stream_t stream);
/* SYNCHRONOUS host copies of the state as doubles in the given layout. */
int lsp_adam_get(lsp_adam_t st, double* m, double* v, int64_t* step, lsp_layout layout);
int lsp_adam_set(lsp_adam_t st, const double* m, const double* v, int64_t step,
                 lsp_layout layout);
int lsp_adam_info(lsp_adam_t st, int* rows, int* cols, double* beta1, double* beta2,
                  double* eps);

/* ----------------------------------------------------------------------------
 * Fused per-matrix step: compress -> Adam -> decompress-and-apply, i.e. one
 * iteration of the per-layer loop of proj/src/trainer.cpp:187-190, with S,
 * the moments and delta kept in the transposed device layout.  `s_out` (may
 * be NULL) receives S^T.  The Adam state must be d x d.
 * -------------------------------------------------------------------------- */
int lsp_step(lsp_pair_t pair, lsp_adam_t st, const void* g, int64_t ldg, lsp_dtype g_dtype,
             void* w, int64_t ldw, lsp_dtype w_dtype, double lr, void* s_out,
             lsp_stream_t stream);
/* Data-parallel split of lsp_step: the caller all-reduces the S^T produced by
 * lsp_compress(..., LSP_LAYOUT_T, ...) (mean over ranks), then calls
 * lsp_update to run Adam and the decompress-and-apply. */
int lsp_update(lsp_pair_t pair, lsp_adam_t st, const void* s_t, void* w, int64_t ldw,
               lsp_dtype w_dtype, double lr, lsp_stream_t stream);

/* ----------------------------------------------------------------------------
 * Per-layer schedule (the body of proj/src/trainer.cpp:186-198 for every
 * linear layer of a block): up to 16 pairs sharing d, r and the compute dtype,
 * stepped with ONE grouped launch per stage.  The layer owns contiguous
 * S^T / delta^T buffers and the Adam moments of all its matrices (beta/eps as
 * make_opt_state), so a data-parallel caller all-reduces a whole layer's S
 * with a single collective between lsp_layer_compress and lsp_layer_update.
 * -------------------------------------------------------------------------- */
int lsp_layer_create(int count, const lsp_pair_t* pairs, double beta1, double beta2, double eps,
                     lsp_layer_t* out);
int lsp_layer_destroy(lsp_layer_t layer);
/* Bind matrix idx's gradient G (m x n) and weight W (m x n); all matrices of a
 * layer must share the G dtype and the W dtype. */
int lsp_layer_bind(lsp_layer_t layer, int idx, const void* g, int64_t ldg, lsp_dtype g_dtype,
                   void* w, int64_t ldw, lsp_dtype w_dtype);
/* Device pointer to the layer's contiguous S^T buffer (count blocks of d x d,
 * compute dtype) and its element count. */
int lsp_layer_s_buffer(lsp_layer_t layer, void** s_t, int64_t* count);
/* S^T_i = (P_i^T G_i Q_i)^T for every matrix (latches the non-finite flag). */
int lsp_layer_compress(lsp_layer_t layer, lsp_stream_t stream);
/* lsp_layer_compress in two enqueued halves (in this order, on any streams
 * ordered by the caller): stage 1 Z^T_i = G_i^T P_i of every matrix (the pass
 * over G), then stage 2 S^T_i = Q_i^T Z^T_i plus the non-finite latch.  Lets a
 * schedule run stage 2 and Adam of one layer beside the Y build of another.
 * Replaces: right_mul then leftT_mul, proj/src/projector.cpp:119-168. */
int lsp_layer_compress_prepare(lsp_layer_t layer, lsp_stream_t stream);
int lsp_layer_compress_finish(lsp_layer_t layer, lsp_stream_t stream);
/* Single-rank forms (no S exchange between compress and Adam): compress (or
 * its stage 2) with the layer's Adam fused into the stage-2 epilogue, i.e.
 * lsp_layer_compress + lsp_layer_adam(check 0) (resp. _compress_finish +
 * _adam) in one launch fewer, bitwise the same S, delta, moments and step.
 * The moments live in a ping-pong pair flipped by the launch's last CTA, only
 * when the layer's S was finite (a non-finite layer keeps its moments and step
 * and latches the flag, as lsp_layer_adam would skip).  Groups the fused
 * kernel does not cover (fp64, d % 4 != 0, LSP_FUSE_ADAM=0) run the unfused
 * pair.  Replaces: compress + adam_step, proj/src/trainer.cpp:186-189. */
int lsp_layer_compress_adam(lsp_layer_t layer, lsp_stream_t stream);
int lsp_layer_compress_finish_adam(lsp_layer_t layer, lsp_stream_t stream);
/* Adam on the layer's S^T (optionally re-checking finiteness, e.g. after an
 * all-reduce) and W_i -= lr * P_i delta_i Q_i^T; skipped if the flag is set. */
int lsp_layer_update(lsp_layer_t layer, double lr, int check_finite, lsp_stream_t stream);
/* The two halves of lsp_layer_update: Adam -> delta^T, then the fused
 * decompress-and-apply of every matrix (one grouped launch each).  With
 * check_finite the re-check runs inside the Adam launch (the moments'
 * ping-pong pair is flipped only when every S element was finite). */
int lsp_layer_adam(lsp_layer_t layer, int check_finite, lsp_stream_t stream);
int lsp_layer_apply(lsp_layer_t layer, double lr, lsp_stream_t stream);
/* compress + update. */
/* lsp_layer_apply in two enqueued halves (same stream, in this order): the
 * Y = delta Q^T build of every matrix, then the streaming apply that reads it.
 * For groups the Y path does not cover, _prepare enqueues nothing and _finish
 * runs the whole apply.  Lets a caller time or overlap the halves.
 * Replaces: decompress (rightT_mul then left_mul) + apply, proj/src/projector.cpp:170-175,
 * proj/src/trainer.cpp:190. */
int lsp_layer_apply_prepare(lsp_layer_t layer, lsp_stream_t stream);
int lsp_layer_apply_finish(lsp_layer_t layer, double lr, lsp_stream_t stream);
int lsp_layer_step(lsp_layer_t layer, double lr, lsp_stream_t stream);
/* SYNCHRONOUS: LSP_ENUMERIC if a non-finite S was seen (clears the flag). */
int lsp_layer_check(lsp_layer_t layer, lsp_stream_t stream);
/* SYNCHRONOUS host copy of matrix idx's moments and the shared step. */
int lsp_layer_adam_get(lsp_layer_t layer, int idx, double* m, double* v, int64_t* step,
                       lsp_layout layout);

/* ----------------------------------------------------------------------------
 * Data-parallel exchange (SURVEY 8(b) lsp_allreduce_S, 8(e)).  The reference
 * steps one process (proj/src/trainer.cpp:186-198: compress -> adam_step ->
 * apply per layer); across ranks only S is exchanged, between compress and
 * Adam: mean(S_rank) == compress(mean G_rank) by linearity
 * (proj/tests/test_projector.cpp:208-235).  The library owns the NCCL
 * communicator; NCCL is loaded at run time (libnccl.so.2, reusing a copy
 * already in the process, e.g. PyTorch's).
 * -------------------------------------------------------------------------- */
#define LSP_COMM_ID_BYTES 128 /* sizeof(ncclUniqueId) */
typedef struct lsp_comm_s* lsp_comm_t;
/* Rank 0 creates the id and ships its LSP_COMM_ID_BYTES bytes to every rank. */
int lsp_comm_unique_id(void* id_out);
/* Collective over all ranks (ncclCommInitRank); the device is the caller's
 * current CUDA device. */
int lsp_comm_init(const void* id, int nranks, int rank, lsp_comm_t* out);
int lsp_comm_destroy(lsp_comm_t comm);
int lsp_comm_size(lsp_comm_t comm, int* nranks, int* rank);
int lsp_nccl_version(int* version);
/* In-place mean over ranks of count elements (ncclAllReduce, ncclAvg) on stream. */
int lsp_allreduce_mean(lsp_comm_t comm, void* buf, int64_t count, lsp_dtype dtype,
                       lsp_stream_t stream);
/* The layer's whole S^T buffer (lsp_layer_s_buffer) averaged over ranks on
 * `stream`, then re-checked for non-finite values so that every rank latches
 * the layer's flag together (call between lsp_layer_compress and
 * lsp_layer_update/_adam; enqueue on the compress stream or join with events). */
int lsp_layer_allreduce(lsp_layer_t layer, lsp_comm_t comm, lsp_stream_t stream);

/* ----------------------------------------------------------------------------
 * Multi-layer step schedule (SURVEY 8(b) lsp_schedule_*): the layer-wise
 * pipeline the reference only models (build_lsp_layerwise,
 * proj/src/schedule_sim.cpp:255-283) in place of its sequential per-layer loop
 * (proj/src/trainer.cpp:186-198).  One step, layers in backward order:
 * [backward(l) on the caller's stream] -> compress(l) -> all-reduce(S_l) on a
 * comm stream (when comm != NULL) -> Adam + apply of layer l+1, with the
 * all-reduce of layer l overlapping the compress of layer l-1.  With a
 * backward callback the LSP work runs on the schedule's own stream, compress(l)
 * gated by an event recorded after backward(l), and the caller's stream joins
 * it at the end.  Side streams are forked from and joined into `stream` by
 * events, so a step can be captured in a CUDA graph.
 * -------------------------------------------------------------------------- */
typedef struct lsp_schedule_s* lsp_schedule_t;
/* Enqueue the backward of layer `layer` (producing its bound gradients) on `stream`. */
typedef void (*lsp_backward_fn)(int layer, lsp_stream_t stream, void* user);
/* layers in forward order; comm may be NULL (single rank, no exchange). */
int lsp_schedule_create(int count, const lsp_layer_t* layers, lsp_comm_t comm, lsp_schedule_t* out);
int lsp_schedule_set_backward(lsp_schedule_t sched, lsp_backward_fn fn, void* user);
/* mode 1: stage 2 (lsp_layer_compress_finish), the all-reduce and Adam of layer
 * l on a side stream beside the Y build of layer l+1; mode 2: beside its Y
 * build and apply; 0 (default): the order above.  Exclusive with a backward
 * callback.  Results are bitwise those of mode 0. */
int lsp_schedule_set_pipeline(lsp_schedule_t sched, int mode);
/* Spatial partition: split the device's SMs into two green contexts,
 * `compress_sms` (rounded up by the driver: multiples of 8 on sm_100) running
 * stage 1 of every layer back to back, the rest running, per layer as soon as
 * its stage 1 is done, stage 2, the all-reduce, Adam, the Y build and the
 * apply (the L2-bound compress and the HBM-bound apply side by side on
 * disjoint SMs).  0 removes the partition.  got_compress / got_update (may be
 * NULL) receive the SM counts provisioned.  Exclusive with the backward and
 * pipeline modes; same kernels on the same data, so bitwise the results of
 * mode 0. */
int lsp_schedule_set_partition(lsp_schedule_t sched, int compress_sms, int* got_compress, int* got_update);
int lsp_schedule_step(lsp_schedule_t sched, double lr, lsp_stream_t stream);
int lsp_schedule_destroy(lsp_schedule_t sched);

/* ----------------------------------------------------------------------------
 * Projector fit (proj/src/projector.cpp:189-315), on the device in fp64.
 * targets: T device pointers to m x n matrices (ld, dtype shared).
 * -------------------------------------------------------------------------- */
/* fit_loss (projector.cpp:189-198). SYNCHRONOUS. */
int lsp_fit_loss(lsp_pair_t pair, const void* const* targets, int t, int64_t ld,
                 lsp_dtype dtype, const lsp_fit_config* cfg, double* loss, lsp_stream_t stream);
/* fit_gradient (projector.cpp:200-236): host arrays laid out like values
 * (m*r and n*r). SYNCHRONOUS. */
int lsp_fit_gradient(lsp_pair_t pair, const void* const* targets, int t, int64_t ld,
                     lsp_dtype dtype, const lsp_fit_config* cfg, double* grad_p,
                     double* grad_q, lsp_stream_t stream);
/* fit (projector.cpp:253-315): updates the pair's projector values in place.
 * loss_curve (may be NULL) receives up to max_curve losses. SYNCHRONOUS. */
int lsp_fit(lsp_pair_t pair, const void* const* targets, int t, int64_t ld, lsp_dtype dtype,
            const lsp_fit_config* cfg, lsp_fit_report* report, double* loss_curve,
            int max_curve, lsp_stream_t stream);

/* ----------------------------------------------------------------------------
 * Optimizer-state transfer after a refit (proj/src/subspace_opt.cpp:59-101)
 * -------------------------------------------------------------------------- */
/* projector_gram: out = A^T B (A.d x B.d, row-major fp64, device). */
int lsp_projector_gram(lsp_projector_t a, lsp_projector_t b, double* out,
                       lsp_stream_t stream);
/* reproject_state: M <- (Pn^T Po) M (Qo^T Qn), V likewise with entrywise- or
 * matrix-squared transfer maps, clamped at zero.  In place on `st`. */
int lsp_reproject_state(lsp_adam_t st, lsp_pair_t old_pair, lsp_pair_t new_pair,
                        lsp_transfer_kind kind, lsp_stream_t stream);

/* ----------------------------------------------------------------------------
 * Bias-gated refresh: maybe_update (proj/src/trainer.cpp:74-112; result struct
 * proj/include/lsp/trainer.hpp:95-104).  Keeps the pair when the relative bias
 * on grad_sub is <= alpha; otherwise draws a fresh pair with init_sparse
 * (seeds derive_seed(reinit_seed, 1 | 2)), fits it on grad_sub plus the
 * non-zero extra targets (fit seed derive_seed(reinit_seed, 3)), and
 * reprojects `st` IN PLACE into the new subspace.  On refresh the new
 * projectors and pair are returned (caller-owned; the old ones are untouched),
 * otherwise *new_p = *new_q = *new_pair = NULL.  A zero grad_sub skips the
 * check (bias NaN).  SYNCHRONOUS.
 * -------------------------------------------------------------------------- */
typedef struct {
  int refreshed;
  int fit_timed_out; /* fit report timed_out || stalled */
  int skipped_zero_grad;
  int fit_steps;
  double bias_before;
  double bias_after;
} lsp_maybe_update_result;
int lsp_maybe_update(lsp_pair_t pair, lsp_adam_t st, const void* grad_sub, int64_t ld,
                     lsp_dtype dtype, const void* const* extra, int n_extra, int r,
                     double alpha, const lsp_fit_config* fit_cfg, lsp_transfer_kind transfer,
                     uint64_t reinit_seed, lsp_projector_t* new_p, lsp_projector_t* new_q,
                     lsp_pair_t* new_pair, lsp_maybe_update_result* res, lsp_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* LSP_B200_H_ */
