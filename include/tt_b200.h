/*
 * tt_b200.h -- C ABI of the B200-native hot path of arXiv 2211.08770
 * ("TT-format orthogonalization": TT-rounding of rank-inflated TT-sums plus batched
 * TT inner products, and the six orthogonalization kernels built on them).
 *
 * Every entry point below is implemented by hand-written sm_100a CUDA kernels in
 * libtt_b200.so (paper_2211_08770_b200/csrc).  No torch types cross this boundary:
 * plain pointers (host or device, as stated per argument) and sizes.
 *
 * Conventions (all calls)
 *   - fp64 everywhere ("u_64 ~ 1e-16 for 64-bit calculation").
 *   - A TT-vector of order d has cores X_k of shape (r_{k-1}, n_k, r_k), r_0 = r_d = 1
 *     (PAPER.md:41-45), stored contiguously in C order with r_k fastest:
 *     element (a, i, b) of core k is core[k][(a * n_k + i) * r_k + b].
 *   - Canonical indices are 1-based psi order, mode 1 fastest.
 *   - Dense m x m outputs (R, Gram) are row-major.
 *   - Calls are enqueued on the context's stream.  Calls that return host scalars or
 *     data-dependent ranks (tt_round*, tt_orth, tt_norm, tt_download) synchronise that
 *     stream; tt_dot_batch, tt_gram, tt_gram_blocks, tt_element do not (device outputs).
 *   - Errors: every call returns a tt_status; TT_OK = 0.  tt_last_error(ctx) returns a
 *     NUL-terminated description of the last failure on that context (owned by ctx,
 *     valid until the next call on it).  No call throws or aborts.
 *   - Value range: the path forms squared norms (column masses, Householder and Jacobi
 *     quantities), so a tensor and every term of a sum must have its Frobenius norm within
 *     about 1e-120 .. 1e120 (roundings checked against the oracle at 1e-120 and 1e140,
 *     tests/test_gpu_batch.py; the drivers against the closed form at 1e-100 and 1e100,
 *     tools/orth_scale_probe.py); a rounding whose ||x|| comes out non-finite fails with
 *     TT_EINVAL.  Scale such inputs by a power of two first (exact).
 *   - Ownership: tt_view arguments are BORROWED (never written; must stay valid until the
 *     call returns).  tt_tensor results are allocated by the library (their ranks are
 *     data-dependent) from the context's stream-ordered pool; release with
 *     tt_tensor_free.  Dense outputs go to caller buffers.
 */
#ifndef TT_B200_H
#define TT_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TT_API __attribute__((visibility("default")))
#else
#define TT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TT_OK = 0,
  TT_EINVAL = 1,          /* bad argument (null pointer, negative size, ...) */
  TT_ESHAPE = 2,          /* operands disagree in order / mode sizes / ranks */
  TT_EINDEX = 3,          /* canonical index outside 1..prod(n) */
  TT_ENOMEM = 4,          /* device allocation failed */
  TT_ECUDA = 5,           /* CUDA runtime error (text in tt_last_error) */
  TT_ENOCONV = 6,         /* Jacobi SVD exceeded its sweep limit */
  TT_ESINGULAR_GRAM = 7,  /* Cholesky of the Gram matrix met a pivot <= 0 */
  TT_ELINDEP = 8,         /* ||p|| <= 1e3 u ||a_i||: linear dependence */
  TT_ENUMDEFECT = 9,      /* ||a||^2 - s < -1e-12 ||a||^2 in TTH-vec (literal beta) */
  TT_ENOTSUP = 10,        /* shape outside what this build supports (message says which) */
  TT_ECOMM = 11           /* a collective of the attached communicator failed (or NCCL missing) */
} tt_status;

typedef struct tt_ctx_s* tt_ctx;
typedef struct tt_tensor_s* tt_tensor;
typedef struct tt_batch_s* tt_batch;

/* A borrowed TT-vector.  n[d], r[d+1] and the array core[d] are HOST arrays; core[k]
 * points to DEVICE memory except for tt_upload (host memory).  norm = ||y|| when known
 * (used for the pre-cancellation scale s(x) of the noise floor), NaN when unknown
 * (the library then computes it). */
typedef struct {
  int32_t d;
  const int64_t* n;
  const int64_t* r;
  const double* const* core;
  double norm;
} tt_view;

/* TT-rounding options (||x - x~|| <= delta ||x||).
 *   rel_tol  delta >= 0.  Per-split threshold tau = max(delta ||x|| / sqrt(d-1),
 *            floor_c * u * s(x)) with s(x) = sum_l |c_l| ||y_l||.
 *            delta = 0: no truncation, no floor (structural ranks kept).
 *   max_rank 0 = none; else every rank is capped (SPEC.md:246 MaxRank mode).
 *   floor_c  noise-floor constant; 0 = paper-pure threshold.  Default 2048.
 *   qrcp_theta  truncated-SVD stopping fraction theta in (0,1]; 0 selects 0.5.  The
 *            decision equals the exact-SVD decision.
 *   rank_revealing  1 (default): the right-to-left sweep uses column-pivoted Householder QR
 *            stopped at the panel's numerical rank in working precision (trailing block
 *            <= 16 u ||A_k||_F); 0: full Householder QR (structural ranks).  Ignored
 *            when rel_tol = 0 (always full). */
typedef struct {
  double rel_tol;
  int64_t max_rank;
  double floor_c;
  double qrcp_theta;
  int32_t rank_revealing;
} tt_round_opts;

typedef struct {
  double norm;   /* ||x|| = ||C_1||_F after the right-to-left sweep */
  double scale;  /* s(x) */
  double tau;    /* per-split threshold used */
  int64_t qrcp_steps;   /* total column-pivoted Householder steps over all splits */
  int64_t resumes;      /* ambiguous decisions resolved by resuming the QRCP */
} tt_round_info;

typedef enum { TT_CGS = 0, TT_MGS = 1, TT_CGS2 = 2, TT_MGS2 = 3, TT_GRAM = 4, TT_HOUSEHOLDER = 5 } tt_orth_kind;

typedef struct {
  tt_round_opts round;
  int32_t hh_beta_literal;  /* 0: R(i,i) = sign * ||round(w - sum_{j<i} r_j e_j)||;
                               1: literal sqrt(||w||^2 - s) of Alg. 6 line 10 */
  int32_t want_loo;         /* fill report->loo_per_step (costs the Q Gram) */
  int32_t hh_mask;          /* Householder only, a DEPARTURE from Alg. 6 lines 4-9:
                               the first TTH-vec rounding takes w with its entries phi(1..i-1) zeroed
                               exactly (Hadamard product with a rank-2 comparison mask) instead of
                               the cancelling TT-sum w - sum_{j<i} r(j) e_j.  0 = Alg. 6 as listed. */
} tt_orth_opts;

typedef struct {
  int64_t rounding_calls;      /* Table 1 ledger */
  int32_t fail_index;          /* 0-based step of a breakdown, -1 otherwise */
  double* loo_per_step;        /* HOST, m entries or NULL: ||I_k - Q_k^T Q_k||_2, Eq. (9) */
  int64_t* max_rank_per_call;  /* HOST or NULL: max output rank of each rounding call (sized
                                  by the Table 1 count) */
  tt_tensor* householder_u;    /* HOST array of m handles or NULL: Householder TT-vectors */
} tt_orth_report;

/* ---------------------------------------------------------------- context */
/* device: CUDA ordinal; stream: a cudaStream_t (NULL = legacy default stream). */
TT_API tt_status tt_ctx_create(int device, void* stream, tt_ctx* out);
TT_API tt_status tt_ctx_destroy(tt_ctx ctx);
TT_API tt_status tt_ctx_set_stream(tt_ctx ctx, void* stream);
TT_API const char* tt_last_error(tt_ctx ctx);
TT_API const char* tt_status_string(tt_status s);
/* Number of this library's kernels launched on ctx so far (evidence for bench.py). */
TT_API int64_t tt_ctx_launch_count(tt_ctx ctx);
/* Stream-synchronise ctx. */
TT_API tt_status tt_ctx_sync(tt_ctx ctx);
/* Per-kernel-class timing with CUDA events recorded on the ctx stream around every
 * launch of this library.  enable = 1 starts (and resets) collection, 0 stops it. */
TT_API tt_status tt_ctx_profile(tt_ctx ctx, int32_t enable);
/* Class idx (0-based; TT_EINDEX past the end): name (copied into name_buf, NUL-terminated,
 * truncated to name_len), launches, summed event milliseconds, and the algorithmic flops
 * and bytes of those launches (the work model of DESIGN.md).  Synchronises the stream. */
TT_API tt_status tt_ctx_profile_query(tt_ctx ctx, int32_t idx, char* name_buf, int32_t name_len,
                                      int64_t* launches, double* ms, double* flops, double* bytes);

/* ---------------------------------------------------------------- tensors */
/* View of a library tensor: pointers stay valid until tt_tensor_free. */
TT_API tt_status tt_tensor_view(tt_tensor t, tt_view* out);
TT_API tt_status tt_tensor_free(tt_ctx ctx, tt_tensor t);
/* Copy a host TT (view with HOST core pointers) to a new device tensor. */
TT_API tt_status tt_upload(tt_ctx ctx, const tt_view* host, tt_tensor* out);
/* Copy a device tensor to caller host buffers host_cores[k] (sized r_{k-1} n_k r_k). */
TT_API tt_status tt_download(tt_ctx ctx, tt_tensor t, double* const* host_cores);

/* ---------------------------------------------------------------- TT algebra */
/* x = sum_{l<K} coeff[l] terms[l], materialised (ranks add; first cores
 * concatenated horizontally with c_l applied, interior block-diagonal, last vertical).
 * coeff: HOST. */
TT_API tt_status tt_sum(tt_ctx ctx, int32_t K, const double* coeff, const tt_view* terms, tt_tensor* out);
/* out = alpha x + y. */
TT_API tt_status tt_axpy(tt_ctx ctx, double alpha, const tt_view* x, const tt_view* y, tt_tensor* out);
/* y = A x for a TT-matrix A (the paper's Krylov workload: x_{j+1} = -Delta_d a_j).
 * A: a view whose core k holds the operator core (ra_k, n_k, n_k, ra_{k+1}) row-major (row index
 * i, then column index j, then ra_{k+1} fastest), passed with modes A->n[k] = n_k^2 (ESHAPE
 * otherwise); x: DEVICE TT-vector with modes n_k.  out: new library tensor with ranks
 * ra_k rx_k, cores Y_k((a, alpha), i, (b, beta)) = sum_j A_k(a, i, j, b) X_k(alpha, j, beta). */
TT_API tt_status tt_matvec(tt_ctx ctx, const tt_view* A, const tt_view* x, tt_tensor* out);
/* out_dev[p] = <x[p], y[p]> for p < P (PAPER.md:19 Euclidean dot through the contraction;
 * W_k = sum_i X_k(i)^T W_{k-1} Y_k(i)).  out_dev: DEVICE, P doubles. */
TT_API tt_status tt_dot_batch(tt_ctx ctx, int32_t P, const tt_view* x, const tt_view* y, double* out_dev);
/* G(i,j) = <a_i, a_j> (Alg. 5 lines 2-6, Eq. (3)); G_dev: DEVICE m*m row-major, symmetric.
 * With a communicator of N ranks attached (tt_ctx_comm_*; N = 1 runs the same path), every rank calls with
 * the same set: the lower triangle is cut into 4 x 4 pair blocks (tt_plan_gram_blocks), each rank
 * evaluates the blocks the LPT plan gives it, one all-gather combines them and every rank
 * receives the whole G.  Ordered on the ctx stream (NCCL). */
TT_API tt_status tt_gram(tt_ctx ctx, int32_t m, const tt_view* a, double* G_dev);
/* Pair blocks of the Gram matrix for sharding: blk (HOST) holds nblk quadruples
 * (i0, j0, bi, bj); block b writes bi*bj doubles <a_{i0+s}, a_{j0+t}> row-major (s,t)
 * at packed_dev + sum of previous block sizes.  packed_dev: DEVICE. */
TT_API tt_status tt_gram_blocks(tt_ctx ctx, int32_t m, const tt_view* a, int32_t nblk,
                         const int32_t* blk, double* packed_dev);
/* out_dev[t] = x(phi(lin_idx[t])) = <x, e_{lin_idx[t]}>;
 * lin_idx: HOST, 1-based psi order.  TT_EINDEX if out of range. */
TT_API tt_status tt_element(tt_ctx ctx, const tt_view* x, int32_t nidx, const int64_t* lin_idx, double* out_dev);
/* ||x|| via the right-to-left QR sweep (||C_1||_F), synchronises. */
TT_API tt_status tt_norm(tt_ctx ctx, const tt_view* x, double* out_host);

/* ---------------------------------------------------------------- TT-rounding */
/* out = TT-round(sum_{l<K} coeff[l] terms[l], opts) (Oseledets'
 * right-to-left Householder QR sweep then left-to-right truncated SVD).
 * The TT-sum is never materialised: block-diagonal cores are read in-kernel.
 * coeff: HOST.  info may be NULL.  Output: cores 1..d-1 left-orthonormal, core d carries
 * the norm.  ||x|| = 0 gives a rank-1 zero tensor; d = 1 returns the summed core. */
TT_API tt_status tt_round(tt_ctx ctx, int32_t K, const double* coeff, const tt_view* terms,
                   const tt_round_opts* opts, tt_tensor* out, tt_round_info* info);
/* B independent roundings (C4): item b rounds sum_{l<K[b]} coeff[b][l] terms[b][l].
 * K, coeff, terms: HOST arrays of length B.  out: HOST array of B handles.
 * ranks_out: HOST B*(d+1) or NULL. */
TT_API tt_status tt_round_batch(tt_ctx ctx, int32_t B, const int32_t* K, const double* const* coeff,
                         const tt_view* const* terms, const tt_round_opts* opts,
                         tt_tensor* out, int64_t* ranks_out);

/* B independent roundings of equally shaped TT-sums (BASELINE.json configs[3], "C4"), all
 * in one call of the batched engine (one CTA per item; csrc/batch_round.cu).  Item b rounds
 * x_b = sum_{l<K} coeff[b*K + l] y_{b,l} (PAPER.md:64 TT-sum, rounding contract as tt_round).
 *   n[d], r[K*(d+1)]        HOST: mode sizes; ranks of term l at r[l*(d+1) + k] (same for every b).
 *   core[K*d]               HOST array of DEVICE base pointers: core k of term l of item b is
 *                           core[l*d + k] + b * item_stride[l*d + k] (doubles), C order as tt_view.
 *   coeff[B*K]              HOST.
 *   norms[B*K]              HOST ||y_{b,l}|| for the noise floor s(x), or NULL / NaN entries
 *                           (then computed on the device).
 * Supported: d >= 2, every formal rank sum_l r_k^(l) <= 64, K <= 16 (TT_ENOTSUP otherwise:
 * use tt_round_batch).  The right-to-left QR keeps structural ranks (opts->rank_revealing and
 * qrcp_theta are ignored); truncation as tt_round.  out: a batch handle owning every result
 * (free with tt_batch_free); synchronises the stream once per wave of items. */
TT_API tt_status tt_round_batch_strided(tt_ctx ctx, int32_t B, int32_t K, int32_t d, const int64_t* n,
                                        const int64_t* r, const double* const* core, const int64_t* item_stride,
                                        const double* coeff, const double* norms, const tt_round_opts* opts,
                                        tt_batch* out);
/* Number of items and order of a batch result. */
TT_API tt_status tt_batch_shape(tt_batch bt, int32_t* B, int32_t* d);
/* ranks[b*(d+1) + k] (HOST, B*(d+1)) and norms[b] = ||x_b|| (HOST, B, may be NULL). */
TT_API tt_status tt_batch_ranks(tt_batch bt, int64_t* ranks, double* norms);
/* View of item b (0-based); pointers valid until tt_batch_free.  TT_EINDEX if out of range. */
TT_API tt_status tt_batch_view(tt_batch bt, int32_t b, tt_view* out);
/* Copy every result core to host (HOST, capacity doubles): items in order, each item's cores
 * in order, each core (r_{k-1}, n_k, r_k) C order; *count = doubles in the batch (also set
 * when capacity is too small: TT_EINVAL).  Synchronises. */
TT_API tt_status tt_batch_download(tt_ctx ctx, tt_batch bt, double* host, int64_t capacity, int64_t* count);
/* Result arena w (0-based) of the batch: *ptr = DEVICE pointer, *count = doubles; the arenas in
 * order hold the items in order, each item's cores in order (C order).  TT_EINDEX past the
 * last arena. */
TT_API tt_status tt_batch_arena(tt_batch bt, int32_t w, const double** ptr, int64_t* count);
TT_API tt_status tt_batch_free(tt_ctx ctx, tt_batch bt);

/* B independent roundings from HOST inputs to HOST results in one call (the end-to-end path of
 * tt_round_batch_strided; BASELINE.json configs[3]).  Arguments as tt_round_batch_strided, except:
 *   host_core[K*d]  HOST base pointers: core k of term l of item b starts at
 *                   host_core[l*d + k] + b * item_stride[l*d + k] (doubles), each core C order.
 *                   Page-locked memory (cudaHostAlloc / cudaHostRegister) lets the copies run
 *                   asynchronously; pageable memory works but serialises them.
 *   slices          the batch is processed in about `slices` contiguous slices (whole waves of the
 *                   engine): the host->device copy of slice c+1 and the device->host copy of slice
 *                   c-1 overlap the rounding of slice c (two copy streams owned by the context).
 *   out_host        HOST, out_capacity doubles: every result core, items in order, each item's
 *                   cores in order, each core (rho_{k-1}, n_k, rho_k) C order.
 *   out_count       doubles of the results (set also when they do not fit: then TT_EINVAL, and
 *                   out_host holds only a prefix -- call again with a larger buffer).
 *   ranks_out       HOST B*(d+1) or NULL; norms_out HOST B (||x_b||) or NULL.
 * The call is one unit in ctx-stream order (it waits for earlier work on that stream, and later
 * work waits for its copies); it returns when every result is in out_host. */
TT_API tt_status tt_round_batch_host(tt_ctx ctx, int32_t B, int32_t K, int32_t d, const int64_t* n,
                                     const int64_t* r, const double* const* host_core,
                                     const int64_t* item_stride, const double* coeff, const double* norms,
                                     const tt_round_opts* opts, int32_t slices, double* out_host,
                                     int64_t out_capacity, int64_t* out_count, int64_t* ranks_out,
                                     double* norms_out);

/* ---------------------------------------------------------------- multi-GPU */
/* A context may hold a communicator over N processes (one GPU each; N = 1 takes the same code path).
 * Then, on every rank with identical arguments:
 *   tt_gram         pair blocks split by LPT, one all-gather (see tt_gram);
 *   tt_orth         every batch of driver TT-dots (projection coefficients <p, q_j>, Q/U Gram rows,
 *                   norms) is split into contiguous slices, one all-gather per batch; the
 *                   independent phase-2 roundings of TT-Gram (q_i = round(sum_k R^{-1}(k,i) a_k),
 *                   PAPER.md:250-258) and TT-Householder (q_i = round(e_i - sum_j beta_ij u_j),
 *                   PAPER.md:414-420) are assigned to ranks by LPT on their modelled flops; each
 *                   owner rounds its q_i, the output ranks and norms are all-gathered and q_i is
 *                   broadcast from its owner, so every rank returns every q_i.  The sequential
 *                   rounding chains (CGS/MGS steps, Householder phase 1) are replicated: a single
 *                   rounding sweep never shards (north star).
 * Batches of independent roundings need no communicator: each rank rounds its tt_plan_slice. */
#define TT_COMM_ID_BYTES 128
/* Caller-supplied collectives (e.g. a host transport).  Both are called after the ctx stream has
 * been synchronised and must complete before returning; return 0 on success.
 *   allgather: every rank contributes `bytes` at send (DEVICE); recv (DEVICE, nranks*bytes)
 *              receives them in rank order.
 *   broadcast: rank root's buf (DEVICE, bytes) is copied into every rank's buf. */
typedef struct {
  int (*allgather)(void* user, const void* send, void* recv, size_t bytes, void* stream);
  int (*broadcast)(void* user, void* buf, size_t bytes, int32_t root, void* stream);
  void* user;
} tt_comm_ops;
/* A fresh NCCL unique id (TT_COMM_ID_BYTES bytes, HOST) for tt_ctx_comm_nccl; call on one rank
 * and pass the bytes to the others.  Loads libnccl.so.2 (TT_ECOMM when it cannot). */
TT_API tt_status tt_comm_nccl_id(uint8_t* id);
/* Attach an NCCL communicator of nranks (collective: every rank calls it with the same id). */
TT_API tt_status tt_ctx_comm_nccl(tt_ctx ctx, int32_t nranks, int32_t rank, const uint8_t* id);
/* Attach caller-supplied collectives (ops copied; ops->user must outlive the attachment). */
TT_API tt_status tt_ctx_comm_ops(tt_ctx ctx, int32_t nranks, int32_t rank, const tt_comm_ops* ops);
TT_API tt_status tt_ctx_comm_detach(tt_ctx ctx);
/* nranks / rank of the attached communicator (1 / 0 without one). */
TT_API tt_status tt_ctx_comm_info(tt_ctx ctx, int32_t* nranks, int32_t* rank);
/* Shard plans (HOST only; no context, no device).
 *   tt_plan_slice       contiguous balanced slice [start, end) of P independent items for rank.
 *   tt_plan_lpt         owner[i] of P items with costs cost[i]: decreasing cost (ties: lower i),
 *                       each to the least-loaded rank (ties: lower rank); deterministic.
 *   tt_plan_gram_blocks the b x b pair blocks (i0, j0, bi, bj) covering i >= j of an m x m Gram
 *                       matrix (diagonal blocks full), into blk[4*nblk], and their LPT owners by
 *                       pair count; *nblk always set, TT_EINVAL when cap < *nblk (cap 0: query). */
TT_API tt_status tt_plan_slice(int64_t P, int32_t nranks, int32_t rank, int64_t* start, int64_t* end);
TT_API tt_status tt_plan_lpt(int32_t P, const double* cost, int32_t nranks, int32_t* owner);
TT_API tt_status tt_plan_gram_blocks(int32_t m, int32_t b, int32_t nranks, int32_t cap, int32_t* blk,
                                     int32_t* owner, int32_t* nblk);

/* ---------------------------------------------------------------- step-level replay */
/* Observer of the drivers' rounding calls (SURVEY.md §8(b) "step-level replay"): when set,
 * tt_orth calls fn before each of its TT-roundings with the call's index in Table 1 order
 * (0-based), the TT-sum's K terms (views of DEVICE cores, norm = the ||y_l||
 * the rounding uses for s(x)), its HOST coefficients and the rounding options.  The ctx stream
 * is synchronised first, so the cores can be read on any stream; everything passed is borrowed
 * for the duration of the callback only.  Used to replay a driver step through another
 * implementation (teacher-forced parity).  fn = NULL removes the observer. */
typedef void (*tt_round_hook)(void* user, int64_t call, int32_t K, const double* coeff, const tt_view* terms,
                              const tt_round_opts* opts);
TT_API tt_status tt_ctx_round_hook(tt_ctx ctx, tt_round_hook fn, void* user);

/* ---------------------------------------------------------------- drivers */
/* Q, R = TT-<kind>(A, delta) (Algs. 1-5, 8).  q_out: HOST array of m
 * handles (library-owned results).  R_host: m*m row-major upper triangular, R(j,i) =
 * coefficient of q_j in a_i.  report may be NULL.  Returns TT_ELINDEP /
 * TT_ESINGULAR_GRAM with report->fail_index on breakdown. */
TT_API tt_status tt_orth(tt_ctx ctx, tt_orth_kind kind, int32_t m, const tt_view* a,
                  const tt_orth_opts* opts, tt_tensor* q_out, double* R_host,
                  tt_orth_report* report);

#ifdef __cplusplus
}
#endif
#endif /* TT_B200_H */
