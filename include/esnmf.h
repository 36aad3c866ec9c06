/*
 * esnmf.h -- C ABI of libesnmf.so: the B200 (sm_100a) hot path of
 * enforced-sparse ALS NMF (Gavin, Gadepally, Kepner, arXiv 1510.05237).
 *
 * Citations: P:n = line n of the paper text; S:n = line n of the
 * CPU-program spec (SPEC.md, interfaces only); readings C1..C16 are listed in
 * DESIGN.md section 2.
 *
 * Problem: A in R^{n x m}, A >= 0 sparse (n terms x m documents,
 * P:23); find U in R^{n x k}, V in R^{m x k}, U, V >= 0, A ~ U V^T.
 * Method (Alg. 2, per-column enforcement P:304): starting
 * from U = U_0, each iteration does
 *   V side: V = A^T U (U^T U + eps I)^{-1}, negatives -> 0,
 *                       keep the t largest entries of every column of V;
 *   U side: U = A V (V^T V + eps I)^{-1},   negatives -> 0,
 *                       keep the t largest entries of every column of U;
 * with eps = ridge_scale * (tr(G)/k + 1) (reading C6), ties at the t-th value
 * broken toward the lower row index so exactly min(t, #positive) entries
 * survive (reading C4), and only strictly positive entries ever kept (C5).
 * Metrics: R = ||U_i - U_{i-1}||_F / ||U_i||_F, computed by direct
 * difference; E = ||A - U V^T||_F / ||A||_F via the trace identity
 * ||A||^2 - 2 tr(U^T (A V)) + tr((U^T U)(V^T V)).
 *
 * Conventions for every entry point:
 *  - Returns ESNMF_OK (0) or an error code; esnmf_last_error() gives a
 *    message for the calling thread.  No entry point aborts the process.
 *  - Matrices are 0-based.  CSR: row_ptr[rows+1] (int64, row_ptr[0] = 0,
 *    non-decreasing, row_ptr[rows] = nnz), col_idx[nnz] (int32, strictly
 *    increasing within a row), val[nnz] (fp32, finite, >= 0).
 *  - Factor output is canonical column-major COO: ascending column, then
 *    ascending row; values are the device fp32 values exactly.
 *  - A handle is not thread-safe; distinct handles are independent.  All
 *    device work is enqueued on the handle's stream; esnmf_iterate and
 *    esnmf_half_step are asynchronous, every getter synchronises the stream.
 *  - Asynchronous CUDA faults surface as ESNMF_ECUDA at the next
 *    synchronising call.
 */
#ifndef ESNMF_H
#define ESNMF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct esnmf esnmf_t; /* opaque; owns all of its device memory */

typedef enum {
  ESNMF_OK = 0,
  ESNMF_EINVAL = 1,      /* bad argument or malformed CSR (message names it) */
  ESNMF_ENOMEM = 2,      /* device or host allocation failed */
  ESNMF_ECUDA = 3,       /* CUDA runtime error (including asynchronous faults) */
  ESNMF_ECOMM = 4,       /* a collective callback returned non-zero */
  ESNMF_ESINGULAR = 5,   /* G + eps I not positive definite / non-finite pivot */
  ESNMF_EDEGENERATE = 6, /* ||U_i||_F == 0: residual undefined */
  ESNMF_ESTATE = 7,      /* call-order violation (e.g. residual before iterate) */
  ESNMF_ETRUNC = 8       /* caller buffer too small; *nnz holds the size needed */
} esnmf_status;

#define ESNMF_T_UNLIMITED (-1) /* Alg. 1, projected ALS: no truncation */
#define ESNMF_T_SAME (-2)      /* esnmf_options.t_u / t_v: use create's t */
#define ESNMF_ENFORCE_COLUMN 0 /* keep the t largest of every topic column (BJ:5) */
#define ESNMF_ENFORCE_MATRIX 1 /* keep the t largest of the whole factor: Alg. 2 as printed */
#define ESNMF_SIDE_V 0         /* half-step 1: V <- A^T U */
#define ESNMF_SIDE_U 1         /* half-step 2: U <- A V */
#define ESNMF_MAX_K 256

/*
 * Collectives for world > 1 (one process per GPU, rows of A and A^T sharded
 * across ranks).  Both callbacks are stream-ordered on `stream` and take
 * DEVICE buffers; they return 0 on success.  The Python binding implements
 * them with torch.distributed (NCCL on GPUs).
 *   allgather: every rank contributes `bytes_per_rank` bytes from `send`;
 *              `recv` receives world * bytes_per_rank bytes in rank order.
 *   allreduce_sum_f64: in-place elementwise sum of `count` doubles.
 */
typedef struct {
  void* ctx;
  int (*allgather)(void* ctx, const void* send, void* recv, int64_t bytes_per_rank, void* stream);
  int (*allreduce_sum_f64)(void* ctx, double* buf, int64_t count, void* stream);
} esnmf_comm;

/*
 * Built-in collectives: an NCCL communicator owned by the library (NVLink /
 * NVSwitch between the GPUs of one box).  The library calls
 * ncclAllGather / ncclAllReduce on its own stream -- no host callback -- so a
 * sharded iteration is captured into a CUDA graph like a single-GPU one.
 * libnccl.so.2 is loaded at run time (dlopen; the one torch loads when present).
 *   esnmf_nccl_unique_id: rank 0 draws the id (NCCL_UNIQUE_ID_BYTES = 128 bytes
 *     into `id`); the caller broadcasts it to every rank (any transport).
 *   esnmf_nccl_comm_create: every rank, collectively, with the same id; `device`
 *     = this rank's CUDA ordinal.  *out is an esnmf_comm for esnmf_options.comm,
 *     owned by the library until esnmf_nccl_comm_destroy (after the handles that
 *     use it are destroyed).
 * Errors: ECOMM (NCCL missing or failed; esnmf_last_error names the cause),
 * EINVAL (NULL, world < 1, rank out of range). */
#define ESNMF_NCCL_ID_BYTES 128
esnmf_status esnmf_nccl_unique_id(void* id);
esnmf_status esnmf_nccl_comm_create(int32_t world, int32_t rank, const void* id, int32_t device, esnmf_comm** out);
void esnmf_nccl_comm_destroy(esnmf_comm* comm);

typedef struct {
  uint64_t seed;        /* U_0 seed (reading C10), default 0 (BJ:7) */
  double ridge_scale;   /* rho of eps = rho (tr G / k + 1), default 1e-10 (C6) */
  int32_t device;       /* CUDA ordinal; -1 = current device (default) */
  void* stream;         /* cudaStream_t to enqueue on; NULL = library-owned stream */
  int32_t world, rank;  /* 1, 0 = single GPU (default) */
  const esnmf_comm* comm; /* required when world > 1; must outlive the handle */
  int32_t inputs_on_device; /* 1: every input pointer below and in create is a
                               device pointer on `device`; 0 (default): host */
  /* optional CSR(A^T) (m rows x n columns); NULL = built on the device */
  const int64_t* at_row_ptr;
  const int32_t* at_col_idx;
  const float* at_val;
  /* optional dense U_0 (n x k row-major fp32); NULL = reading C10 formula:
     U0[i,c] = ((splitmix64(seed ^ 0x55305F494E495430 ^ (i*k + c)) >> 41) + 0.5) * 2^-23 */
  const float* U0;
  /* V-side tensor-core head: the product A^T Z is split
     by term; the `head_terms` most frequent terms (a multiple of 64, <= 1024)
     run as a dense fp16-split GEMM on the tensor cores, the rest as a sparse
     row gather.  -1 (default) = automatic (terms in >= 4 % of the documents),
     0 = off.  The result is the same product to fp32 accuracy either way. */
  int32_t head_terms;
  /* Separate budgets of Alg. 2 ("t_u, t_v"): ESNMF_T_SAME (default) = create's
     t, ESNMF_T_UNLIMITED = no truncation of that factor (U-only / V-only
     enforcement), >= 0 = that budget. */
  int64_t t_u, t_v;
  /* ESNMF_ENFORCE_COLUMN (default) or ESNMF_ENFORCE_MATRIX (whole-factor top-t,
     ties -> lower column, then lower row; single GPU only: EINVAL with world > 1). */
  int32_t enforce;
  /* Sparse initial guess (P:289-298 vary the nnz of U_0; reading C18): 0 (default) =
     dense U_0; > 0 = keep U0[i,c] only where splitmix64(seed ^ 0x55305F4D41534B30 ^
     (i*k + c)) >> 11 < init_nnz * 2^53 / n (expected init_nnz entries per column). */
  int64_t init_nnz;
  /* Sequential ALS (Alg. 3; NEXT-2): 0 (default) = off; k2 > 0 (dividing k)
     = find the k topics in k / k2 blocks of k2.  Block b (columns [b k2, (b+1) k2))
     starts from U_2 = U_0 (the reading C10 formula with k2 columns, index i*k2 + c;
     masked per init_nnz) and runs `seq_iters` >= 1 iterations of Eq. (7) / (8)
      with the converged columns held fixed; then the next block starts.
     esnmf_iterate counts iterations over the whole schedule (k / k2 * seq_iters in
     all; ESTATE after that).  Records cover the whole factors U = [U_1 U_2 0],
     V = [V_1 V_2 0]; esnmf_get_U / _V return them (k columns).  The least-squares
     buffer (esnmf_get_ls), the Gram, esnmf_set_factor and esnmf_truncate act on the
     current block (k2 columns, info.ls_cols).  t_u / t_v bound each column of the
     block (ESNMF_ENFORCE_COLUMN) or the whole block (ESNMF_ENFORCE_MATRIX, Alg. 3
     steps 2 and 4 as printed).  Single GPU; U0 must be NULL.  EINVAL otherwise. */
  int32_t seq_k2;
  int32_t seq_iters;
  /* Row normalisation ("divide each row of the data matrix by the number of
     nonzero entries in that row"; NEXT-4): 1 = every a_ij is replaced by a_ij / nnz(row i)
     on the device at create (fp32, correctly rounded; A^T alike), before ||A|| and
     everything else; 0 (default) = A as given. */
  int32_t row_normalize;
  /* The V side's pre-clamp least-squares buffer (esnmf_get_ls).  0 (default): when
     the V side's selection runs from the candidates the head kernel's epilogue
     collects (per-column top-t with a predicted threshold, one GPU), esnmf_iterate
     writes the LS buffer only if some column's prediction failed (its exact path
     reads it): 400 MB of stores per iteration at Large saved; esnmf_get_ls(V) then
     fails with ESTATE.  1: every V side writes it.  esnmf_half_step always does. */
  int32_t keep_ls;
} esnmf_options;

typedef struct {
  int32_t it;            /* 1-based iteration index */
  double R;              /* relative residual of U after this iteration; -1 if undefined */
  double E;              /* relative error after this iteration */
  int64_t nnz_u, nnz_v;  /* stored entries of U and V ("NNZ") */
  int32_t dead_u, dead_v;/* all-zero columns (dead topics, reading C6) */
  int64_t active_u, active_v; /* rows holding at least one entry */
  int64_t peak_u, peak_v;     /* positive entries of the clamped least-squares factor before
                                 truncation: the peak stored nnz of that half-step (P:289-298,
                                 S:226-229 peak_nnz); this rank's share when world > 1 */
} esnmf_record;

/* Fill *opt with the defaults above.  Always ESNMF_OK (EINVAL if opt NULL). */
esnmf_status esnmf_options_init(esnmf_options* opt);

/*
 * Create a solver for A (n x m, CSR by term rows) of rank k keeping t entries
 * per topic column (t >= 0, or ESNMF_T_UNLIMITED).  1 <= k <= ESNMF_MAX_K,
 * 1 <= n, m < 2^31, nnz >= 1.  Inputs are validated and copied (host->device
 * when inputs_on_device == 0); the caller may free them on return.  Empty
 * rows / columns are accepted.  Sets U = U_0 (reading C11).
 * Errors: EINVAL (shape, non-monotone row_ptr, column out of range or not
 * strictly increasing, negative or non-finite value, k or t out of range),
 * ENOMEM, ECUDA.  On error *out is set to NULL.
 */
esnmf_status esnmf_create(esnmf_t** out, int64_t n, int64_t m, int32_t k, int64_t t,
                          const int64_t* row_ptr, const int32_t* col_idx, const float* val,
                          const esnmf_options* opt);

/* Run `iters` >= 0 iterations {V side; U side} of Alg. 2, and
 * record R and E for each.  Asynchronous on the handle's stream. */
esnmf_status esnmf_iterate(esnmf_t* h, int32_t iters);

/* One half-step only (side = ESNMF_SIDE_V or ESNMF_SIDE_U); test hook for
 * per-half-step parity.  The V side reads the current U; the U side reads the
 * current V and replaces U (the previous U is kept for R).  No record. */
esnmf_status esnmf_half_step(esnmf_t* h, int32_t side);

/* R of the last completed iteration (synchronises).  ESTATE before the first
 * iteration; EDEGENERATE if ||U_i|| == 0. */
esnmf_status esnmf_residual(esnmf_t* h, double* R);

/* E of the last completed iteration (synchronises).  ESTATE before the first. */
esnmf_status esnmf_error(esnmf_t* h, double* E);

/* Copy out up to `cap` per-iteration records, oldest first; *count = number
 * of records held.  ETRUNC if cap < *count (the first cap are written). */
esnmf_status esnmf_records(esnmf_t* h, int64_t cap, int64_t* count, esnmf_record* out);

/* Current U (n x k) / V (m x k) as canonical column-major COO (synchronises).
 * Two-call pattern: if cap < nnz (or any array is NULL) returns ETRUNC with
 * *nnz = entries needed; otherwise fills row/col/val and *nnz. */
esnmf_status esnmf_get_U(esnmf_t* h, int64_t cap, int64_t* nnz, int32_t* row, int32_t* col, float* val);
esnmf_status esnmf_get_V(esnmf_t* h, int64_t cap, int64_t* nnz, int32_t* row, int32_t* col, float* val);

/* Replace U (side U) or V (side V) by a caller COO (host arrays, canonical
 * order, values > 0, row < n or m, col < k).  Test hook: start a half-step
 * from a given state.  Invalidates the stored records' "last" R/E. */
esnmf_status esnmf_set_factor(esnmf_t* h, int32_t side, int64_t nnz, const int32_t* row,
                              const int32_t* col, const float* val);

/* Pre-clamp least-squares rows of the last half-step of `side` for this
 * rank's row shard, written row-major (rows_local x k) into `out` (host).
 * *rows receives rows_local; *row0 the global index of the first row. */
esnmf_status esnmf_get_ls(esnmf_t* h, int32_t side, int64_t* row0, int64_t* rows, float* out);

/* Gram matrix (unregularised, k x k row-major fp64) used by the last
 * half-step of `side` (side V: U^T U; side U: V^T V), and its eps. */
esnmf_status esnmf_get_gram(esnmf_t* h, int32_t side, double* gram, double* eps);

typedef struct {
  int64_t n, m, nnz;
  int32_t k;
  int64_t t;
  int32_t world, rank;
  int64_t v_row0, v_rows;   /* this rank's document rows (V side) */
  int64_t u_row0, u_rows;   /* this rank's term rows (U side) */
  int64_t iterations;       /* completed iterations */
  int64_t device_bytes;     /* device memory owned by the handle */
  double normA2;            /* ||A||_F^2 */
  int64_t launches;         /* CUDA kernels enqueued by this handle so far */
  int32_t head_terms;       /* V-side tensor-core head size (0 = none) */
  int32_t head_dense;       /* of its 64-term chunks, how many are stored as dense tiles */
  int32_t ls_cols;          /* columns of esnmf_get_ls / esnmf_get_gram / esnmf_set_factor:
                               k, or k2 (the current block) in sequential mode */
  int32_t seq_block;        /* sequential mode: index of the current block (0-based) */
} esnmf_info;

esnmf_status esnmf_get_info(esnmf_t* h, esnmf_info* info);

/* Per-half-step cost model of the last V side, from the compact
 * factor and the document frequencies df_i of A (O(k t) work per half-step),
 * plus the U side's product count for the current V.  The V-side tail order
 * is chosen from it on the device each half-step: the paper's order
 * (A^T_tail U) W when v_tail_products * ratio <= v_tail_gather_fma (ratio =
 * the measured cost of one fixed-point shared-memory product over one gathered
 * FMA, 8), else the reassociated A^T_tail (U W) gather -- and the gather also
 * whenever W is too ill-conditioned for fp16 hi/lo operands (kappa_inf(G + eps I)
 * > 1e4, or a column of W whose absolute sum exceeds 8 times its diagonal).
 * Synchronises.  ESTATE before the first V side; EINVAL for NULL. */
typedef struct {
  double v_tail_products;    /* paper order: sum over active tail terms i of df_i * nnz(U row i) */
  double v_tail_gather_fma;  /* reassociated: sum over active tail terms i of df_i * k */
  double v_tail_active;      /* active tail entries of A^T (df summed over active tail terms) */
  double v_head_products;    /* head terms: sum over active head terms of df_i * nnz(U row i) */
  double v_head_mma_flops;   /* tensor-core flops the head issues (dense 128 x 64 tiles, 3 fp16 passes) */
  double v_yw_mma_flops;     /* tensor-core flops of the (Y_tail W) chunks (paper order only) */
  double u_products;         /* U side, paper order: sum over stored entries (d, c) of V of nnz(A^T row d) */
  int32_t head_terms;        /* h */
  int32_t v_tail_gather;     /* 1: the last V side ran the Z-row gather */
  int32_t v_gather_by_cost;  /* ... chosen by the cost model (else by the conditioning) */
  int32_t paper_order_tail;  /* 1: this handle has the paper-order tail (else always the gather) */
} esnmf_cost;

esnmf_status esnmf_cost_model(esnmf_t* h, esnmf_cost* out);

/* Per-phase device timing with CUDA events on the handle's stream (the same
 * stream the kernels run on).  esnmf_profile(h, 1) clears the accumulators and
 * starts recording an event pair around every phase of every later half-step;
 * esnmf_profile(h, 0) stops.  esnmf_phase_times synchronises and returns one
 * entry per phase: "<side>.<phase>" with side V or U and phase one of gram,
 * solve, form_z, spmm, select, rowview; plus "iter.metrics" (R, E, next Gram).
 * ETRUNC if cap < *count. */
typedef struct {
  char name[32];
  int64_t calls;  /* launches of the phase since profiling started */
  double ms;      /* summed device time, milliseconds */
} esnmf_phase;

esnmf_status esnmf_profile(esnmf_t* h, int32_t enable);
esnmf_status esnmf_phase_times(esnmf_t* h, int64_t cap, int64_t* count, esnmf_phase* out);

/* Free all device memory of the handle (NULL is a no-op). */
void esnmf_destroy(esnmf_t* h);

const char* esnmf_strerror(esnmf_status s);
const char* esnmf_last_error(void);

/* Clustering accuracy of the document topics, Eq. (3)-(4) (NEXT-4).
 * labels: HOST array of m journal ids in [0, n_journals); acc: HOST array of k
 * doubles.  For every topic column c of the current V (all k columns, also in
 * sequential mode) the documents "belonging" to it are its stored entries
 * (n_D of them); acc[c] = (same-journal pairs - alpha) / (beta - alpha) with
 * alpha = floor(n_D/n_J) (n_J (floor(n_D/n_J) - 1)/2 + n_D mod n_J) and
 * beta = n_D (n_D - 1)/2; 1 when n_D <= 1 or beta == alpha (n_J = 1).  Counts are
 * exact (integer-valued fp64 atomics).  Synchronous.  EINVAL (bad labels),
 * ESTATE (V not set). */
esnmf_status esnmf_topic_accuracy(esnmf_t* h, const int32_t* labels, int32_t n_journals, double* acc);

/* Enforce-after: clamp and truncate the CURRENT
 * factor of `side` once, in place -- the t largest entries per column
 * (enforce = ESNMF_ENFORCE_COLUMN) or of the whole factor (ESNMF_ENFORCE_MATRIX),
 * same tie rules as the iteration (C4, C17).  Typical use: create with t =
 * ESNMF_T_UNLIMITED (Alg. 1), iterate, then truncate U and V.  Records are not
 * changed.  Errors: EINVAL (side, t < 0), ESTATE (factor not set), ECUDA.
 * Single GPU only (EINVAL with world > 1). */
esnmf_status esnmf_truncate(esnmf_t* h, int32_t side, int64_t t, int32_t enforce);

/* Host-only helper (no GPU needed): nnz-balanced contiguous partition of
 * `rows` rows into `world` ranges; bounds[world+1].  Used for the row shards
 * of A; A^T rows are split in equal counts. */
esnmf_status esnmf_partition_rows(int64_t rows, const int64_t* row_ptr, int32_t world, int64_t* bounds);

/* Library version string (build id). */
const char* esnmf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ESNMF_H */
