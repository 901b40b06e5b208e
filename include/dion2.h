/*
 * dion2.h -- C ABI of the B200-native Dion2 optimizer step (arXiv 2512.16928).
 *
 * The library implements Algorithm 1 of the paper ("alpha-Dion2(G, M)",
 * PAPER.md P:177-191) for a batch of weight matrices on one GPU:
 *
 *   l.2  M <- M + G
 *   l.3  K <- Select_alpha(M)  (top l1 rows or columns)
 *   l.4  O <- NewtonSchulz(M[K, :])
 *   l.5  M[K, :] <- mu * M[K, :]   Eq. (error-feedback)
 *   l.6  W[K, :] <- W[K, :] - eta*sqrt(fan-out/fan-in)*O  Eq. (orth-update)
 *
 * "Column-selection is analogous"; auto mode selects along the
 * shorter dimension.  The readings taken where the paper is silent
 * (NS coefficients/steps/normalisation, k rounding, tie-break, orientation)
 * are listed in DESIGN.md "Readings".
 *
 * Conventions
 *  - Every pointer is a DEVICE pointer unless marked HOST.
 *  - Matrices are row-major: element (i, j) of W is W[i*ld + j]; rows =
 *    fan-out, cols = fan-in (y = W x).
 *  - The caller owns every buffer (W, M, G, workspace, optional outputs); size
 *    the workspace with dion2_workspace_size() and pass it to every step.  The
 *    library's device allocations are a small plan-owned table (matrix
 *    descriptors and work lists, a few hundred bytes per matrix), made once per (shapes,
 *    config, workspace) plan on its first step, reused by every later step and freed by
 *    dion2_release_workspace(); and, for the distributed entry points with
 *    DION2_FLAG_DIST_DIRECT, the plan's two NCCL symmetric-memory windows.
 *  - All work is enqueued asynchronously on `stream` (a cudaStream_t passed
 *    as void*; NULL = legacy default stream).  No host synchronisation
 *    happens inside a step.  Calls that touch the same matrices must not
 *    overlap.  The workspace may not be shared by concurrent calls.
 *  - CUDA graphs: after a plan's first step, a step on the SAME matrix
 *    pointers enqueues only kernels and memsets (no allocation, no host copy)
 *    and may be captured.  The plan's descriptor table holds the pointers of
 *    its latest eager step, so graphs of different pointer sets need distinct
 *    plans: pass distinct workspace base pointers (the plan cache is keyed by
 *    it; the Python Dion2(cuda_graph=True) offsets the base by 4 KiB per set).
 *    The tensor-core NS kernels use programmatic dependent launch.
 *  - Return value: a dion2_status code.  Codes 1-4 are detected on the host
 *    before anything is enqueued.  Non-finite scores are detected on the
 *    device: that matrix's W and M[K] writes are skipped and
 *    dion2_get_status() reports it (ENONFINITE).
 */
#ifndef DION2_H_
#define DION2_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DION2_ABI_VERSION 7
#define DION2_MAX_NS_STEPS 16
/* dion2_config.reserved0 flag: the sparse update reads eta on the device from the fp32 word at
   byte offset 8 of the workspace's 4096-byte-aligned base (the first multiple of 4096 at or
   after `workspace`; the caller writes it, stream-ordered, before the step)
   instead of cfg.lr, so a CUDA graph of the step follows a learning-rate schedule without being
   re-captured.  cfg.lr must still be a valid eta (it is validated, then ignored by the kernels). */
#define DION2_FLAG_LR_DEVICE 1
/* dion2_config.reserved0 flag (ABI v7), read by dion2_step_batched_dist / _loopback only:
   the exchange pieces travel by direct peer stores and loads instead of NCCL send / recv
   (the fused gather + send).  K3 stores each piece of X straight into its
   owner's receive buffer and K7 loads its piece of O straight from the owner's outgoing buffer;
   with NCCL these are symmetric-memory windows (ncclMemAlloc + ncclCommWindowRegister, NCCL
   >= 2.28 device API) separated by LSA barriers, allocated collectively on the first step of a
   plan and kept for the process lifetime; in loopback they are the other ranks' workspaces.
   Requires every rank in one load/store (NVLink) domain, else DION2_EUNSUPPORTED; forces one
   owner chunk.  Results are bitwise those of the NCCL exchange (same kernels, same bytes).
   dion2_step_batched_dpsync (P <= 8) reads it too: each replica packs M[K] into its input
   window, and after an LSA barrier sums its 1/P slice over all replicas' windows in rank order
   and stores the sum into every replica's output window (a reduce-scatter + all-gather by
   peer loads / stores, 2 (P-1)/P of the buffer per rank like a ring all-reduce), a second
   barrier, then unpacks: the same rank-order sums as the loopback emulation, bit-identical on
   every replica by construction.  Where the windows are unavailable both entry points fall
   back to NCCL (dion2_dist_exchange_mode reports which ran). */
#define DION2_FLAG_DIST_DIRECT 2

typedef enum {
  DION2_OK = 0,
  DION2_EINVAL_CONFIG = 1, /* alpha not in (0,1], mu not in [0,1), lr < 0, ns_steps not in [1,16], eps <= 0, bad enum */
  DION2_EINVAL_SHAPE = 2,  /* rows/cols < 1, ld < cols, NULL W/M/G, d > DION2_MAX_SELECT_DIM */
  DION2_EWORKSPACE = 3,    /* workspace NULL or smaller than dion2_workspace_size() */
  DION2_EUNSUPPORTED = 4,  /* a configuration this build does not implement */
  DION2_ECUDA = 5,         /* a CUDA runtime / launch error */
  DION2_ENCCL = 6,         /* an NCCL call failed (distributed / DP-sync entry points) */
  DION2_ENONFINITE = 7     /* (device-side) a matrix's scores were NaN/Inf */
} dion2_status;

/* Longest selection axis supported by the single-CTA top-k kernel. */
#define DION2_MAX_SELECT_DIM 49152

typedef enum { DION2_AXIS_ROWS = 0, DION2_AXIS_COLS = 1, DION2_AXIS_AUTO = 2 } dion2_axis;
typedef enum { DION2_SELECT_L1 = 0, DION2_SELECT_RANDOM = 1 } dion2_select;
/* Newton-Schulz arithmetic.  DION2_NS_BF16 (= DION2_NS_TC16, the name kept from ABI v1-v5) is the
   tcgen05 tensor-core path: since ABI v6 its operands are fp16 (10-bit mantissa) with fp32
   accumulation, X stored as fp16(2^e X) with a power-of-two prescale chosen from the matrix's
   largest l1 score so no entry can overflow (reading R24); FP32 is the SIMT fp32 validation path. */
typedef enum { DION2_NS_BF16 = 0, DION2_NS_FP32 = 1 } dion2_precision;
#define DION2_NS_TC16 DION2_NS_BF16
typedef enum { DION2_DT_F32 = 0, DION2_DT_BF16 = 1 } dion2_dtype;
/* How the tensor-core Newton-Schulz map is evaluated (readings R23, R24).  Both forms compute
   the same polynomial map X_T = p_T(... p_1(X_0)) of Alg. 1 l.4; they differ only in rounding.
   DIRECT: T iterations on X (p x q): A = X X^T, C = a I + b A + c A^2, X <- C X (fp16).
   GRAM:   the iteration carried out on p x p matrices, in restart segments of consecutive
           iterations whose growth prod |a_t| stays <= 64 ([0,3) + [3,5) for the default quintic):
           per segment A = X_in X_in^T once, then C_t = a I + b A_t + c A_t^2,
           Q_{t+1} = C_t Q_t, A_{t+1} = C_t (C_t A_t) (fp16, fp32 accumulation), and
           X_out = Q X_in once.  Fewer FLOPs when q >= 2p (1.85x at p = 512, q in {2048, 8192}).
   AUTO:   an X of at most 128 rows is evaluated in high precision (Gram space straight from the
           pre-decay momentum, fp64 / fp32 recursion, X_T stored once as fp16; reading R25);
           otherwise GRAM for a shape
           group whose padded X has q_pad >= 2 p_pad or whose every member has q >= 2p, provided
           every member has p >= 64 rows (R25: the fp16 Gram matrix of a short X rounds away too
           much of its small eigenvalues); DIRECT otherwise.  AUTO meets the 2e-2 parity gate on
           Gaussian and on ill-conditioned (spiked / power-law) momenta
           (tests/test_gpu_conditioning.py, tests/test_gpu_fuzz.py); the 16-bit forms forced on
           short X can miss it (up to 3.6% on 2-row X of extreme spikes). */
typedef enum { DION2_NS_FORM_AUTO = 0, DION2_NS_FORM_DIRECT = 1, DION2_NS_FORM_GRAM = 2 } dion2_ns_form;

/* One weight matrix and its optimizer state. */
typedef struct {
  int64_t rows;        /* m = fan-out, >= 1 */
  int64_t cols;        /* n = fan-in,  >= 1 */
  int64_t ld;          /* row stride in elements of W, M and G; >= cols */
  float* W;            /* [rows x ld] fp32, updated in place (selected rows/cols only) */
  float* M;            /* [rows x ld] fp32 momentum, updated in place */
  const void* G;       /* [rows x ld] gradient, dtype cfg.grad_dtype, read only */
  int32_t* sel_out;    /* optional [k] int32: the selected indices, ascending (NULL = not written) */
  float* O_out;        /* optional fp32 copy of O in natural orientation: [k x cols] (rows mode) or
                          [rows x k] (cols mode), dense row-major (NULL = not written) */
  int32_t m_transposed; /* 0: M has W's layout.  1: M is stored TRANSPOSED, [cols x ldm] row-major
                           (element (i, j) of M at M[j*ldm + i]); only for matrices whose resolved
                           selection axis is COLS, where it turns the column gather of M[:, K] into a
                           contiguous row gather (DION2_EUNSUPPORTED otherwise) */
  int32_t storage_transposed; /* 0: W, M, G are stored [rows x ld] (PyTorch (out, in)).  1: they are stored
                           TRANSPOSED, [cols x ld] row-major, ld >= rows (JAX / Flax (in, out) kernels):
                           element (i, j) of the logical m x n matrix at W[j*ld + i].  rows / cols stay
                           the LOGICAL fan-out / fan-in: the axis (with its square tie-break), k and the
                           sqrt(fan-out/fan-in) scale follow them, while every kernel runs on the storage
                           layout (a logical column selection becomes a contiguous row selection).
                           sel_out holds logical indices; O_out is written in the storage orientation.
                           m_transposed then means M in the logical layout ([rows x ldm]) */
  int64_t ldm;          /* row stride of the transposed M (>= the storage rows); ignored when m_transposed = 0 */
} dion2_matrix;

/* Hyper-parameters of Alg. 1.  Fill with dion2_config_init() first. */
typedef struct {
  float alpha;        /* selection fraction in (0, 1]; k = max(1, floor(alpha*d + 1/2)) (reading R7) */
  float mu;           /* momentum decay in [0, 1), default 0.95 (Alg. 1 header) */
  float lr;           /* eta >= 0, default 0.02 */
  int32_t ns_steps;   /* Newton-Schulz iterations T in [1, 16], default 5 (reading R2) */
  float ns_coeffs[DION2_MAX_NS_STEPS][3]; /* (a, b, c) per iteration, default (3.4445, -4.7750, 2.0315) (reading R1) */
  float ns_eps;       /* X0 = X / (||X||_F + eps), default 1e-7 (reading R3) */
  int32_t axis;       /* dion2_axis, default AUTO (shorter dimension) */
  int32_t select;     /* dion2_select, default L1 (largest l1 norm).  RANDOM: the k indices
                         with the smallest keys Philox4x32-10(ctr = (index, step_lo, step_hi, matrix id in
                         the batch), key = (seed_lo, seed_hi)) word 0, lower index on ties (reading R22) */
  int32_t precision;  /* dion2_precision: BF16 (= TC16) = tcgen05 tensor-core NS on fp16 operands (hot path);
                         FP32 = SIMT fp32 NS (validation) */
  int32_t grad_dtype; /* dion2_dtype of G, default F32 */
  int32_t decay_mode; /* 0 = selective decay Eq. (error-feedback) (paper); 1 = full decay M <- mu*M (ablation) */
  int32_t scale_mode; /* 0 = eta*sqrt(rows/cols) of the full W (Alg. 1 l.6); 1 = sqrt of the submatrix dims (SPEC S:360 flag) */
  uint64_t seed;      /* random selection key (unused for L1) */
  uint64_t step;      /* random selection counter: the caller's step index (unused for L1) */
  int32_t ns_form;    /* dion2_ns_form, default AUTO (BF16 precision only; FP32 is always DIRECT) */
  int32_t reserved0;  /* flags: 0, DION2_FLAG_LR_DEVICE, DION2_FLAG_DIST_DIRECT (other bits must be 0) */
  int32_t w_dtype;    /* dion2_dtype of W (ABI v6): F32 (default) or BF16 -- bf16 weights; the update
                         is computed in fp32 and rounded to nearest once (w <- bf16(float(w) - s o)).
                         M stays fp32 (its l1 scores decide the selection) */
} dion2_config;

/* Fill *cfg with the defaults above.  Always returns DION2_OK. */
int dion2_config_init(dion2_config* cfg);

/* Bytes of device workspace a step over mats[0..n) with *cfg needs (HOST
 * mats/cfg; the W/M/G pointers are not read).  Returns EINVAL_* on a bad
 * configuration or shape. */
int dion2_workspace_size(const dion2_matrix* mats, int32_t n, const dion2_config* cfg, size_t* bytes_out);

/* One Dion2 step on one matrix (== dion2_step_batched with n = 1). */
int dion2_step(const dion2_matrix* mat, const dion2_config* cfg, void* workspace, size_t ws_bytes, void* stream);

/* One Dion2 step on every matrix of mats[0..n) (HOST array of descriptors).
 * Matrices are independent (Alg. 1 is per matrix parameter); the
 * library batches each phase over all of them. */
int dion2_step_batched(const dion2_matrix* mats, int32_t n, const dion2_config* cfg,
                       void* workspace, size_t ws_bytes, void* stream);

/* Reads the workspace's status word after the work already enqueued on `stream` (the stream
 * the step ran on) has finished: an asynchronous copy on `stream`, then a synchronisation of
 * that stream only (other streams keep running).  Returns DION2_OK or DION2_ENONFINITE (and the
 * index of the first matrix whose scores were non-finite in *first_bad_matrix, -1 if none),
 * DION2_ECUDA on a CUDA error.  The status word is cleared at the start of every step. */
int dion2_get_status(const void* workspace, void* stream, int32_t* first_bad_matrix);

/* Drops every cached plan (and frees its device tables) whose workspace base lies in
 * [workspace, workspace + bytes): call it before freeing or reusing a workspace allocation.
 * Plans are otherwise kept for the life of the process, one per (shapes, config, workspace
 * address).  Synchronises the device (the tables may be in use).  Returns the number of plans
 * dropped. */
int32_t dion2_release_workspace(const void* workspace, size_t bytes);

/* Human-readable name of a status code (static storage). */
const char* dion2_strerror(int code);

/* Per-phase device timing (CUDA events recorded on the step's stream around
 * every kernel launch).  Off by default; enabling it adds event records only. */
int dion2_set_phase_timing(int32_t enable);
/* Synchronises; writes the accumulated milliseconds and launch counts per
 * phase since the last reset (HOST arrays of cap entries), then resets. */
int dion2_get_phase_times(float* ms_out, int32_t* launches_out, int32_t cap, int32_t* n_phases_out);
/* Name of phase i ("momentum_score", "select", "gather", "ns_gram", "ns_poly", "ns_apply", "scatter", ...). */
const char* dion2_phase_name(int32_t i);

/* ------------------------------------------------------------------------------------------
 * Multi-GPU: owner-compute step over P ranks (paper P:113: "only the
 * selected subset of the matrix ... communicated").
 *
 * Every matrix is sharded over the P ranks along its NON-selection axis (the selection axis
 * is resolved from the GLOBAL shape exactly as in dion2_step: auto = rows iff m <= n):
 *   rows mode: rank r holds columns [r*n/P, (r+1)*n/P) of W, M, G   (shard rows x cols/P)
 *   cols mode: rank r holds rows    [r*m/P, (r+1)*m/P) of W, M, G   (shard rows/P x cols)
 * so every rank owns a slice of EVERY row (column) that can be selected.  The step:
 *   1. M <- M + G and partial l1 scores on the local shard            (K1, local)
 *   2. all-gather of the partial scores, summed in rank order         (NCCL; identical on all ranks)
 *   3. top-k on every rank (identical K everywhere; no index traffic)  (K2)
 *   4. X-piece = wide(M[K])[:, this rank's block] (k x o/P, fp16 with the prescale of R24), local selective decay
 *   5. pieces -> owner of the matrix (grouped ncclSend/ncclRecv)      (bytes ~ alpha)
 *   6. owner: assemble X, Newton-Schulz, split O into pieces           (tcgen05 NS)
 *   7. O pieces -> back to every rank; local W[K] update              (K7, local)
 * Short X under ns_form AUTO (k <= 128, reading R25) skip steps 4-7's exchange: after step 3
 * every rank writes the fp64 Gram matrix of its column block X_r, one all-reduce sums them
 * (A = sum_r X_r X_r^T), and every rank runs the recursion and applies X_T,r = s Q X_r to its
 * own block before the decay -- exact, no pieces, no owner.
 * Owners are assigned by LPT on NS FLOPs, identically on every rank.  All sizes are known on the
 * host, so nothing synchronises the host inside a step.  Requirements: the sharded dimension
 * divisible by P; rows mode n/P % 8 == 0; cols mode m/P % 32 == 0 and k <= 1024; k <= the other
 * dimension (always true in auto mode); tensor-core NS.  Otherwise DION2_EUNSUPPORTED.
 * ------------------------------------------------------------------------------------------ */
typedef struct {
  int64_t rows;        /* GLOBAL m = fan-out */
  int64_t cols;        /* GLOBAL n = fan-in */
  int64_t ld;          /* row stride (elements) of the local shard, >= shard cols */
  float* W;            /* local shard of W, fp32 */
  float* M;            /* local shard of M, fp32 */
  const void* G;       /* local shard of G, dtype cfg.grad_dtype */
  int32_t* sel_out;    /* optional [k]: the selected indices (identical on every rank) */
  int32_t m_transposed; /* 1: the local M shard is stored TRANSPOSED, [shard cols x ldm] row-major
                           (column-mode matrices only, DION2_EUNSUPPORTED otherwise): the local
                           column gather becomes a row gather; local to this rank, the exchanged
                           pieces are the same either way */
  int32_t reserved;     /* must be 0 */
  int64_t ldm;          /* row stride of the transposed M shard (>= shard rows) */
} dion2_shard;

/* Host-only layout query for rank `rank` of `world` (no device work).  Any output may be NULL.
 *   axis_out[n]          resolved selection axis per matrix
 *   owner_out[n]         owning rank per matrix (LPT on NS FLOPs, ties -> lower index / rank)
 *   shard_rows_out[n], shard_cols_out[n]   local shard shape
 *   send_bytes_out[world], recv_bytes_out[world]   bytes this rank sends to / receives from each
 *                        peer in ONE exchange direction (gather-to-owner; scatter-back mirrors it)
 *   ws_bytes_out         workspace this rank needs */
int dion2_dist_info(const dion2_shard* shards, int32_t n, const dion2_config* cfg, int32_t world, int32_t rank,
                    int32_t* axis_out, int32_t* owner_out, int64_t* shard_rows_out, int64_t* shard_cols_out,
                    int64_t* send_bytes_out, int64_t* recv_bytes_out, size_t* ws_bytes_out);

/* One distributed step on this rank.  nccl_comm: an ncclComm_t (e.g. torch's
 * ProcessGroupNCCL._comm_ptr()) spanning `world` ranks; NCCL calls are enqueued on `stream`.
 * comm_bytes_out (HOST, optional): bytes this rank sent over the interconnect in this step. */
int dion2_step_batched_dist(const dion2_shard* shards, int32_t n, const dion2_config* cfg, void* workspace,
                            size_t ws_bytes, void* nccl_comm, int32_t world, int32_t rank, void* stream,
                            uint64_t* comm_bytes_out);

/* Exchange mode of the last distributed or DP-sync step on `workspace` (the same pointer passed
 * to dion2_step_batched_dist / _dpsync): 1 = direct peer stores / loads over symmetric memory
 * (DION2_FLAG_DIST_DIRECT honoured), 0 = NCCL send / recv (flag unset, or the fallback when the
 * NCCL device API or a single NVLink domain is unavailable -- decided identically on every
 * rank), -1 = no distributed plan on that workspace.  Host-only. */
int dion2_dist_exchange_mode(const void* workspace);

/* Loopback: all `world` ranks in this process on ONE device, exchanges done with device copies
 * on `stream` (tests the distributed layout and kernels without NCCL or several GPUs).
 * shards: [world * n], rank-major; workspaces: [world] HOST array of per-rank workspaces. */
int dion2_step_batched_loopback(const dion2_shard* shards, int32_t n, const dion2_config* cfg,
                                void* const* workspaces, size_t ws_bytes, int32_t world, void* stream,
                                uint64_t* comm_bytes_out);

/* ------------------------------------------------------------------------------------------
 * Compressed DP-sync (paper 3.2): `world` data-parallel replicas, each holding the
 * FULL W and M and its OWN local gradient G (no gradient all-reduce).  With the random rule
 * (cfg.select = DION2_SELECT_RANDOM, identical seed/step on every replica) the selection needs
 * no global state, so each replica accumulates M <- M + G locally, draws the same K, and only
 * the selected fp32 submatrix M[K, :] (or M[:, K]) is averaged across replicas (one
 * ncclAllReduce of sum_j k_j*o_j floats instead of sum_j m_j*n_j).  Every replica then runs the
 * rest of Alg. 1 on identical rows, so W stays identical while unselected momentum rows diverge;
 * by linearity the mean momentum equals the full-sync momentum and the W trajectory equals
 * full gradient sync ("the information that is synchronized suffices to compute the correct
 * parameter update").  cfg.select must be RANDOM (EUNSUPPORTED otherwise).  Matrices
 * with m_transposed = 1 contribute the rows of S^T = M^T[K, :] to the averaged buffer; every
 * replica must pass the same m_transposed flags.
 * ------------------------------------------------------------------------------------------ */
int dion2_dpsync_workspace_size(const dion2_matrix* mats, int32_t n, const dion2_config* cfg, int32_t world,
                                size_t* bytes_out);
int dion2_step_batched_dpsync(const dion2_matrix* mats, int32_t n, const dion2_config* cfg, void* workspace,
                              size_t ws_bytes, void* nccl_comm, int32_t world, int32_t rank, void* stream,
                              uint64_t* comm_bytes_out);
/* All replicas in one process on one device (mats: [world * n], replica-major; the all-reduce is
 * emulated with device copies and a fixed-order sum). */
int dion2_step_batched_dpsync_loopback(const dion2_matrix* mats, int32_t n, const dion2_config* cfg,
                                       void* const* workspaces, size_t ws_bytes, int32_t world, void* stream,
                                       uint64_t* comm_bytes_out);

/* Number of kernel launches the last step enqueued. */
int32_t dion2_last_launch_count(void);

int32_t dion2_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DION2_H_ */
