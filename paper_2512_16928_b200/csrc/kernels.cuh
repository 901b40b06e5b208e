// kernels.cuh -- kernel entry points of the Dion2 step (launched by dion2_api.cu).
#pragma once
#include "common.cuh"

namespace dion2 {

constexpr int kMaxPieceRanks = 8;  // distributed owner step: piece tensor maps are made for P <= 8

// ---------------- K1 momentum + l1 score (k_momentum_score.cu)
constexpr int kColRowBlock = 256;  // rows per column-mode partial-sum block
__global__ void k_momentum_score_rows(const MatDesc* __restrict__ mats, const int32_t* __restrict__ row_mats,
                                      const int64_t* __restrict__ row_prefix, int n_row_mats, int64_t total_rows);
__global__ void k_momentum_score_cols(const MatDesc* __restrict__ mats, const int32_t* __restrict__ col_mats,
                                      const int64_t* __restrict__ tile_prefix, int n_col_mats, int64_t total_tiles);
// cols mode with M stored transposed: units = (row block of kColRowBlock rows, 32 columns)
__global__ void k_momentum_score_cols_mt(const MatDesc* __restrict__ mats, const int32_t* __restrict__ col_mats,
                                         const int64_t* __restrict__ tile_prefix, int n_col_mats,
                                         int64_t total_tiles);

// cols mode on tall matrices: scores[j] = sum of the K1 row-block partials of column j in a
// fixed order (8 strided row-block groups, then the groups in order), 32 columns per block
// over all listed matrices (prefix: int64 column offsets); K2 then reads final scores
__global__ void k_col_scores_finalize(const MatDesc* __restrict__ mats, const int32_t* __restrict__ list,
                                      const int64_t* __restrict__ prefix, int n_list, int64_t total);

// 16-B aligned whole tiles (rows % 256 == 0, cols % 64 == 0), fp32 or bf16 G: cp.async-pipelined
// variant of k_momentum_score_cols_mt over the same units; stages 2 / 3 / 4
void launch_momentum_score_cols_mt_pipe(int stages, bool bf16, int blocks, cudaStream_t s, const MatDesc* mats,
                                        const int32_t* col_mats, const int64_t* tile_prefix, int n_col_mats,
                                        int64_t total_units);
int momentum_score_cols_mt_pipe_attrs(int stages, bool bf16);  // sets the smem attributes; returns blocks per SM

// ---------------- K2 top-k select (k_select.cu)
constexpr int kSelectThreads = 1024;
// random_sel = 1: Random rule with Philox keys (seed, step, md.mid); else the l1 rule
// list: [gridDim.x] matrix indices, or null = matrices 0 .. gridDim.x - 1
__global__ void k_topk_select(const MatDesc* __restrict__ mats, const int32_t* __restrict__ list,
                              int32_t* __restrict__ bad, int32_t* __restrict__ status,
                              int random_sel, uint64_t seed, uint64_t step);


// ---------------- K3 gather + decay + sum of squares, norm finalize; K7 scatter (k_gather_scatter.cu)
constexpr int kTileA = 32;   // S rows per gather/scatter tile
constexpr int kTileB = 64;   // S cols per gather/scatter tile
// host launchers (the templates are instantiated in their own translation unit)
void launch_gather_decay(bool x16, int blocks, cudaStream_t s, const MatDesc* mats, const int32_t* tile_prefix_mats,
                         int n_mats, int total_tiles, const int32_t* bad, int decay, float mu);
// lr_dev (optional): eta read on the device at run time (CUDA graphs under a schedule), else lr
// w_bf16: W stored as bf16 (dion2_config.w_dtype), the update computed in fp32 and rounded once
void launch_scatter_update(bool x16, bool w_bf16, int blocks, cudaStream_t s, const MatDesc* mats,
                           const int32_t* tile_prefix_mats, int n_mats, int total_tiles, const int32_t* bad, float lr,
                           const float* lr_dev);
__global__ void k_norm_finalize(const MatDesc* __restrict__ mats, int n_mats, float eps);

// streaming fast paths (k_gather_scatter_fast.cu): rows mode X = S, cols mode X = S^T
#define DION2_MAX_SELECT_DIM_WORDS 1536  // DION2_MAX_SELECT_DIM / 32
constexpr int kMaxColKFast = 1024;          // largest k of the cols streaming gather (32-row smem tile)
constexpr int kMaxColKScatter = 4096;       // largest k of the cols streaming scatter (8-row tile above 1024)
size_t cols_t_smem_bytes(int k, int mask_words);
void launch_fast_paths_attrs();
void launch_gather_rows(int blocks, cudaStream_t s, const MatDesc* mats, const int32_t* lm, const int32_t* lp, int nl,
                        int units, const int32_t* bad, float mu);
// TMA-staged rows gather (k_gather_tma.cu): 16-B aligned rows, n % 8 == 0; stages 4 or 6
void launch_gather_rows_tma(int stages, int blocks_per_sm_cap, cudaStream_t s, const MatDesc* mats, const int32_t* lm,
                            const int32_t* lp, int nl, int units, const int32_t* bad, float mu, int sms);
void launch_scatter_rows(bool w_bf16, int blocks, cudaStream_t s, const MatDesc* mats, const int32_t* lm,
                         const int32_t* lp, int nl, int units, const int32_t* bad, float lr, const float* lr_dev);
// max_k / max_n: largest k and column count over the matrices of the list (sizes the smem)
void launch_gather_cols_t(int blocks, int max_k, int64_t max_n, cudaStream_t s, const MatDesc* mats, const int32_t* lm,
                          const int32_t* lp, int nl, int units, const int32_t* bad, float mu);
void launch_scatter_cols_t(bool w_bf16, int blocks, int max_k, int64_t max_n, cudaStream_t s, const MatDesc* mats,
                           const int32_t* lm, const int32_t* lp, int nl, int units, const int32_t* bad, float lr,
                           const float* lr_dev);
__global__ void k_full_decay(const MatDesc* __restrict__ mats, int n_mats, const int32_t* __restrict__ bad, float mu);

// ---------------- distributed step (k_dist.cu)
struct PieceTable {
  const int32_t* gidx;     // [n_owned] global matrix index
  const int32_t* inplace;  // [n_owned] 1: the NS kernels read / write the pieces in place (no copy)
  const int64_t* roff;     // [n_owned * world] byte offset of owned matrix jj's piece in rank r's section
  int64_t rstride;         // bytes between consecutive ranks' sections
  int32_t world;
};
void launch_cols_local_scores(cudaStream_t s, const MatDesc* mats, const int32_t* col_mats, int n_col_mats,
                              int64_t max_cols);
void launch_sum_rank_scores(cudaStream_t s, const float* gathered, float* out, int64_t total, int world);
void launch_piece_sumsq(cudaStream_t s, const MatDesc* mats, int n, float* out);
void launch_assemble(cudaStream_t s, const MatDesc* omats, int n_owned, int max_p_pad, const PieceTable& T,
                     const uint8_t* recv, const float* sumsq_all, const float* xs_all, int n_total, float eps);
void launch_disassemble(cudaStream_t s, const MatDesc* omats, int n_owned, int max_k, const PieceTable& T,
                        uint8_t* send);


// ---------------- compressed DP-sync (k_dpsync.cu): M[K] <-> contiguous fp32 buffer
// tail[2 n]: combine = 0 packs {largest score, non-finite flag} per matrix before the all-reduce;
// combine = 1 reads the sums back: global non-finite flag (bad, status) and the fp16 prescale
void launch_dp_tail(cudaStream_t s, const MatDesc* mats, int n_mats, float* tail, int32_t* bad, int32_t* status,
                    bool combine);
void launch_dp_pack(bool unpack, cudaStream_t s, const MatDesc* mats, const int32_t* row_prefix, const int64_t* buf_off,
                    int n_mats, int total_rows, float* buf, float scale, const int32_t* bad);
// direct DP-sync exchange (peer memory): every replica's packed input and reduced output buffer
struct DpPeerBufs {
  const float* in[kMaxPieceRanks];
  float* out[kMaxPieceRanks];
};
void launch_dp_reduce_direct(cudaStream_t s, const DpPeerBufs& B, int P, int rank, int64_t total, int sms);

// ---------------- K4-K6 Newton-Schulz GEMMs
// D = oscale * (cacc * Aop . Bop + cC * C), written as OutT.
//   Aop: [M x K] row-major (K-major); Bop(k, n) = B[n][k] (b_kmajor) or B[k][n].
constexpr int kMaxGroups = 4;

struct NsGroup {
  int count;                 // matrices in the group
  int m_tiles, n_tiles, k_blocks;
  int tile_base;             // first global tile of the group
  const int32_t* gmats;      // [count] global matrix index (for the per-matrix scale)
  const void* a;  long long a_mstride; int lda;
  const void* b;  long long b_mstride; int ldb;
  void* out;      long long out_mstride; int out_ld;
  const void* cin; long long cin_mstride; int cin_ld;
  // distributed owner step (dion2_dist.cu): X0 / X_T live as P column pieces [rank][matrix][k][qo]
  // in the exchange buffers; the gram / apply read (and the apply writes) them through the
  // per-rank tensor maps NsTcParams::mapP[group][kind * P + r] (kind 0: box {64, 128} loads,
  // 1: box {64, 64} MN-major loads, 2: box {32, 32} stores).  pieces_qo = 0: plain layout.
  int pieces_qo, pieces_P, pieces_map;
  int pieces_load;           // gram / apply: the X operand is read from the received pieces
  int pieces_store;          // apply: X_T TMA-stored into the outgoing pieces (else into `out`)
};

struct NsParams {
  NsGroup g[kMaxGroups];
  int ngroups, total_tiles;
  float cacc, cC;
  float diag;                // added on the global diagonal (poly: C = a*I + b*A + c*A^2)
  int scale_sel;             // 0: oscale = 1; 1: s; 2: s^2
  int sym;                   // symmetric output: upper-triangle tiles only, mirrored by the epilogue (pair kernel)
  const float* ns_scale_all; // [n_mats][4] (MatDesc::ns_scale)
  int b_kmajor;
  int b_is_a;                // pair kernel: every group's B operand is its A operand (gram X X^T, poly
                             // A A): diagonal tiles load the A half only and use it for both
  int in_f16;                // operands (and cin) are fp16, else bf16
  int out_f16;               // output written as fp16, else bf16
  int reverse;               // walk the tile list backwards (L2 reuse of the previous launch's last writes)
  // upper-triangle storage of symmetric p x p buffers (pair kernel, Gram-space launches):
  int sym_in;                // operands hold only their upper 256 x 256 tiles: a lower k-block is read
                             // transposed (MN-major) from the stored upper tile
  int no_mirror;             // sym output: do not write the mirrored lower tiles
  // split-K (pair kernel, long-K gram launches that cannot fill the GPU): work item w =
  // tile * splitk + slice runs k-blocks [slice KB / splitk, (slice + 1) KB / splitk) and
  // stores raw fp32 accumulators to partial[w][256][256]; k_splitk_reduce sums the slices
  // in order (deterministic) and applies the epilogue
  int splitk;                // <= 1: off
  float* partial;
  // resident-A apply (k_ns_apply_pair.cu): total_tiles counts chunks of up to chunk_len column
  // blocks of one 256-row block, NsGroup::tile_base the group's first chunk
  int chunk_len;
};

// tcgen05 path (k_ns_tcgen05.cu): tensor maps for the TMA operand loads.
struct NsTcParams {
  CUtensorMap mapA[kMaxGroups];
  CUtensorMap mapB[kMaxGroups];
  CUtensorMap mapD[kMaxGroups];  // output (TMA store): box {32 cols, 32 rows, 1}, SWIZZLE_64B
  CUtensorMap mapAT[kMaxGroups]; // sym_in: the A buffer with box {64, 64} for transposed k-blocks
  CUtensorMap mapBT[kMaxGroups]; // sym_in: the B buffer with box {64, 64}
  // distributed owner step: per-rank piece maps of each group (see NsGroup::pieces_qo), kind-major
  CUtensorMap mapP[kMaxGroups][3 * kMaxPieceRanks];
  NsParams p;
};
void ns_tc_set_attrs();
void launch_ns_tc(int bn, int grid, cudaStream_t s, const NsTcParams& P);
void ns_pair_set_attrs();
void launch_ns_pair(int grid, cudaStream_t s, const NsTcParams& P);
void launch_splitk_reduce(cudaStream_t s, const NsParams& p);  // after a split-K pair launch
// apply on a CTA pair with A resident in shared memory (k_ns_apply_pair.cu): groups with
// k_blocks <= kMaxResidentKB (p_pad <= 512), m_tiles = p_pad / 256, MN-major B
constexpr int kMaxResidentKB = 8;
void ns_apply_pair_set_attrs();
void launch_ns_apply_pair(int grid, cudaStream_t s, const NsTcParams& P);

template <int BN>
constexpr int ns_tc_stages() { return BN == 256 ? 4 : 6; }
template <int BN>
constexpr int ns_tc_smem_bytes() {
  return 1024 /*align slack*/ + ns_tc_stages<BN>() * (128 * 64 * 2 + BN * 64 * 2) + 1024 /*barriers*/ +
         4 * 2 * 2048 /*epilogue staging: 4 warps x 2 buffers x (32 x 32 bf16)*/;
}

// Short X (p <= kTinyP rows) under ns_form AUTO (k_ns_small.cu): NS in fp64 Gram space straight
// from the pre-decay momentum, X_T stored as fp16 into X1; one CTA per matrix of `list`.
constexpr int kTinyP = 128;
struct NsSmallCoeffs {
  float c[16][3];
  int T;
  float eps;
};
// wide = false: p <= 64 (fp64 recursion); true: 64 < p <= 128 (fp32 recursion)
void launch_ns_small(cudaStream_t s, const MatDesc* mats, const int32_t* list, int n_list, const int32_t* bad,
                     const NsSmallCoeffs& C, bool wide);
// distributed step: per-rank partial Gram matrices of the local column blocks (fp64, kTinyP^2
// apart from Abase), then -- after their all-reduce -- the recursion and the local apply
void launch_ns_small_partial(cudaStream_t s, const MatDesc* mats, const int32_t* list, int n_list, double* Abase,
                             bool wide);
void launch_ns_small_finish(cudaStream_t s, const MatDesc* mats, const int32_t* list, int n_list, const int32_t* bad,
                            const double* Abase, const NsSmallCoeffs& C, bool wide);
void launch_add_f64(cudaStream_t s, double* dst, const double* src, int64_t n);

// fp32 SIMT validation path (k_ns_simt.cu): grid (n_tiles, m_tiles, count) per group.
__global__ void k_ns_gemm_simt_f32(const NsParams P, int group);

}  // namespace dion2
