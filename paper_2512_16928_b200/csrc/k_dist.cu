// Kernels of the owner-compute distributed step (dion2_dist.cu).
//
// Every matrix is sharded over P ranks along its NON-selection axis (rows mode:
// column shards m x n/P; cols mode: row shards m/P x n).  Each rank then holds a
// complete slice of every row (column) of the selection axis, so
//   * its l1 scores are partial sums that combine exactly across ranks
//     (k_sum_rank_scores, fixed rank order -> bit-identical scores everywhere), and
//   * its piece of the selected submatrix X = wide(M[K]) is a fixed k x (o/P)
//     column block of X, so the gather-to-owner and scatter-back exchanges have
//     host-known sizes (no per-step host synchronisation).
// The owner assembles X from the P column blocks (k_assemble_pieces), runs NS,
// and splits X_T back into blocks (k_disassemble_pieces).
#include <algorithm>

#include "kernels.cuh"

namespace dion2 {

// cols-mode shards: local column scores = fixed-order sum of K1's row-block partials
__global__ void k_cols_local_scores(const MatDesc* __restrict__ mats, const int32_t* __restrict__ col_mats,
                                    int n_col_mats) {
  const int li = blockIdx.y;
  if (li >= n_col_mats) return;
  const MatDesc& md = mats[col_mats[li]];
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < md.cols; c += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int rb = 0; rb < md.rowblocks; ++rb) s += md.col_partials[(int64_t)rb * md.cols + c];
    md.scores[c] = s;
  }
}

// out[x] = sum_{r = 0..P-1} gathered[r * total + x], in rank order
__global__ void k_sum_rank_scores(const float* __restrict__ gathered, float* __restrict__ out, int64_t total,
                                  int world) {
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int r = 0; r < world; ++r) s += gathered[(int64_t)r * total + x];
    out[x] = s;
  }
}

// per matrix: raw sum of the K3 unit partials (fixed order) -> out[mi]
__global__ void k_piece_sumsq(const MatDesc* __restrict__ mats, int n_mats, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int mi = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (mi >= n_mats) return;
  const MatDesc& md = mats[mi];
  float s = 0.f;
  for (int i = lane; i < md.n_sumsq; i += 32) s += md.sumsq_partials[i];
  s = warp_sum(s);
  if (lane == 0) out[mi] = s;
}

// Owner side.  For owned matrix jj (global index gj): X0[i][r*qo + c] = piece_r[i][c]
// for i < k, c < qo; zeros elsewhere in [p_pad x q_pad].  One block per (row i, matrix).
// xs_all: the rank's [n_total][4] NS scale words; word 2 of matrix g is its fp16 prescale (K2 ran
// on every rank with the same combined scores, so it is the prescale of every piece)
__global__ void k_assemble_pieces(const MatDesc* __restrict__ omats, PieceTable T, const uint8_t* __restrict__ recv,
                                  const float* __restrict__ sumsq_all, const float* __restrict__ xs_all, int n_total,
                                  float eps) {
  const int jj = blockIdx.y;
  const MatDesc& md = omats[jj];
  const int i = blockIdx.x;
  if (i >= md.p_pad) return;
  const int qo = md.q / T.world;
  __half* xrow = reinterpret_cast<__half*>(md.X0) + (int64_t)i * md.q_pad;
  if (T.inplace[jj]) {
    // the NS kernels read the pieces in place: only the norm below
  } else if (i < md.k) {
    for (int r = 0; r < T.world; ++r) {
      const __half* src = reinterpret_cast<const __half*>(recv + r * T.rstride + T.roff[jj * T.world + r]) +
                                 (int64_t)i * qo;
      const uint4* s16 = reinterpret_cast<const uint4*>(src);
      uint4* d16 = reinterpret_cast<uint4*>(xrow + (int64_t)r * qo);
      for (int c = threadIdx.x; c < qo / 8; c += blockDim.x) d16[c] = s16[c];
    }
    for (int c = md.q + threadIdx.x; c < md.q_pad; c += blockDim.x) xrow[c] = __float2half_rn(0.f);
  } else {
    uint4* d16 = reinterpret_cast<uint4*>(xrow);
    for (int c = threadIdx.x; c < md.q_pad / 8; c += blockDim.x) d16[c] = make_uint4(0, 0, 0, 0);
  }
  if (i == 0 && threadIdx.x == 0) {
    float s = 0.f;
    for (int r = 0; r < T.world; ++r) s += sumsq_all[(int64_t)r * n_total + T.gidx[jj]];
    const float inv = 1.0f / (sqrtf(s) + eps) / xs_all[4 * (int64_t)T.gidx[jj] + 2];  // reading R24
    md.ns_scale[0] = inv;
    md.ns_scale[1] = inv * inv;
  }
}

// piece_r[i][c] = X_T[i][r*qo + c] for i < k
__global__ void k_disassemble_pieces(const MatDesc* __restrict__ omats, PieceTable T, uint8_t* __restrict__ send) {
  const int jj = blockIdx.y;
  const MatDesc& md = omats[jj];
  const int i = blockIdx.x;
  if (i >= md.k || T.inplace[jj] == 1) return;  // in place: the apply wrote the pieces itself
  const int qo = md.q / T.world;
  const __half* xrow =
      reinterpret_cast<const __half*>(md.final_in_x1 ? md.X1 : md.X0) + (int64_t)i * md.q_pad;
  for (int r = 0; r < T.world; ++r) {
    __half* dst = reinterpret_cast<__half*>(send + r * T.rstride + T.roff[jj * T.world + r]) +
                         (int64_t)i * qo;
    const uint4* s16 = reinterpret_cast<const uint4*>(xrow + (int64_t)r * qo);
    uint4* d16 = reinterpret_cast<uint4*>(dst);
    for (int c = threadIdx.x; c < qo / 8; c += blockDim.x) d16[c] = s16[c];
  }
}

void launch_cols_local_scores(cudaStream_t s, const MatDesc* mats, const int32_t* col_mats, int n_col_mats,
                              int64_t max_cols) {
  dim3 grid((unsigned)((max_cols + 255) / 256), n_col_mats);
  k_cols_local_scores<<<grid, 256, 0, s>>>(mats, col_mats, n_col_mats);
}
void launch_sum_rank_scores(cudaStream_t s, const float* gathered, float* out, int64_t total, int world) {
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  k_sum_rank_scores<<<blocks, 256, 0, s>>>(gathered, out, total, world);
}
void launch_piece_sumsq(cudaStream_t s, const MatDesc* mats, int n, float* out) {
  k_piece_sumsq<<<(n + 7) / 8, 256, 0, s>>>(mats, n, out);
}
void launch_assemble(cudaStream_t s, const MatDesc* omats, int n_owned, int max_p_pad, const PieceTable& T,
                     const uint8_t* recv, const float* sumsq_all, const float* xs_all, int n_total, float eps) {
  dim3 grid(max_p_pad, n_owned);
  k_assemble_pieces<<<grid, 256, 0, s>>>(omats, T, recv, sumsq_all, xs_all, n_total, eps);
}
void launch_disassemble(cudaStream_t s, const MatDesc* omats, int n_owned, int max_k, const PieceTable& T,
                        uint8_t* send) {
  dim3 grid(max_k, n_owned);
  k_disassemble_pieces<<<grid, 256, 0, s>>>(omats, T, send);
}

}  // namespace dion2
