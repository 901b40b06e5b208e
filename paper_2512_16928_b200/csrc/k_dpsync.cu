// Compressed DP-sync: pack the selected fp32 submatrix
// S = M[K, :] (or M[:, K]) of every matrix into one contiguous buffer for the
// all-reduce, and write the averaged rows back.  One warp per row of S; rows
// mode streams contiguous rows of M, cols mode gathers the selected columns, and cols
// mode with transposed M packs the contiguous rows of S^T (every replica must use the
// same layout).
#include <algorithm>

#include "kernels.cuh"

namespace dion2 {

__device__ __forceinline__ int find_row(const int32_t* __restrict__ prefix, int n, int t) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// unit = one row a of S of one matrix; row_prefix[mi] = first unit of matrix mi
template <bool kUnpack>
__global__ void __launch_bounds__(256) k_dp_pack(const MatDesc* __restrict__ mats, const int32_t* __restrict__ row_prefix,
                                                 const int64_t* __restrict__ buf_off, int n_mats, int total_rows,
                                                 float* __restrict__ buf, float scale, const int32_t* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int warp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  for (int u = warp; u < total_rows; u += nwarps) {
    const int mi = find_row(row_prefix, n_mats, u);
    const MatDesc& md = mats[mi];
    if (kUnpack && bad[mi]) continue;
    const int a = u - row_prefix[mi];
    if (md.mt) {
      // transposed M (cols mode): unit a = row sel[a] of M^T = S^T row a, contiguous
      float* b = buf + buf_off[mi] + (int64_t)a * md.rows;
      float* mrow = md.M + (int64_t)md.sel[a] * md.ldm;
      for (int c = lane; c < md.rows; c += 32) {
        if (kUnpack) mrow[c] = scale * b[c];
        else b[c] = mrow[c];
      }
      continue;
    }
    float* b = buf + buf_off[mi] + (int64_t)a * md.sc;
    if (md.axis == kAxisRows) {
      float* mrow = md.M + (int64_t)md.sel[a] * md.ld;
      for (int c = lane; c < md.sc; c += 32) {
        if (kUnpack) mrow[c] = scale * b[c];
        else b[c] = mrow[c];
      }
    } else {
      float* mrow = md.M + (int64_t)a * md.ld;
      for (int c = lane; c < md.sc; c += 32) {
        float* p = mrow + md.sel[c];
        if (kUnpack) *p = scale * b[c];
        else b[c] = *p;
      }
    }
  }
}

// The all-reduced buffer ends with two floats per matrix: the replica's largest score and its
// non-finite flag.  After the sum every replica sees the same totals, so every replica skips a
// matrix that is non-finite on ANY replica (no NaN rows unpacked, no W / M[K] writes, status
// reported everywhere) and takes the same fp16 prescale from the summed bound (>= the largest
// score of every replica, hence >= any entry of the averaged rows; reading R24).
__global__ void k_dp_tail(const MatDesc* __restrict__ mats, int n_mats, float* __restrict__ tail,
                          int32_t* __restrict__ bad, int32_t* __restrict__ status, int combine) {
  const int mi = blockIdx.x * blockDim.x + threadIdx.x;
  if (mi >= n_mats) return;
  const MatDesc& md = mats[mi];
  if (!combine) {
    tail[2 * mi] = bad[mi] ? 0.f : md.ns_scale[3];
    tail[2 * mi + 1] = bad[mi] ? 1.f : 0.f;
    return;
  }
  const bool any_bad = tail[2 * mi + 1] != 0.f || !(tail[2 * mi] <= 3.402823466e38f);
  if (any_bad) {
    bad[mi] = 1;
    set_status_bad(status, md.mid);
  }
  md.ns_scale[2] = (md.x16 && !any_bad) ? x16_prescale(tail[2 * mi]) : 1.f;
}

// Direct (peer-memory) reduce-scatter + all-gather of the packed buffers (DION2_FLAG_DIST_DIRECT):
// this rank owns floats [rank * per, (rank + 1) * per) of the buffer; it sums them over the P
// replicas' input buffers in rank order (as k_sum_rank_scores: the same bits on every replica)
// and stores the sum into every replica's output buffer.  in / out may alias (loopback).
__global__ void __launch_bounds__(256) k_dp_reduce_direct(DpPeerBufs B, int P, int rank, int64_t total) {
  const int64_t per = (total + 4 * (int64_t)P - 1) / (4 * (int64_t)P) * 4;
  const int64_t lo = (int64_t)rank * per, hi = lo + per < total ? lo + per : total;
  for (int64_t x = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < hi; x += (int64_t)gridDim.x * blockDim.x) {
    float v[kMaxPieceRanks];
#pragma unroll
    for (int r = 0; r < kMaxPieceRanks; ++r)
      if (r < P) v[r] = __ldcg(B.in[r] + x);
    float s = 0.f;
#pragma unroll
    for (int r = 0; r < kMaxPieceRanks; ++r)
      if (r < P) s += v[r];
#pragma unroll
    for (int r = 0; r < kMaxPieceRanks; ++r)
      if (r < P) B.out[r][x] = s;
  }
}

void launch_dp_reduce_direct(cudaStream_t s, const DpPeerBufs& B, int P, int rank, int64_t total, int sms) {
  const int64_t per = (total + 4 * (int64_t)P - 1) / (4 * (int64_t)P) * 4;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((per + 255) / 256, (int64_t)sms * 8));
  k_dp_reduce_direct<<<(unsigned)blocks, 256, 0, s>>>(B, P, rank, total);
}

void launch_dp_tail(cudaStream_t s, const MatDesc* mats, int n_mats, float* tail, int32_t* bad, int32_t* status,
                    bool combine) {
  k_dp_tail<<<(n_mats + 127) / 128, 128, 0, s>>>(mats, n_mats, tail, bad, status, combine ? 1 : 0);
}

void launch_dp_pack(bool unpack, cudaStream_t s, const MatDesc* mats, const int32_t* row_prefix, const int64_t* buf_off,
                    int n_mats, int total_rows, float* buf, float scale, const int32_t* bad) {
  const int blocks = (total_rows + 7) / 8;
  if (unpack)
    k_dp_pack<true><<<blocks, 256, 0, s>>>(mats, row_prefix, buf_off, n_mats, total_rows, buf, scale, bad);
  else
    k_dp_pack<false><<<blocks, 256, 0, s>>>(mats, row_prefix, buf_off, n_mats, total_rows, buf, scale, bad);
}

}  // namespace dion2
