// K3: gather + selective decay + sum of squares; norm finalize; K7: sparse update.
//
//   K3  X = wide(M[K, :])  (pre-decay, Alg. 1 l.4 before l.5)
//       M[K, :] <- mu * M[K, :]   Eq. (error-feedback)
//       partial sums of x^2 for X0 = X / (||X||_F + eps)   (reading R3)
//   K7  W[K, :] <- W[K, :] - eta*sqrt(fan-out/fan-in) * O  (Alg. 1 l.6)
//       unselected rows/columns of W are never touched (bit-identical).
//
// Both kernels walk the selected submatrix S (rows mode: S = M[K,:], k x n;
// cols mode: S = M[:,K], m x k) in 32 x 64 tiles.  X (and O) are stored in
// the wide orientation (p <= q): X = S, or X = S^T through a shared-memory
// transpose so both the M/W side and the X side stay coalesced.
#include "kernels.cuh"

namespace dion2 {

template <typename XT> __device__ __forceinline__ XT to_x(float v);
template <> __device__ __forceinline__ float to_x<float>(float v) { return v; }
template <> __device__ __forceinline__ __half to_x<__half>(float v) { return __float2half_rn(v); }
__device__ __forceinline__ float from_x(float v) { return v; }
__device__ __forceinline__ float from_x(__half v) { return __half2float(v); }

__device__ __forceinline__ int find_mat(const int32_t* __restrict__ prefix, int n, int t) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// element (a, b) of S lives at M[row(a) * ld + col(b)]
__device__ __forceinline__ int64_t s_row(const MatDesc& md, int a) { return md.axis == kAxisRows ? md.sel[a] : a; }
__device__ __forceinline__ int64_t s_col(const MatDesc& md, int b) { return md.axis == kAxisRows ? b : md.sel[b]; }

template <typename XT>
__global__ void __launch_bounds__(256) k_gather_decay(const MatDesc* __restrict__ mats,
                                                      const int32_t* __restrict__ tile_prefix_mats, int n_mats,
                                                      int total_tiles, const int32_t* __restrict__ bad, int decay, float mu_arg) {
  __shared__ float tile[kTileA][kTileB + 1];
  __shared__ float wsum[8];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 col-quads x 16 rows
  for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
    const int mi = find_mat(tile_prefix_mats, n_mats, t);
    const MatDesc& md = mats[mi];
    if (md.mt) continue;  // transposed M: gathered by the row path on M^T (block-uniform)
    const int local = t - md.gather_tile_base;
    const int ta = local / md.gather_tiles_b, tb = local % md.gather_tiles_b;
    const int a0 = ta * kTileA, b0 = tb * kTileB;
    const bool skip = bad[mi] != 0;
    const float mu = decay ? mu_arg : 1.f;
    float ss = 0.f;
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int al = ty + 16 * rr, a = a0 + al;
      const int bl = tx * 4, b = b0 + bl;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (a < md.sr) {
        const int64_t row = s_row(md, a);
        float* mrow = md.M + row * md.ld;
        if (md.axis == kAxisRows && md.vec4 && b + 3 < md.sc) {
          float4* p = reinterpret_cast<float4*>(mrow + b);
          float4 x = *p;
          v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
          if (!skip && decay) *p = make_float4(mu * x.x, mu * x.y, mu * x.z, mu * x.w);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (b + c < md.sc) {
              float* p = mrow + s_col(md, b + c);
              v[c] = *p;
              if (!skip && decay) *p = mu * v[c];
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        tile[al][bl + c] = v[c];
        ss += v[c] * v[c];
      }
    }
    // deterministic block reduce of the tile's sum of squares
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
      float s = 0.f;
      for (int w = 0; w < 8; ++w) s += wsum[w];
      md.sumsq_partials[local] = s;
    }
    // The tile grid covers the padded extent of X, so every step also rewrites
    // X's zero padding (zero rows / columns are exact no-ops for NS) and the
    // workspace needs no state between calls.
    XT* X = reinterpret_cast<XT*>(md.X0);
    const float xs = md.ns_scale[2];  // fp16 prescale (K2, reading R24); 1 on the fp32 path
    if (!md.transposed) {
      // X[a][b] = S[a][b]
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int al = ty + 16 * rr, a = a0 + al;
        if (a < md.sa_pad) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int b = b0 + tx * 4 + c;
            if (b < md.sb_pad) X[(int64_t)a * md.q_pad + b] = to_x<XT>(xs * tile[al][tx * 4 + c]);
          }
        }
      }
    } else {
      // X[b][a] = S[a][b]: thread -> (b_local = tid/4, 8 consecutive a)
      const int bl = threadIdx.x >> 2, ac = (threadIdx.x & 3) * 8;
      const int b = b0 + bl;
      if (b < md.sb_pad) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int a = a0 + ac + i;
          if (a < md.sa_pad) X[(int64_t)b * md.q_pad + a] = to_x<XT>(xs * tile[ac + i][bl]);
        }
      }
    }
    __syncthreads();
  }
}
void launch_gather_decay(bool x16, int blocks, cudaStream_t s, const MatDesc* mats, const int32_t* tile_prefix_mats,
                         int n_mats, int total_tiles, const int32_t* bad, int decay, float mu) {
  if (x16)
    k_gather_decay<__half><<<blocks, 256, 0, s>>>(mats, tile_prefix_mats, n_mats, total_tiles, bad, decay, mu);
  else
    k_gather_decay<float><<<blocks, 256, 0, s>>>(mats, tile_prefix_mats, n_mats, total_tiles, bad, decay, mu);
}

// One warp per matrix: fixed-order sum of the tile partials -> s = 1 / (||X||_F + eps), stored
// as s' = s / xs (the stored X is xs X, reading R24) with s'^2.
__global__ void k_norm_finalize(const MatDesc* __restrict__ mats, int n_mats, float eps) {
  const int lane = threadIdx.x & 31;
  const int mi = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (mi >= n_mats) return;
  const MatDesc& md = mats[mi];
  const int nt = md.n_sumsq;
  float s = 0.f;
  for (int i = lane; i < nt; i += 32) s += md.sumsq_partials[i];
  s = warp_sum(s);
  if (lane == 0) {
    const float inv = 1.0f / (sqrtf(s) + eps) / md.ns_scale[2];
    md.ns_scale[0] = inv;
    md.ns_scale[1] = inv * inv;
  }
}

template <typename XT, typename WT>
__global__ void __launch_bounds__(256) k_scatter_update(const MatDesc* __restrict__ mats,
                                                        const int32_t* __restrict__ tile_prefix_mats, int n_mats,
                                                        int total_tiles, const int32_t* __restrict__ bad, float lr,
                                                        const float* __restrict__ lr_dev) {
  __shared__ float tile[kTileA][kTileB + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
    const int mi = find_mat(tile_prefix_mats, n_mats, t);
    const MatDesc& md = mats[mi];
    if (bad[mi] || md.spath != 0) continue;  // block-uniform; spath != 0: a streaming scatter owns it
    const int local = t - md.gather_tile_base;
    const int ta = local / md.gather_tiles_b, tb = local % md.gather_tiles_b;
    const int a0 = ta * kTileA, b0 = tb * kTileB;
    if (a0 >= md.sr || b0 >= md.sc) continue;  // padding-only tile (block-uniform)
    const XT* X = reinterpret_cast<const XT*>(md.final_in_x1 ? md.X1 : md.X0);
    if (md.transposed) {
      // O_S[a][b] = X[b][a]: coalesced read along a, stage in smem
      const int bl = threadIdx.x >> 2, ac = (threadIdx.x & 3) * 8;
      const int b = b0 + bl;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int a = a0 + ac + i;
        tile[ac + i][bl] = (b < md.sc && a < md.sr) ? from_x(X[(int64_t)b * md.q_pad + a]) : 0.f;
      }
      __syncthreads();
    }
    const float sc = (lr_dev ? __ldg(lr_dev) : lr) * md.update_scale;
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int al = ty + 16 * rr, a = a0 + al;
      if (a >= md.sr) continue;
      const int64_t row = s_row(md, a);
      WT* wrow = reinterpret_cast<WT*>(md.W) + row * md.ld;
      float o[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int b = b0 + tx * 4 + c;
        o[c] = 0.f;
        if (b < md.sc) o[c] = md.transposed ? tile[al][tx * 4 + c] : from_x(X[(int64_t)a * md.q_pad + b]);
      }
      const int b = b0 + tx * 4;
      if (md.axis == kAxisRows && md.vec4 && b + 3 < md.sc) {
        float4 w = ld_w4(wrow, b >> 2);
        w.x -= sc * o[0]; w.y -= sc * o[1]; w.z -= sc * o[2]; w.w -= sc * o[3];
        st_w4(wrow, b >> 2, w);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (b + c < md.sc) {
            WT* p = wrow + s_col(md, b + c);
            st_w(p, ld_w(p) - sc * o[c]);
          }
        }
      }
      if (md.O_out) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (b + c < md.sc) md.O_out[(int64_t)a * md.sc + b + c] = o[c];
      }
    }
    if (md.transposed) __syncthreads();
  }
}
void launch_scatter_update(bool x16, bool w_bf16, int blocks, cudaStream_t s, const MatDesc* mats,
                           const int32_t* tile_prefix_mats, int n_mats, int total_tiles, const int32_t* bad, float lr,
                           const float* lr_dev) {
  if (x16 && w_bf16)
    k_scatter_update<__half, __nv_bfloat16><<<blocks, 256, 0, s>>>(mats, tile_prefix_mats, n_mats, total_tiles, bad, lr,
                                                                   lr_dev);
  else if (x16)
    k_scatter_update<__half, float><<<blocks, 256, 0, s>>>(mats, tile_prefix_mats, n_mats, total_tiles, bad, lr, lr_dev);
  else if (w_bf16)
    k_scatter_update<float, __nv_bfloat16><<<blocks, 256, 0, s>>>(mats, tile_prefix_mats, n_mats, total_tiles, bad, lr,
                                                                  lr_dev);
  else
    k_scatter_update<float, float><<<blocks, 256, 0, s>>>(mats, tile_prefix_mats, n_mats, total_tiles, bad, lr, lr_dev);
}

// Full-decay ablation: M <- mu * M on the UNSELECTED part (the
// selected part was decayed by K3).  One block per (matrix, 64-row slab).
__global__ void k_full_decay(const MatDesc* __restrict__ mats, int n_mats, const int32_t* __restrict__ bad, float mu) {
  const int mi = blockIdx.y;
  if (mi >= n_mats) return;
  const MatDesc& md = mats[mi];
  if (bad[mi]) return;
  // mark selected indices of the selection axis in shared memory
  extern __shared__ unsigned char is_sel[];
  for (int i = threadIdx.x; i < md.d; i += blockDim.x) is_sel[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < md.k; i += blockDim.x) is_sel[md.sel[i]] = 1;
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * 64;
  const int64_t rend = md.rows < r0 + 64 ? md.rows : r0 + 64;
  for (int64_t r = r0; r < rend; ++r) {
    if (md.axis == kAxisRows && is_sel[r]) continue;
    for (int64_t c = threadIdx.x; c < md.cols; c += blockDim.x) {
      if (md.axis == kAxisCols && is_sel[c]) continue;
      md.M[r * md.ld + c] *= mu;
    }
  }
}

}  // namespace dion2
