// fp32 SIMT Newton-Schulz GEMM: the validation path (precision = FP32).
// Same three phases and epilogue algebra as the tcgen05 kernel
// (k_ns_tcgen05.cu), fp32 FFMA throughout (TF32 would miss the 1e-5 gate).
// Not the hot path: it exists so the GPU step can be checked against the
// fp64 oracle to ~1e-6 (SURVEY 8(c.3) "fp32 validation NS").
#include "kernels.cuh"

namespace dion2 {

constexpr int kSB = 64, kSK = 16;

__global__ void __launch_bounds__(256) k_ns_gemm_simt_f32(const NsParams P, int group) {
  const NsGroup& g = P.g[group];
  const int z = blockIdx.z;
  const int m0 = blockIdx.y * kSB, n0 = blockIdx.x * kSB;
  const float* A = reinterpret_cast<const float*>(g.a) + (int64_t)z * g.a_mstride;
  const float* B = reinterpret_cast<const float*>(g.b) + (int64_t)z * g.b_mstride;
  float* D = reinterpret_cast<float*>(g.out) + (int64_t)z * g.out_mstride;
  const float* C = g.cin ? reinterpret_cast<const float*>(g.cin) + (int64_t)z * g.cin_mstride : nullptr;
  const int K = g.k_blocks * 64;

  __shared__ float As[kSK][kSB + 4];
  __shared__ float Bs[kSK][kSB + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += kSK) {
    // 64x16 A tile and 16x64 B tile: 1024 elements each, 4 per thread
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = threadIdx.x + 256 * i;
      const int r = e / kSK, c = e % kSK;  // A: row r (m), col c (k)
      As[c][r] = A[(int64_t)(m0 + r) * g.lda + k0 + c];
      if (P.b_kmajor) {
        Bs[c][r] = B[(int64_t)(n0 + r) * g.ldb + k0 + c];         // Bop(k, n) = B[n][k]
      } else {
        const int kr = e / kSB, nc = e % kSB;
        Bs[kr][nc] = B[(int64_t)(k0 + kr) * g.ldb + n0 + nc];     // Bop(k, n) = B[k][n]
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kSK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  float osc = 1.f;
  if (P.scale_sel) osc = P.ns_scale_all[4 * g.gmats[z] + (P.scale_sel - 1)];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + ty * 4 + i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = n0 + tx * 4 + j;
      float v = P.cacc * acc[i][j];
      if (C) v += P.cC * C[(int64_t)r * g.cin_ld + c];
      if (r == c) v += P.diag;
      D[(int64_t)r * g.out_ld + c] = osc * v;
    }
  }
}

}  // namespace dion2
