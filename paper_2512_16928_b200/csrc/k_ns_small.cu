// Newton-Schulz of short X (p <= kTinyP = 64 rows) in fp64 Gram space, straight from the momentum.
//
// The 16-bit tensor-core path rounds X once per entry (fp16, 2^-11 relative).  On an X of a few
// rows whose spectrum is dominated by one or a few directions (a selected submatrix of a spiked
// momentum), that rounding is a large fraction of the weak directions, and a short X has few
// directions to average it over: emulated and measured up to 2-3.6% on the cumulative update at
// p <= 30 and 1.7-1.9% at p = 33..63 for sigma_1 / median ~ 250 (reading R25).  Such matrices are cheap, so
// AUTO evaluates them exactly instead: one CTA per matrix reads X = wide(M[K]) (pre-decay, fp32;
// launched after K2 and before K3's decay), accumulates A = X X^T in fp64, runs the whole
// polynomial recursion of Alg. 1 l.4 (readings R1-R5, R23's Gram-space algebra)
// on p x p fp64 matrices, and writes X_T = s Q X as fp16 into X1, where K7 reads it
// (MatDesc::final_in_x1 = 1).  The only rounding left is that final fp16 store.
#include "kernels.cuh"

namespace dion2 {

namespace {

constexpr int kP = kTinyP;      // max rows
constexpr int kLd = kP + 1;     // padded smem row of the p x p matrices
constexpr int kChunk = 64;      // X columns per pass chunk
constexpr int kThreads = 256;

// element (i, j) of the wide X = S (rows mode) or S^T (cols mode; M transposed or not)
__device__ __forceinline__ float x_at(const MatDesc& md, int i, int64_t j) {
  const int64_t r = md.sel[i];
  if (!md.transposed) return md.M[r * md.ld + j];
  if (md.mt) return md.M[r * md.ldm + j];
  return md.M[j * md.ld + r];
}

// C = A B for p x p row-major smem matrices (ld kLd), all threads
__device__ __forceinline__ void mm(double* C, const double* A, const double* B, int p) {
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int i = e / p, k = e % p;
    double acc = 0.0;
    for (int l = 0; l < p; ++l) acc += A[i * kLd + l] * B[l * kLd + k];
    C[i * kLd + k] = acc;
  }
}

}  // namespace

constexpr size_t kSmem = 4 * sizeof(double) * kP * kLd + sizeof(float) * kP * (kChunk + 1);

__global__ void __launch_bounds__(kThreads) k_ns_small(const MatDesc* __restrict__ mats, const int32_t* __restrict__ list,
                                                       int n_list, const int32_t* __restrict__ bad, NsSmallCoeffs C) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  double* A = reinterpret_cast<double*>(smem_raw);
  double* B = A + kP * kLd;
  double* Cm = B + kP * kLd;
  double* Q = Cm + kP * kLd;
  float (*xs)[kChunk + 1] = reinterpret_cast<float (*)[kChunk + 1]>(Q + kP * kLd);
  __shared__ double red;
  const int mi = list[blockIdx.x];
  const MatDesc& md = mats[mi];
  if (bad[mi]) return;  // block-uniform: K7 skips the matrix too
  const int p = md.p;
  const int64_t q = md.q;
  // ---- A = X X^T (upper triangle accumulated per thread over all column chunks)
  constexpr int kMaxPairs = kP * (kP + 1) / 2;
  double acc[(kMaxPairs + kThreads - 1) / kThreads] = {};
  const int npairs = p * (p + 1) / 2;
  for (int64_t j0 = 0; j0 < q; j0 += kChunk) {
    const int w = (int)(q - j0 < kChunk ? q - j0 : kChunk);
    for (int e = threadIdx.x; e < p * kChunk; e += blockDim.x) {
      const int i = e / kChunk, jj = e % kChunk;
      xs[i][jj] = jj < w ? x_at(md, i, j0 + jj) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < (kMaxPairs + kThreads - 1) / kThreads; ++s) {
      const int pr = threadIdx.x + s * kThreads;
      if (pr < npairs) {
        int i = 0, r = pr;
        while (r >= p - i) { r -= p - i; ++i; }
        const int k = i + r;
        // fp32 products within a 64-column chunk, fp64 across chunks: ~2^-24 relative, far below
        // the final fp16 store
        float a = 0.f;
        for (int jj = 0; jj < w; ++jj) a = fmaf(xs[i][jj], xs[k][jj], a);
        acc[s] += (double)a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int s = 0; s < (kMaxPairs + kThreads - 1) / kThreads; ++s) {
    const int pr = threadIdx.x + s * kThreads;
    if (pr < npairs) {
      int i = 0, r = pr;
      while (r >= p - i) { r -= p - i; ++i; }
      const int k = i + r;
      A[i * kLd + k] = acc[s];
      A[k * kLd + i] = acc[s];
    }
  }
  __syncthreads();
  // ---- s = 1 / (||X||_F + eps) (reading R3), A <- s^2 A, Q <- I
  if (threadIdx.x == 0) {
    double tr = 0.0;
    for (int i = 0; i < p; ++i) tr += A[i * kLd + i];
    red = 1.0 / (sqrt(tr) + (double)C.eps);
  }
  __syncthreads();
  const double sc = red;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int i = e / p, k = e % p;
    A[i * kLd + k] *= sc * sc;
    Q[i * kLd + k] = i == k ? 1.0 : 0.0;
  }
  __syncthreads();
  // ---- per iteration: C = aI + bA + cA^2, Q <- C Q, A <- C (C A)   (X_{t+1} = C_t X_t)
  for (int t = 0; t < C.T; ++t) {
    const double a = C.c[t][0], b = C.c[t][1], c = C.c[t][2];
    mm(B, A, A, p);
    __syncthreads();
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
      const int i = e / p, k = e % p;
      Cm[i * kLd + k] = (i == k ? a : 0.0) + b * A[i * kLd + k] + c * B[i * kLd + k];
    }
    __syncthreads();
    mm(B, Cm, Q, p);
    __syncthreads();
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) Q[(e / p) * kLd + e % p] = B[(e / p) * kLd + e % p];
    __syncthreads();
    if (t + 1 < C.T) {
      mm(B, Cm, A, p);
      __syncthreads();
      mm(A, Cm, B, p);
      __syncthreads();
    }
  }
  // ---- X_T = s Q X -> fp16 into X1 (row i, column j at i * q_pad + j)
  __half* out = reinterpret_cast<__half*>(md.X1);
  for (int64_t j0 = 0; j0 < q; j0 += kChunk) {
    const int w = (int)(q - j0 < kChunk ? q - j0 : kChunk);
    for (int e = threadIdx.x; e < p * kChunk; e += blockDim.x) {
      const int i = e / kChunk, jj = e % kChunk;
      xs[i][jj] = jj < w ? x_at(md, i, j0 + jj) : 0.f;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < p * w; e += blockDim.x) {
      const int i = e / w, jj = e % w;
      double o = 0.0;
      for (int l = 0; l < p; ++l) o += Q[i * kLd + l] * (double)xs[l][jj];
      out[(int64_t)i * md.q_pad + j0 + jj] = __float2half_rn((float)(sc * o));
    }
    __syncthreads();
  }
}

void launch_ns_small(cudaStream_t s, const MatDesc* mats, const int32_t* list, int n_list, const int32_t* bad,
                     const NsSmallCoeffs& C) {
  static const bool attr = cudaFuncSetAttribute(k_ns_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)kSmem) == cudaSuccess;
  (void)attr;
  if (n_list > 0) k_ns_small<<<n_list, kThreads, kSmem, s>>>(mats, list, n_list, bad, C);
}

}  // namespace dion2
