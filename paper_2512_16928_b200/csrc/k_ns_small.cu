// Newton-Schulz of short X (p <= kTinyP = 128 rows) in Gram space, straight from the momentum.
//
// The 16-bit tensor-core path rounds X once per entry (fp16, 2^-11 relative).  On an X of few
// rows whose spectrum is dominated by one or a few directions (a selected submatrix of a spiked
// momentum), that rounding is a large fraction of the weak directions, and a short X has few
// directions to average it over: emulated and measured up to 2-3.6% on the cumulative update at
// p <= 30, 1.7-1.9% at p = 33..63 and ~1.5% up to p = 128 for sigma_1 / median ~ 250
// (reading R25).  Such matrices are cheap, so AUTO evaluates them in high
// precision instead: one CTA per matrix reads X = wide(M[K]) (pre-decay, fp32; launched after
// K2 and before K3's decay), accumulates A = X X^T (fp32 products per 32/64-column chunk, fp64
// across chunks), runs the whole polynomial recursion of Alg. 1 l.4 (readings
// R1-R5, R23's Gram-space algebra) on p x p matrices -- in fp64 for p <= 64, in fp32 for
// p <= 128 (shared memory) -- and writes X_T = s Q X as fp16 into X1, where K7 reads it
// (MatDesc::final_in_x1 = 1).  Products are staged through registers, so three p x p buffers
// (A, C, Q) suffice.
#include <algorithm>

#include "kernels.cuh"

namespace dion2 {

namespace {

constexpr int kThreads = 256;

// element (i, j) of the wide X = S (rows mode) or S^T (cols mode; M transposed or not)
__device__ __forceinline__ float x_at(const MatDesc& md, int i, int64_t j) {
  const int64_t r = md.sel[i];
  if (!md.transposed) return md.M[r * md.ld + j];
  if (md.mt) return md.M[r * md.ldm + j];
  return md.M[j * md.ld + r];
}

template <int P, typename R>
struct Small {
  static constexpr int kLd = P + 1;
  static constexpr int kChunk = P <= 64 ? 64 : 32;
  static constexpr int kOut = (P * P + kThreads - 1) / kThreads;  // outputs per thread of a p x p product
  static constexpr size_t kSmem = 3 * sizeof(R) * P * kLd + sizeof(float) * P * (kChunk + 1);
};

// D = X Y (p x p, row-major smem, ld P + 1), staged through registers: D may alias X or Y
template <int P, typename R>
__device__ __forceinline__ void mm_inplace(R* D, const R* X, const R* Y, int p) {
  constexpr int kLd = Small<P, R>::kLd;
  R v[Small<P, R>::kOut];
#pragma unroll
  for (int s = 0; s < Small<P, R>::kOut; ++s) {
    const int e = threadIdx.x + s * kThreads;
    R acc = 0;
    if (e < p * p) {
      const int i = e / p, k = e % p;
      for (int l = 0; l < p; ++l) acc += X[i * kLd + l] * Y[l * kLd + k];
    }
    v[s] = acc;
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < Small<P, R>::kOut; ++s) {
    const int e = threadIdx.x + s * kThreads;
    if (e < p * p) D[(e / p) * kLd + e % p] = v[s];
  }
  __syncthreads();
}

}  // namespace

template <int P, typename R>
__global__ void __launch_bounds__(kThreads) k_ns_small(const MatDesc* __restrict__ mats, const int32_t* __restrict__ list,
                                                       int n_list, const int32_t* __restrict__ bad, NsSmallCoeffs C) {
  using S = Small<P, R>;
  constexpr int kLd = S::kLd, kChunk = S::kChunk;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  R* A = reinterpret_cast<R*>(smem_raw);
  R* Cm = A + P * kLd;
  R* Q = Cm + P * kLd;
  float (*xs)[kChunk + 1] = reinterpret_cast<float (*)[kChunk + 1]>(Q + P * kLd);
  __shared__ double red;
  const int mi = list[blockIdx.x];
  const MatDesc& md = mats[mi];
  if (bad[mi]) return;  // block-uniform: K7 skips the matrix too
  const int p = md.p;
  const int64_t q = md.q;
  // ---- A = X X^T (upper triangle accumulated per thread over all column chunks)
  constexpr int kMaxPairs = P * (P + 1) / 2;
  constexpr int kPairsPer = (kMaxPairs + kThreads - 1) / kThreads;
  double acc[kPairsPer];
#pragma unroll
  for (int s = 0; s < kPairsPer; ++s) acc[s] = 0.0;
  const int npairs = p * (p + 1) / 2;
  for (int64_t j0 = 0; j0 < q; j0 += kChunk) {
    const int w = (int)(q - j0 < kChunk ? q - j0 : kChunk);
    for (int e = threadIdx.x; e < p * kChunk; e += blockDim.x) {
      const int i = e / kChunk, jj = e % kChunk;
      xs[i][jj] = jj < w ? x_at(md, i, j0 + jj) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kPairsPer; ++s) {
      const int pr = threadIdx.x + s * kThreads;
      if (pr < npairs) {
        int i = 0, r = pr;
        while (r >= p - i) { r -= p - i; ++i; }
        const int k = i + r;
        // fp32 products within a chunk, fp64 across chunks (~2^-24 relative, far below the
        // final fp16 store)
        float a = 0.f;
        for (int jj = 0; jj < w; ++jj) a = fmaf(xs[i][jj], xs[k][jj], a);
        acc[s] += (double)a;
      }
    }
    __syncthreads();
  }
  // ---- s = 1 / (||X||_F + eps) (reading R3) from the fp64 trace; A <- s^2 A; Q <- I
  if (threadIdx.x == 0) red = 0.0;
  __syncthreads();
#pragma unroll
  for (int s = 0; s < kPairsPer; ++s) {
    const int pr = threadIdx.x + s * kThreads;
    if (pr < npairs) {
      int i = 0, r = pr;
      while (r >= p - i) { r -= p - i; ++i; }
      if (r == 0) atomicAdd(&red, acc[s]);  // a diagonal entry
    }
  }
  __syncthreads();
  const double sc = 1.0 / (sqrt(red) + (double)C.eps);
#pragma unroll
  for (int s = 0; s < kPairsPer; ++s) {
    const int pr = threadIdx.x + s * kThreads;
    if (pr < npairs) {
      int i = 0, r = pr;
      while (r >= p - i) { r -= p - i; ++i; }
      const int k = i + r;
      const R v = (R)(acc[s] * sc * sc);
      A[i * kLd + k] = v;
      A[k * kLd + i] = v;
    }
  }
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) Q[(e / p) * kLd + e % p] = (e / p == e % p) ? R(1) : R(0);
  __syncthreads();
  // ---- per iteration: C = aI + bA + cA^2, Q <- C Q, A <- C (C A)   (X_{t+1} = C_t X_t)
  for (int t = 0; t < C.T; ++t) {
    const R a = C.c[t][0], b = C.c[t][1], c = C.c[t][2];
    mm_inplace<P, R>(Cm, A, A, p);  // Cm = A^2
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
      const int i = e / p, k = e % p;
      Cm[i * kLd + k] = (i == k ? a : R(0)) + b * A[i * kLd + k] + c * Cm[i * kLd + k];
    }
    __syncthreads();
    mm_inplace<P, R>(Q, Cm, Q, p);
    if (t + 1 < C.T) {
      mm_inplace<P, R>(A, Cm, A, p);
      mm_inplace<P, R>(A, Cm, A, p);
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
      for (int l = 0; l < p; ++l) o += (double)Q[i * kLd + l] * (double)xs[l][jj];
      out[(int64_t)i * md.q_pad + j0 + jj] = __float2half_rn((float)(sc * o));
    }
    __syncthreads();
  }
}

void launch_ns_small(cudaStream_t s, const MatDesc* mats, const int32_t* list, int n_list, const int32_t* bad,
                     const NsSmallCoeffs& C, bool wide) {
  if (n_list <= 0) return;
  if (!wide) {
    using S = Small<64, double>;
    static const bool attr = cudaFuncSetAttribute(k_ns_small<64, double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)S::kSmem) == cudaSuccess;
    (void)attr;
    k_ns_small<64, double><<<n_list, kThreads, S::kSmem, s>>>(mats, list, n_list, bad, C);
  } else {
    using S = Small<128, float>;
    static const bool attr = cudaFuncSetAttribute(k_ns_small<128, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)S::kSmem) == cudaSuccess;
    (void)attr;
    k_ns_small<128, float><<<n_list, kThreads, S::kSmem, s>>>(mats, list, n_list, bad, C);
  }
}

}  // namespace dion2

// ---------------------------------------------------------------- distributed short X
// In the distributed step every rank holds a column block X_r of a short X (its shard of the
// selected rows / columns), and A = X X^T = sum_r X_r X_r^T.  Each rank writes its partial
// Gram matrix (fp64, p x p at Abase + idx * kTinyP^2); the step all-reduces them; each rank then
// runs the recursion on the summed A and applies s Q to its own X_r (no pieces are exchanged).
namespace dion2 {

template <int P>
__global__ void __launch_bounds__(kThreads) k_ns_small_partial(const MatDesc* __restrict__ mats,
                                                               const int32_t* __restrict__ list, int n_list,
                                                               double* __restrict__ Abase) {
  constexpr int kChunk = Small<P, float>::kChunk;
  __shared__ float xs[P][kChunk + 1];
  const int mi = list[blockIdx.x];
  const MatDesc& md = mats[mi];
  const int p = md.p;
  const int64_t q = md.q;  // this rank's columns of X
  double* Aout = Abase + (int64_t)blockIdx.x * kTinyP * kTinyP;
  constexpr int kMaxPairs = P * (P + 1) / 2;
  constexpr int kPairsPer = (kMaxPairs + kThreads - 1) / kThreads;
  double acc[kPairsPer];
#pragma unroll
  for (int s = 0; s < kPairsPer; ++s) acc[s] = 0.0;
  const int npairs = p * (p + 1) / 2;
  for (int64_t j0 = 0; j0 < q; j0 += kChunk) {
    const int w = (int)(q - j0 < kChunk ? q - j0 : kChunk);
    for (int e = threadIdx.x; e < p * kChunk; e += blockDim.x) {
      const int i = e / kChunk, jj = e % kChunk;
      xs[i][jj] = jj < w ? x_at(md, i, j0 + jj) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kPairsPer; ++s) {
      const int pr = threadIdx.x + s * kThreads;
      if (pr < npairs) {
        int i = 0, r = pr;
        while (r >= p - i) { r -= p - i; ++i; }
        const int k = i + r;
        float a = 0.f;
        for (int jj = 0; jj < w; ++jj) a = fmaf(xs[i][jj], xs[k][jj], a);
        acc[s] += (double)a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int s = 0; s < kPairsPer; ++s) {
    const int pr = threadIdx.x + s * kThreads;
    if (pr < npairs) {
      int i = 0, r = pr;
      while (r >= p - i) { r -= p - i; ++i; }
      const int k = i + r;
      Aout[i * kTinyP + k] = acc[s];
      Aout[k * kTinyP + i] = acc[s];
    }
  }
}

template <int P, typename R>
__global__ void __launch_bounds__(kThreads) k_ns_small_finish(const MatDesc* __restrict__ mats,
                                                              const int32_t* __restrict__ list, int n_list,
                                                              const int32_t* __restrict__ bad,
                                                              const double* __restrict__ Abase, NsSmallCoeffs C) {
  using S = Small<P, R>;
  constexpr int kLd = S::kLd, kChunk = S::kChunk;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  R* A = reinterpret_cast<R*>(smem_raw);
  R* Cm = A + P * kLd;
  R* Q = Cm + P * kLd;
  float (*xs)[kChunk + 1] = reinterpret_cast<float (*)[kChunk + 1]>(Q + P * kLd);
  __shared__ double red;
  const int mi = list[blockIdx.x];
  const MatDesc& md = mats[mi];
  if (bad[mi]) return;
  const int p = md.p;
  const int64_t q = md.q;
  const double* Ain = Abase + (int64_t)blockIdx.x * kTinyP * kTinyP;
  if (threadIdx.x == 0) {
    double tr = 0.0;
    for (int i = 0; i < p; ++i) tr += Ain[i * kTinyP + i];
    red = 1.0 / (sqrt(tr) + (double)C.eps);
  }
  __syncthreads();
  const double sc = red;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int i = e / p, k = e % p;
    A[i * kLd + k] = (R)(Ain[i * kTinyP + k] * sc * sc);
    Q[i * kLd + k] = i == k ? R(1) : R(0);
  }
  __syncthreads();
  for (int t = 0; t < C.T; ++t) {
    const R a = C.c[t][0], b = C.c[t][1], c = C.c[t][2];
    mm_inplace<P, R>(Cm, A, A, p);
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
      const int i = e / p, k = e % p;
      Cm[i * kLd + k] = (i == k ? a : R(0)) + b * A[i * kLd + k] + c * Cm[i * kLd + k];
    }
    __syncthreads();
    mm_inplace<P, R>(Q, Cm, Q, p);
    if (t + 1 < C.T) {
      mm_inplace<P, R>(A, Cm, A, p);
      mm_inplace<P, R>(A, Cm, A, p);
    }
  }
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
      for (int l = 0; l < p; ++l) o += (double)Q[i * kLd + l] * (double)xs[l][jj];
      out[(int64_t)i * md.q_pad + j0 + jj] = __float2half_rn((float)(sc * o));
    }
    __syncthreads();
  }
}

__global__ void k_add_f64(double* __restrict__ dst, const double* __restrict__ src, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

void launch_ns_small_partial(cudaStream_t s, const MatDesc* mats, const int32_t* list, int n_list, double* Abase,
                             bool wide) {
  if (n_list <= 0) return;
  if (!wide)
    k_ns_small_partial<64><<<n_list, kThreads, 0, s>>>(mats, list, n_list, Abase);
  else
    k_ns_small_partial<128><<<n_list, kThreads, 0, s>>>(mats, list, n_list, Abase);
}

void launch_ns_small_finish(cudaStream_t s, const MatDesc* mats, const int32_t* list, int n_list, const int32_t* bad,
                            const double* Abase, const NsSmallCoeffs& C, bool wide) {
  if (n_list <= 0) return;
  if (!wide) {
    using S = Small<64, double>;
    static const bool attr = cudaFuncSetAttribute(k_ns_small_finish<64, double>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::kSmem) == cudaSuccess;
    (void)attr;
    k_ns_small_finish<64, double><<<n_list, kThreads, S::kSmem, s>>>(mats, list, n_list, bad, Abase, C);
  } else {
    using S = Small<128, float>;
    static const bool attr = cudaFuncSetAttribute(k_ns_small_finish<128, float>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::kSmem) == cudaSuccess;
    (void)attr;
    k_ns_small_finish<128, float><<<n_list, kThreads, S::kSmem, s>>>(mats, list, n_list, bad, Abase, C);
  }
}

void launch_add_f64(cudaStream_t s, double* dst, const double* src, int64_t n) {
  if (n > 0) k_add_f64<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, s>>>(dst, src, n);
}

}  // namespace dion2
