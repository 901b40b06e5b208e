// K2: per-matrix top-k selection  K <- Select_alpha(M)  (Alg. 1 l.3).
// One CTA (kSelectThreads) per matrix; the selection itself is select_impl.cuh.
#include "kernels.cuh"
#include "select_impl.cuh"

namespace dion2 {

__global__ void __launch_bounds__(kSelectThreads) k_topk_select(const MatDesc* __restrict__ mats,
                                                                const int32_t* __restrict__ list,
                                                                int32_t* __restrict__ bad,
                                                                int32_t* __restrict__ status, int random_sel,
                                                                uint64_t seed, uint64_t step) {
  extern __shared__ uint32_t keys[];  // [d]
  __shared__ SelectSmem sh;
  const int mi = list ? list[blockIdx.x] : (int)blockIdx.x;
  select_matrix(mats[mi], mi, keys, sh, bad, status, random_sel, seed, step);
}

// block = 32 columns x 8 row-block groups: thread (g, c) sums the partials of row blocks
// g, g + 8, g + 16, ... of column c (4 loads in flight), then the 8 group sums are added
// in group order: a fixed order, deterministic run to run.
__global__ void __launch_bounds__(256) k_col_scores_finalize(const MatDesc* __restrict__ mats,
                                                             const int32_t* __restrict__ list,
                                                             const int64_t* __restrict__ prefix, int n_list,
                                                             int64_t total) {
  __shared__ float red[8][33];
  const int c = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t gc = (int64_t)blockIdx.x * 32 + c;
  const bool valid = gc < total;
  int li = 0;
  if (valid) {
    int lo = 0, hi = n_list - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (prefix[mid] <= gc) lo = mid; else hi = mid - 1;
    }
    li = lo;
  }
  const MatDesc& md = mats[list[li]];
  const int64_t j = gc - prefix[li];
  float s = 0.f;
  if (valid) {
    const float* col = md.col_partials + j;
    const int R = md.rowblocks;
    int rb = g;
    for (; rb + 24 < R; rb += 32) {
      const float a0 = __ldcg(col + (int64_t)rb * md.cols), a1 = __ldcg(col + (int64_t)(rb + 8) * md.cols);
      const float a2 = __ldcg(col + (int64_t)(rb + 16) * md.cols), a3 = __ldcg(col + (int64_t)(rb + 24) * md.cols);
      s += a0; s += a1; s += a2; s += a3;
    }
    for (; rb < R; rb += 8) s += __ldcg(col + (int64_t)rb * md.cols);
  }
  red[g][c] = s;
  __syncthreads();
  if (g == 0 && valid) {
    float t = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += red[q][c];
    md.scores[j] = t;
  }
}

}  // namespace dion2
