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

__global__ void __launch_bounds__(256) k_col_scores_finalize(const MatDesc* __restrict__ mats,
                                                             const int32_t* __restrict__ list,
                                                             const int64_t* __restrict__ prefix, int n_list,
                                                             int64_t total) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= total) return;
  int lo = 0, hi = n_list - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= g) lo = mid; else hi = mid - 1;
  }
  const MatDesc& md = mats[list[lo]];
  const int64_t j = g - prefix[lo];
  float s = 0.f;
  for (int rb = 0; rb < md.rowblocks; ++rb) s += md.col_partials[(int64_t)rb * md.cols + j];
  md.scores[j] = s;
}

}  // namespace dion2
