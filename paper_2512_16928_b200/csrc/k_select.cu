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

}  // namespace dion2
