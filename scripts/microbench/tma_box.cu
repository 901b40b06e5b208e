// Microbenchmark (diagnosis only, not part of the library): TMA streaming bandwidth of a
// row-major fp16 matrix [R][C] for the two tile walks of the Newton-Schulz kernels:
//   walk 0 ("gram", K-major):  boxes {64 cols, BR rows}, consecutive loads advance along the columns
//   walk 1 ("apply", MN-major): boxes {64 cols, BR rows}, consecutive loads advance along the rows
// Each CTA streams a disjoint set of (row block, column block) tiles through an S-stage ring;
// the consumer only releases stages.  Prints GB/s per configuration.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0,1,0,P;\n\t}" : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(su32(dst)), "l"((uint64_t)m), "r"(su32(bar)), "r"(c0), "r"(c1) : "memory");
}

template <int S>
__global__ void __launch_bounds__(64, 1) k_stream(const __grid_constant__ CUtensorMap map, int R, int C, int BR, int walk,
                                                 int tiles_per_cta, int box_bytes) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* ring = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(ring + S * box_bytes);
  uint64_t* empty = full + S;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nrb = R / BR, ncb = C / 64;
  // a CTA owns a contiguous run of `tiles_per_cta` tiles of the walk order
  const long long t0 = (long long)blockIdx.x * tiles_per_cta;
  if (threadIdx.x == 0) {
    int st = 0; uint32_t ph = 0;
    for (int i = 0; i < tiles_per_cta; ++i) {
      const long long t = t0 + i;
      int rb, cb;
      if (walk == 0) { rb = (int)((t / ncb) % nrb); cb = (int)(t % ncb); }   // along columns
      else { cb = (int)((t / nrb) % ncb); rb = (int)(t % nrb); }             // along rows
      mbar_wait(&empty[st], ph ^ 1);
      mbar_expect(&full[st], box_bytes);
      tma2d(ring + st * box_bytes, &map, &full[st], cb * 64, rb * BR);
      if (++st == S) { st = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int st = 0; uint32_t ph = 0;
    for (int i = 0; i < tiles_per_cta; ++i) {
      mbar_wait(&full[st], ph);
      mbar_arrive(&empty[st]);
      if (++st == S) { st = 0; ph ^= 1; }
    }
  }
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int R = 512 * 48, C = 8192;  // 48 matrices of 512 x 8192 fp16 stacked: 0.4 GB
  void* buf = nullptr;
  cudaMalloc(&buf, (size_t)R * C * 2);
  cudaMemset(buf, 0, (size_t)R * C * 2);
  for (int BR : {64, 128}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
    cuuint64_t str[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)BR};
    cuuint32_t es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int box_bytes = 64 * BR * 2;
    const long long tiles = (long long)(R / BR) * (C / 64);
    for (int walk : {0, 1}) {
      for (int ctas_per_sm : {1, 2}) {
        const int grid = sms * ctas_per_sm;
        const int per = (int)(tiles / grid);
        const int S = 8;
        const size_t smem = 1024 + S * box_bytes + 2 * S * 8;
        cudaFuncSetAttribute(k_stream<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        for (int w = 0; w < 2; ++w) k_stream<8><<<grid, 64, smem>>>(map, R, C, BR, walk, per, box_bytes);
        cudaEventRecord(a);
        const int it = 5;
        for (int w = 0; w < it; ++w) k_stream<8><<<grid, 64, smem>>>(map, R, C, BR, walk, per, box_bytes);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0; cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)per * grid * box_bytes;
        printf("box {64, %3d} walk %s ctas/sm %d stages %d in-flight/SM %6.0f KB: %7.1f GB/s\n", BR,
               walk ? "rows(apply)" : "cols(gram) ", ctas_per_sm, S, ctas_per_sm * S * box_bytes / 1024.0,
               bytes / (ms / it * 1e-3) / 1e9);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
