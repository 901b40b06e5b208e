// K3 rows path, TMA-staged (Alg. 1 l.4-5): X row r = fp16(xs * M[sel[r], :]) (xs: reading R24)
// (rows mode; with transposed momentum the row sel[r] of M^T), M[sel[r], :] <- mu * M[sel[r], :],
// per-row sum of squares for ||X||_F.  Same semantics, unit list and outputs as
// k_gather_rows (k_gather_scatter_fast.cu); the data moves through the bulk-copy (TMA) engine:
//
//   warp 0 (one lane)   cp.async.bulk global -> shared of 8 KB row chunks into an S-stage ring
//                       (mbarrier complete_tx), S - 1 chunks ahead of the consumers
//   warps 1..4          decay + convert in shared memory; one elected thread then issues
//                       cp.async.bulk shared -> global stores of the decayed M chunk and the
//                       fp16 X chunk, and releases the stage once the stores have read it
//
// so the loads in flight per SM are bounded by shared memory, not by registers.  Requires
// 16-byte aligned rows with a multiple of 8 elements (vec4 and n % 8 == 0); the launcher
// falls back to k_gather_rows otherwise.
#include <algorithm>

#include "kernels.cuh"

namespace dion2 {

namespace {

constexpr int kCh = 2048;            // fp32 elements per chunk (8 KB)
constexpr int kConsumers = 128;      // 4 consumer warps
constexpr int kThreads = 32 + kConsumers;

__device__ __forceinline__ int find_unit_tma(const int32_t* __restrict__ prefix, int n, int t) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void bulk_load(void* smem_dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(smem_src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory"); }

struct RowUnit {
  const MatDesc* md;
  int r, n, nch, mi;
  const float* mrow;  // valid for r < k
};

__device__ __forceinline__ RowUnit row_unit(const MatDesc* __restrict__ mats, const int32_t* __restrict__ lm,
                                            const int32_t* __restrict__ lp, int nl, int u) {
  RowUnit w;
  const int li = find_unit_tma(lp, nl, u);
  w.mi = lm[li];
  w.md = &mats[w.mi];
  w.r = u - lp[li];
  w.n = (int)(w.md->mt ? w.md->rows : w.md->cols);
  w.nch = (w.n + kCh - 1) / kCh;
  w.mrow = w.r < w.md->k ? w.md->M + (int64_t)w.md->sel[w.r] * (w.md->mt ? w.md->ldm : w.md->ld) : nullptr;
  return w;
}

}  // namespace

template <int S>
__global__ void __launch_bounds__(kThreads) k_gather_rows_tma(const MatDesc* __restrict__ mats,
                                                              const int32_t* __restrict__ lm,
                                                              const int32_t* __restrict__ lp, int nl, int total_units,
                                                              const int32_t* __restrict__ bad, float mu) {
  extern __shared__ __align__(128) uint8_t sm[];
  float* sm_m = reinterpret_cast<float*>(sm);                                    // [S][kCh]
  __half* sm_x = reinterpret_cast<__half*>(sm + S * kCh * 4);                    // [S][kCh]
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * kCh * 6);
  uint64_t* empty = full + S;
  __shared__ float red[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- producer
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
        const RowUnit w = row_unit(mats, lm, lp, nl, u);
        const int nch = w.r < w.md->k ? w.nch : 1;  // zero rows: one empty item
        for (int c = 0; c < nch; ++c) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (w.mrow) {
            const uint32_t bytes = (uint32_t)min(kCh, w.n - c * kCh) * 4;
            mbar_arrive_expect_tx(&full[stage], bytes);
            bulk_load(sm_m + stage * kCh, w.mrow + (int64_t)c * kCh, bytes, &full[stage]);
          } else {
            mbar_arrive(&full[stage]);
          }
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
    return;
  }
  // ---------------- consumers (128 threads)
  const int ct = threadIdx.x - 32, cw = warp - 1;
  int stage = 0;
  uint32_t phase = 0;
  int pending = -1;  // stage whose bulk stores are the most recent committed group (elected thread)
  for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
    const RowUnit w = row_unit(mats, lm, lp, nl, u);
    const MatDesc& md = *w.md;
    __half* xrow = reinterpret_cast<__half*>(md.X0) + (int64_t)w.r * md.q_pad;
    if (!w.mrow) {
      // X row r >= k: zeros (q_pad % 256 == 0: whole 16-B chunks), no M traffic
      mbar_wait(&full[stage], phase);
      uint4* x16 = reinterpret_cast<uint4*>(xrow);
      for (int c = ct; c < md.q_pad / 8; c += kConsumers) x16[c] = make_uint4(0, 0, 0, 0);
      consumer_sync();
      if (ct == 0) {
        md.sumsq_partials[w.r] = 0.f;
        if (pending >= 0) {  // release the held stage too: runs of zero rows must not starve the producer
          bulk_wait_read<0>();
          mbar_arrive(&empty[pending]);
          pending = -1;
        }
        mbar_arrive(&empty[stage]);
      }
      if (++stage == S) { stage = 0; phase ^= 1; }
      continue;
    }
    const float f = bad[w.mi] ? 1.f : mu;
    const float xs = md.ns_scale[2];  // fp16 prescale (K2, reading R24)
    float ss = 0.f;
    for (int c = 0; c < w.nch; ++c) {
      mbar_wait(&full[stage], phase);
      const int len = min(kCh, w.n - c * kCh);
      float4* m4 = reinterpret_cast<float4*>(sm_m + stage * kCh);
      uint2* x4 = reinterpret_cast<uint2*>(sm_x + stage * kCh);
#pragma unroll 4
      for (int j = ct; j < len / 4; j += kConsumers) {
        const float4 v = m4[j];
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
        x4[j] = pack4_h(xs * v.x, xs * v.y, xs * v.z, xs * v.w);
        m4[j] = make_float4(f * v.x, f * v.y, f * v.z, f * v.w);
      }
      fence_proxy_async_smem();  // the shared writes are visible to the bulk-copy engine
      consumer_sync();
      if (ct == 0) {
        bulk_store(const_cast<float*>(w.mrow) + (int64_t)c * kCh, sm_m + stage * kCh, (uint32_t)len * 4);
        bulk_store(xrow + (int64_t)c * kCh, sm_x + stage * kCh, (uint32_t)len * 2);
        bulk_commit();
        if (pending >= 0) {
          bulk_wait_read<1>();  // the previous stage's stores have read their shared data
          mbar_arrive(&empty[pending]);
        }
        pending = stage;
      }
      if (++stage == S) { stage = 0; phase ^= 1; }
    }
    // zero padding of X columns [n, q_pad) and the row's sum of squares (fixed order)
    for (int c = w.n + ct * 8; c < md.q_pad; c += kConsumers * 8)
      *reinterpret_cast<uint4*>(xrow + c) = make_uint4(0, 0, 0, 0);
    ss = warp_sum(ss);
    if (lane == 0) red[cw] = ss;
    consumer_sync();
    if (ct == 0) md.sumsq_partials[w.r] = (red[0] + red[1]) + (red[2] + red[3]);
    consumer_sync();  // red[] is rewritten by the next row
  }
  if (ct == 0) {
    bulk_wait_all();  // global writes of the last stores complete before the kernel ends
    if (pending >= 0) mbar_arrive(&empty[pending]);
  }
}

template <int S>
constexpr size_t gather_tma_smem() { return (size_t)S * kCh * 6 + 2 * S * 8; }

void launch_gather_rows_tma(int stages, int blocks_per_sm_cap, cudaStream_t s, const MatDesc* mats, const int32_t* lm,
                            const int32_t* lp, int nl, int units, const int32_t* bad, float mu, int sms) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gather_rows_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gather_tma_smem<4>());
    cudaFuncSetAttribute(k_gather_rows_tma<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gather_tma_smem<6>());
    cudaFuncSetAttribute(k_gather_rows_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gather_tma_smem<8>());
    attr = true;
  }
  int nb = 0;
  if (stages == 8) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_gather_rows_tma<8>, kThreads, gather_tma_smem<8>());
    nb = std::max(1, std::min(nb, blocks_per_sm_cap));
    k_gather_rows_tma<8><<<std::max(1, std::min(units, nb * sms)), kThreads, gather_tma_smem<8>(), s>>>(
        mats, lm, lp, nl, units, bad, mu);
  } else if (stages == 6) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_gather_rows_tma<6>, kThreads, gather_tma_smem<6>());
    nb = std::max(1, std::min(nb, blocks_per_sm_cap));
    k_gather_rows_tma<6><<<std::max(1, std::min(units, nb * sms)), kThreads, gather_tma_smem<6>(), s>>>(
        mats, lm, lp, nl, units, bad, mu);
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_gather_rows_tma<4>, kThreads, gather_tma_smem<4>());
    nb = std::max(1, std::min(nb, blocks_per_sm_cap));
    k_gather_rows_tma<4><<<std::max(1, std::min(units, nb * sms)), kThreads, gather_tma_smem<4>(), s>>>(
        mats, lm, lp, nl, units, bad, mu);
  }
}

}  // namespace dion2
