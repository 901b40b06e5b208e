// Fused pre-stage for rows-mode matrices: K1 momentum + l1 score, K2 select and K3
// gather + selective decay in ONE persistent launch (Alg. 1 l.2-5).
//
// Why: the separate launches stream the whole model's M through HBM in K1, then re-read
// the selected rows M[K] and write mu*M[K] back in K3, long after they left L2.  Here a
// global ticket hands out tasks in an order that keeps each matrix's gather a few
// matrices behind its K1, so the selected rows of M are still in the 126 MB L2 when K3
// reads and decays them: the K3 read of M[K] and the second write-back of M[K] never
// reach HBM.  G is streamed with an L2 evict-first policy so it does not displace M.
//
// Tasks (host-built table, in ticket order; dependencies always point to EARLIER
// tickets, which are held by running CTAs, so the dynamic ticket cannot deadlock):
//   type 0  K1 of rows [u0, u1) of matrix mi (the whole CTA on one row at a time:
//           a small in-flight window, so a matrix's K1 completes soon after its last
//           task is handed out); +1 on k1_done[mi] when done
//   type 1  K2 select of matrix mi after k1_done[mi] == k1_need[mi]; sel_ready[mi] = 1
//   type 2  K3 gather of X rows [u0, u1) of matrix mi after sel_ready[mi] (warp per row)
// Cross-CTA data (scores, M rows, sel, bad) is read with ld.global.cg after an acquire
// by thread 0 and a CTA barrier; producers publish with barrier + __threadfence + atomic
// (the cooperative-groups grid-barrier pattern).
//
// Semantics are exactly those of k_momentum_score_rows + k_topk_select + k_gather_rows;
// the l1 score of a row is summed in a different (still fixed) order.
#include "kernels.cuh"
#include "select_impl.cuh"

namespace dion2 {

namespace {

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ float4 ld_g_f32x4(const float* p, uint64_t pol, bool hint) {
  float4 v;
  if (hint)
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
  else
    v = __ldg(reinterpret_cast<const float4*>(p));
  return v;
}

__device__ __forceinline__ float4 ld_g_bf16x4(const __nv_bfloat16* p, uint64_t pol, bool hint) {
  uint2 raw;
  if (hint)
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
                 : "=r"(raw.x), "=r"(raw.y)
                 : "l"(p), "l"(pol));
  else
    raw = __ldg(reinterpret_cast<const uint2*>(p));
  const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(&raw.x);
  const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&raw.y);
  return make_float4(__low2float(lo), __high2float(lo), __low2float(hi), __high2float(hi));
}

__device__ __forceinline__ void wait_geq(const int32_t* p, int32_t v) {
  int32_t x;
  const long long t0 = clock64();
  for (;;) {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(x) : "l"(p) : "memory");
    if (x >= v) return;
    __nanosleep(64);
    if (clock64() - t0 > DION2_WATCHDOG_CYCLES) __trap();
  }
}

__device__ __forceinline__ uint2 pack4_bf16_f(float a, float b, float c, float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&lo);
  u.y = *reinterpret_cast<uint32_t*>(&hi);
  return u;
}

// K1 of rows r and r + 1 (nr = 1 or 2) by the whole CTA: M <- M + G; the rows' l1 norms
// land in sc[0..nr).  Each half of the CTA (128 threads) streams one row with U float4 of
// M and of G per thread in flight, so a 2048-column row pair is one iteration and a task
// completes within a few microseconds.
template <bool kBf16G, bool kHint>
__device__ __forceinline__ void k1_rows_cta(const MatDesc& md, int64_t r, int nr, uint64_t pol, float* red,
                                            float* sc) {
  const int half = threadIdx.x >> 7, ht = threadIdx.x & 127;
  const int n = (int)md.cols;
  const int n4 = md.vec4 ? n >> 2 : 0;  // unaligned rows: the scalar loop takes the row
  float acc = 0.f;
  if (half < nr) {
    const int64_t ri = r + half;
    float4* __restrict__ M4 = reinterpret_cast<float4*>(md.M + ri * md.ld);
    constexpr int U = 4;
    int j = ht;
    for (; j + 128 * (U - 1) < n4; j += 128 * U) {
      float4 m[U], g[U];
#pragma unroll
      for (int u = 0; u < U; ++u) m[u] = __ldcg(M4 + j + 128 * u);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if constexpr (kBf16G)
          g[u] = ld_g_bf16x4(reinterpret_cast<const __nv_bfloat16*>(md.G) + ri * md.ld + 4 * (j + 128 * u), pol, kHint);
        else
          g[u] = ld_g_f32x4(reinterpret_cast<const float*>(md.G) + ri * md.ld + 4 * (j + 128 * u), pol, kHint);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        m[u].x += g[u].x; m[u].y += g[u].y; m[u].z += g[u].z; m[u].w += g[u].w;
        M4[j + 128 * u] = m[u];
        acc += fabsf(m[u].x) + fabsf(m[u].y) + fabsf(m[u].z) + fabsf(m[u].w);
      }
    }
    for (; j < n4; j += 128) {
      float4 m = __ldcg(M4 + j);
      float4 g;
      if constexpr (kBf16G)
        g = ld_g_bf16x4(reinterpret_cast<const __nv_bfloat16*>(md.G) + ri * md.ld + 4 * j, pol, kHint);
      else
        g = ld_g_f32x4(reinterpret_cast<const float*>(md.G) + ri * md.ld + 4 * j, pol, kHint);
      m.x += g.x; m.y += g.y; m.z += g.z; m.w += g.w;
      M4[j] = m;
      acc += fabsf(m.x) + fabsf(m.y) + fabsf(m.z) + fabsf(m.w);
    }
    float* Mrow = md.M + ri * md.ld;
    for (int t = 4 * n4 + ht; t < n; t += 128) {
      const float g = kBf16G ? bf16_to_f(reinterpret_cast<const __nv_bfloat16*>(md.G)[ri * md.ld + t])
                             : reinterpret_cast<const float*>(md.G)[ri * md.ld + t];
      const float v = __ldcg(Mrow + t) + g;
      Mrow[t] = v;
      acc += fabsf(v);
    }
  }
  acc = warp_sum(acc);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = acc;
  __syncthreads();
  if (threadIdx.x < 2) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) s += red[4 * threadIdx.x + w];  // fixed order: deterministic
    sc[threadIdx.x] = s;
  }
  __syncthreads();
}

// K3 of X row r (warp): rows mode, X = M[K, :] pre-decay; M[K] <- f * M[K]; sum of squares.
template <int D>
__device__ __forceinline__ void gather_row_warp(const MatDesc& md, int r, float f) {
  const int lane = threadIdx.x & 31;
  __nv_bfloat16* xrow = reinterpret_cast<__nv_bfloat16*>(md.X0) + (int64_t)r * md.q_pad;
  float ss = 0.f;
  if (r < md.k) {
    float* mrow = md.M + (int64_t)__ldcg(md.sel + r) * md.ld;
    const int n = (int)md.cols;
    const int n4 = md.vec4 ? n >> 2 : 0;
    float4* m4 = reinterpret_cast<float4*>(mrow);
    uint2* x4 = reinterpret_cast<uint2*>(xrow);
    int j = lane;
    for (; j + 32 * (D - 1) < n4; j += 32 * D) {
      float4 v[D];
#pragma unroll
      for (int q = 0; q < D; ++q) v[q] = __ldcg(m4 + j + 32 * q);
#pragma unroll
      for (int q = 0; q < D; ++q) {
        ss += v[q].x * v[q].x + v[q].y * v[q].y + v[q].z * v[q].z + v[q].w * v[q].w;
        x4[j + 32 * q] = pack4_bf16_f(v[q].x, v[q].y, v[q].z, v[q].w);
        m4[j + 32 * q] = make_float4(f * v[q].x, f * v[q].y, f * v[q].z, f * v[q].w);
      }
    }
    for (; j < n4; j += 32) {
      float4 v = __ldcg(m4 + j);
      ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      x4[j] = pack4_bf16_f(v.x, v.y, v.z, v.w);
      m4[j] = make_float4(f * v.x, f * v.y, f * v.z, f * v.w);
    }
    for (int c = 4 * n4 + lane; c < n; c += 32) {
      float v = __ldcg(mrow + c);
      ss += v * v;
      xrow[c] = __float2bfloat16_rn(v);
      mrow[c] = f * v;
    }
    for (int c = n + lane; c < md.q_pad; c += 32) xrow[c] = __float2bfloat16_rn(0.f);
  } else {
    uint4* x16 = reinterpret_cast<uint4*>(xrow);  // q_pad % 256 == 0: whole 16-B chunks
    for (int c = lane; c < md.q_pad / 8; c += 32) x16[c] = make_uint4(0, 0, 0, 0);
  }
  ss = warp_sum(ss);
  if (lane == 0) md.sumsq_partials[r] = ss;
}

}  // namespace

template <bool kHint>
__global__ void __launch_bounds__(256) k_pre_fused_rows(const MatDesc* __restrict__ mats,
                                                        const int4* __restrict__ tasks, int n_tasks,
                                                        int32_t* __restrict__ ctr, const int32_t* __restrict__ k1_need,
                                                        int n_mats, int32_t* __restrict__ bad,
                                                        int32_t* __restrict__ status, float mu, int random_sel,
                                                        uint64_t seed, uint64_t step) {
  extern __shared__ uint32_t keys[];  // [max d] select keys
  __shared__ SelectSmem sh;
  __shared__ float red[8];
  __shared__ float sc[2];
  __shared__ int s_next;
  int32_t* ticket = ctr;
  int32_t* k1_done = ctr + 1;
  int32_t* sel_ready = ctr + 1 + n_mats;
  const uint64_t pol = kHint ? policy_evict_first() : 0ull;

  if (threadIdx.x == 0) s_next = atomicAdd(ticket, 1);
  __syncthreads();
  int t = s_next;
  while (t < n_tasks) {
    // fetch the next ticket while this task runs (hides the atomic's round trip)
    int nxt = 0;
    if (threadIdx.x == 0) nxt = atomicAdd(ticket, 1);
    const int4 tk = tasks[t];
    const int mi = tk.y;
    const MatDesc& md = mats[mi];
    if (tk.x == 0) {
      for (int r = tk.z; r < tk.w; r += 2) {
        const int nr = min(2, tk.w - r);
        if (md.grad_bf16) k1_rows_cta<true, kHint>(md, r, nr, pol, red, sc);
        else k1_rows_cta<false, kHint>(md, r, nr, pol, red, sc);
        if (threadIdx.x < nr) md.scores[r + threadIdx.x] = sc[threadIdx.x];
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(k1_done + mi, 1);
      }
    } else if (tk.x == 1) {
      if (threadIdx.x == 0) wait_geq(k1_done + mi, k1_need[mi]);
      __syncthreads();
      select_matrix(md, mi, keys, sh, bad, status, random_sel, seed, step);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicExch(sel_ready + mi, 1);
      }
    } else {
      if (threadIdx.x == 0) wait_geq(sel_ready + mi, 1);
      __syncthreads();
      const float f = __ldcg(bad + mi) ? 1.f : mu;
      const int r = tk.z + (threadIdx.x >> 5);
      if (r < tk.w) gather_row_warp<8>(md, r, f);
    }
    if (threadIdx.x == 0) s_next = nxt;
    __syncthreads();
    t = s_next;
    __syncthreads();
  }
}

void launch_pre_fused_rows(bool hint, int blocks, size_t smem, cudaStream_t s, const MatDesc* mats,
                           const int4* tasks, int n_tasks, int32_t* ctr, const int32_t* k1_need, int n_mats,
                           int32_t* bad, int32_t* status, float mu, int random_sel, uint64_t seed, uint64_t step) {
  if (hint)
    k_pre_fused_rows<true><<<blocks, 256, smem, s>>>(mats, tasks, n_tasks, ctr, k1_need, n_mats, bad, status, mu,
                                                      random_sel, seed, step);
  else
    k_pre_fused_rows<false><<<blocks, 256, smem, s>>>(mats, tasks, n_tasks, ctr, k1_need, n_mats, bad, status, mu,
                                                       random_sel, seed, step);
}

int pre_fused_blocks_per_sm(bool hint, size_t smem) {
  int nb = 0;
  if (hint)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_pre_fused_rows<true>, 256, smem);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_pre_fused_rows<false>, 256, smem);
  return nb;
}

}  // namespace dion2
