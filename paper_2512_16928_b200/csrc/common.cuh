// common.cuh -- device-side types and PTX helpers shared by the Dion2 kernels.
// sm_100a only (tcgen05 / TMA / mbarrier).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dion2 {

constexpr int kAxisRows = 0;
constexpr int kAxisCols = 1;

// Per-matrix device descriptor (built by the host plan, dion2_api.cu).
// S is the selected submatrix: S = M[K, :] (rows mode, sr = k, sc = n) or
// S = M[:, K] (cols mode, sr = m, sc = k).  X is its wide orientation
// (p <= q): X = S, or X = S^T when `transposed` (reading R4).
struct MatDesc {
  float* W;             // fp32, or bf16 under dion2_config.w_dtype = DION2_DT_BF16 (the K7 kernels cast)
  float* M;
  const void* G;
  int32_t* sel_out;
  float* O_out;
  int64_t rows, cols, ld;
  int32_t axis;        // resolved: kAxisRows / kAxisCols
  int32_t d, o, k;     // selection axis length, other axis length, selected count
  int32_t sr, sc;      // S dims
  int32_t transposed;  // X = S^T
  int32_t p, q;        // X dims (p <= q)
  int32_t p_pad, q_pad;
  int32_t vec4;        // 16-B aligned rows: float4 (and bf16x8 for bf16 G) loads allowed
  int32_t grad_bf16;
  float update_scale;  // sqrt(fan-out / fan-in) (times eta at launch)
  // workspace slices
  float* scores;          // [d]
  float* col_partials;    // [rowblocks][cols]  (cols mode)
  int32_t* sel;           // [k] ascending
  float* sumsq_partials;  // [n_gather_tiles]
  // [4] = { s', s'^2, xs, smax }: xs = 2^e, the power-of-two prescale K3 applies when it stores X as
  // fp16 (written by K2 from the largest l1 score, reading R24; 1 on the fp32 path), and
  // s' = s / xs with s = 1 / (||X||_F + eps) of the unscaled fp32 values (K3's sum of squares),
  // so s' * X0_stored = s * X exactly (powers of two); smax = the largest score (K2)
  float* ns_scale;
  void* X0;               // [p_pad x q_pad] fp16 (tensor-core path) or fp32: NS input / ping
  void* X1;               // pong
  int32_t final_in_x1;    // X_T lives in X1 (T odd)
  int32_t gather_tile_base, gather_tiles_a, gather_tiles_b;
  int32_t sa_pad, sb_pad;  // padded extents of S such that wide(S_pad) = X_pad (p_pad x q_pad)
  int32_t path;            // gather/scatter path: 0 generic tiles, 1 rows streaming, 2 cols streaming (X = S^T)
  int32_t n_sumsq;         // number of sum-of-squares partials K3 writes
  int32_t scores_final;    // select reads `scores` as final (distributed step: combined across ranks)
  int32_t mid;             // matrix id in the batch (random-selection key)
  int32_t mt;              // M stored transposed ([cols x ldm], cols mode only): K3 gathers rows of M^T
  int32_t spath;           // scatter path when it differs from `path` (single-GPU plans: 2 = cols streaming
                           // for k > kMaxColKFast); the generic K7 tiles skip matrices with spath != 0
  int64_t ldm;             // row stride of the transposed M
  int32_t rowblocks;      // ceil(rows / kColRowBlock) (cols mode partials)
  int32_t x16;            // X is stored as fp16 with the prescale xs (tensor-core path); 0: fp32, xs = 1
};

// ----------------------------------------------------------------------------- small helpers

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float bf16_to_f(__nv_bfloat16 x) { return __bfloat162float(x); }

// X / O storage of the tensor-core path: fp16 (10-bit mantissa; reading R24).  K3 stores
// X * xs (xs = 2^e, exact) so the largest entry sits near 2^15; O (|o| <= ~1.2) is unscaled.
__device__ __forceinline__ uint2 pack4_h(float a, float b, float c, float d) {
  __half2 lo = __floats2half2_rn(a, b), hi = __floats2half2_rn(c, d);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&lo);
  u.y = *reinterpret_cast<uint32_t*>(&hi);
  return u;
}
// Reading R24: the power-of-two prescale of the fp16 X.  Every entry of X lies in a selected
// row (column) of M, whose l1 norm bounds it, so max|x| <= smax and x * 2^e with
// e = 15 - exponent(smax) stays below 2^15 (fp16 max 65504); e is clamped to [-100, 64]
// (all-zero input: e = 0).
__device__ __forceinline__ float x16_prescale(float smax) {
  if (!(smax > 0.f)) return 1.f;
  int E;
  frexpf(smax, &E);  // smax = m 2^E, m in [0.5, 1)
  const int e = max(-100, min(64, 15 - E));
  return ldexpf(1.f, e);
}

// W element access of the sparse update (K7): fp32 W, or bf16 W (f4 "bf16 W variant": the update
// is computed in fp32 and rounded to nearest once, w <- bf16(float(w) - sc o)).
__device__ __forceinline__ float ld_w(const float* p) { return *p; }
__device__ __forceinline__ float ld_w(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void st_w(float* p, float v) { *p = v; }
__device__ __forceinline__ void st_w(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
// 4 consecutive elements j*4 .. j*4+3 (16-B aligned fp32 / 8-B aligned bf16 rows)
__device__ __forceinline__ float4 ld_w4(const float* row, int j) { return reinterpret_cast<const float4*>(row)[j]; }
__device__ __forceinline__ float4 ld_w4(const __nv_bfloat16* row, int j) {
  const uint2 u = reinterpret_cast<const uint2*>(row)[j];
  const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
  const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
  return make_float4(__low2float(lo), __high2float(lo), __low2float(hi), __high2float(hi));
}
__device__ __forceinline__ void st_w4(float* row, int j, float4 v) { reinterpret_cast<float4*>(row)[j] = v; }
__device__ __forceinline__ void st_w4(__nv_bfloat16* row, int j, float4 v) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
  reinterpret_cast<uint2*>(row)[j] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
}

__device__ __forceinline__ uint32_t pack2_h(float a, float b) {
  __half2 v = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Philox-4x32-10 (Salmon et al., SC'11), word 0 of the output block: the key of
// index i for random selection (counter = (i, step_lo, step_hi, matrix), key = seed).
__device__ __forceinline__ uint32_t philox_word0(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                                 uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return c0;
}

// Programmatic dependent launch (the NS kernels are launched with the programmatic stream
// serialization attribute): a kernel may start its prologue (barriers, TMEM, tensor-map
// prefetch) while the previous launch drains, and waits here before touching global memory.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void set_status_bad(int32_t* status, int mat) {
  atomicOr(&status[0], 1);
  atomicMin(&status[1], mat);
}

// ----------------------------------------------------------------------------- mbarrier

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Watchdog: a barrier that never completes (a pipeline bug) traps after ~4 s
// of spinning instead of hanging the GPU.
#ifndef DION2_WATCHDOG_CYCLES
#define DION2_WATCHDOG_CYCLES (8ll << 30)
#endif
__device__ __forceinline__ uint32_t mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(done)
      : "r"(addr), "r"(parity)
      : "memory");
  return done;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(addr, parity)) {
    if (clock64() - t0 > DION2_WATCHDOG_CYCLES) __trap();
  }
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ----------------------------------------------------------------------------- TMA

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// L2 prefetch of a 3-D tensor box (no shared-memory destination, no completion tracking)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* smem_src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// explicit shared-space stores (generic stores through a uintptr-aligned smem pointer
// compile to ST.E, not STS)
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void sts16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}

// ----------------------------------------------------------------------------- tcgen05

// One lane of the (converged) warp: the MMA issuer runs as a whole warp with warp-uniform loop
// state, so the descriptors stay in uniform registers and only the issue is predicated (a
// lane-0-only issuer made the compiler wrap every tcgen05.mma in an R2UR / ELECT waterfall:
// ~30 instructions per MMA, ncu round 2).
__device__ __forceinline__ bool elect_one_sync() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor (tcgen05 "matrix descriptor"):
//  [0,14) start addr >> 4, [16,30) LBO >> 4, [32,46) SBO >> 4, [46,48) version = 1,
//  [49,52) base offset = 0, [52] lbo mode = 0, [61,64) layout: 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16, dense.
//  [4,6) c_format = 1 (F32), [7,10) a_format = 1 (BF16), [10,13) b_format = 1 (BF16),
//  [15] a_major (0 = K), [16] b_major (0 = K, 1 = MN), [17,23) N >> 3, [24,29) M >> 4.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N, int b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

// ----------------------------------------------------------------------------- CTA pair (cta_group::2)
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address -> the same offset in CTA `rank` of the cluster (shared::cluster window)
__device__ __forceinline__ uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// Relaxed: used only to hand TMEM back to the leader's MMA (the tcgen05.ld's are complete
// after tcgen05.wait::ld + tcgen05.fence::before_thread_sync); .release here emitted a
// MEMBAR.ALL.CTA that stalled the epilogue behind its own TMA stores (ncu: 25% of samples).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA load into the local CTA's smem, completion counted on the pair leader's barrier
__device__ __forceinline__ void tma_load_3d_pair(void* smem_dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                 int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_ss_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                  uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrive on the barrier at this smem offset in both CTAs of the pair when the MMAs complete
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

// 32 lanes x 32 consecutive fp32 columns: thread t of the warp gets lane (base_lane + t).
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace dion2
