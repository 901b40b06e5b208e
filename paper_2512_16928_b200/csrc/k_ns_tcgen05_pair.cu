// K4-K6 on a CTA pair: tcgen05.mma.cta_group::2, 256 x 256 x 16 per instruction.
//
// Same three Newton-Schulz phases and epilogue algebra as k_ns_tcgen05.cu
// (gram A = s^2 X X^T; poly C = a I + b A + c A A^T; apply X' = s C X; PAPER.md
// P:65, Alg. 1 l.4, readings R1-R6), but each tile is computed by a cluster
// of two CTAs on one TPC: CTA r stages rows [128 r, 128 r + 128) of the A
// operand and half of the B operand, the leader CTA issues one 256 x 256 MMA
// that reads both CTAs' shared memory, and each CTA's TMEM receives its 128
// accumulator rows.  Per SM this halves the B-operand shared-memory traffic
// (TMA write + MMA read), which caps the 1-CTA 128 x 256 tile near 65-70% of
// peak (ncu: profiles/).
//
// Operand / output element type per launch: bf16 or fp16 (p.in_f16, p.out_f16; the
// Gram-space products of reading R23 run on fp16 with fp32 accumulation).
//
// Roles per CTA (320 threads): warp 0 TMA producer (both CTAs; completion is
// counted on the leader's full barrier), warp 1 TMEM allocator (both) + MMA
// issuer (leader only), warps 2-5 epilogue (both; TMEM -> bf16 -> swizzled
// smem -> TMA store).  TMEM: two 256-column fp32 accumulators.
#include "kernels.cuh"

namespace dion2 {

namespace {

constexpr int kBK = 64;
constexpr int kStagesPair = 5;
// 8 epilogue warps: two per TMEM lane group, each draining half of the tile's 256 columns
// (with K = p = 512 the 1-warp-per-lane-group epilogue was the bottleneck: ncu showed the
// MMA waiting on TMEM release while the producer waited on a full ring)
constexpr int kEpiWarps = 8;
constexpr int kPairThreads = 64 + 32 * kEpiWarps;
constexpr uint32_t kAB = 128 * kBK * 2;      // A half-tile per CTA (128 rows x 64 k)
constexpr uint32_t kBB = 128 * kBK * 2;      // B half-tile per CTA (128 n x 64 k)
constexpr uint32_t kStage = kAB + kBB;       // 32 KiB
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kIdescK = umma_idesc_bf16(256, 256, 0);
constexpr uint32_t kIdescMN = umma_idesc_bf16(256, 256, 1);

struct TileCoord {
  int group, z, tm, tn;
};

__device__ __forceinline__ TileCoord decode_tile(const NsParams& p, int t) {
  if (p.reverse) t = p.total_tiles - 1 - t;
  int g = 0;
#pragma unroll
  for (int i = 1; i < kMaxGroups; ++i)
    if (i < p.ngroups && t >= p.g[i].tile_base) g = i;
  const NsGroup& G = p.g[g];
  const int local = t - G.tile_base;
  TileCoord c;
  c.group = g;
  if (p.sym) {
    // symmetric output (gram A = X X^T, poly C = aI + bA + cA^2): upper-triangle tiles only,
    // row tm holds tiles tn = tm .. T-1
    const int T = G.m_tiles;
    const int per = T * (T + 1) / 2;
    c.z = local / per;
    int r = local % per, tm = 0;
    while (r >= T - tm) {
      r -= T - tm;
      ++tm;
    }
    c.tm = tm;
    c.tn = tm + r;
    return c;
  }
  const int per = G.m_tiles * G.n_tiles;
  c.z = local / per;
  const int r = local % per;
  c.tm = r / G.n_tiles;
  c.tn = r % G.n_tiles;
  return c;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// a/b operand format fields of the instruction descriptor: 1 = bf16, 0 = fp16
constexpr uint32_t kIdescAbFmt = (7u << 7) | (7u << 10);

}  // namespace

constexpr int ns_pair_smem_bytes() { return 1024 + kStagesPair * (int)kStage + 1024 + kEpiWarps * 4 * 2048; }

template <bool kSymIn>  // = P.p.sym_in (a template so non-symmetric launches carry no per-k-block logic)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
    k_ns_gemm_tc_pair(const __grid_constant__ NsTcParams P) {
  constexpr int S = kStagesPair;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * kStage);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  uint8_t* stage_base = smem + S * kStage + 1024;

  const NsParams& p = P.p;
  const int SK = p.splitk > 1 ? p.splitk : 1;
  const int nwork = p.total_tiles * SK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 2 * kEpiWarps);  // one arrival per epilogue warp of both CTAs
    }
    fence_mbar_init();
    for (int gi = 0; gi < p.ngroups; ++gi) {
      tma_prefetch_desc(&P.mapA[gi]);
      tma_prefetch_desc(&P.mapB[gi]);
      tma_prefetch_desc(&P.mapD[gi]);
      if (kSymIn) {
        tma_prefetch_desc(&P.mapAT[gi]);
        tma_prefetch_desc(&P.mapBT[gi]);
      }

    }
  }
  if (warp == 1) tmem_alloc_pair(tmem_base_slot, kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  pdl_wait();               // the previous launch's outputs are complete and visible
  pdl_launch_dependents();  // the next NS launch may begin its prologue on SMs we free

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      for (int w = cid; w < nwork; w += ncl) {
        const int t = w / SK, slice = w - (w / SK) * SK;
        const TileCoord c = decode_tile(p, t);
        const NsGroup& G = p.g[c.group];
        const int kb1 = (slice + 1) * G.k_blocks / SK;
        for (int kb = slice * G.k_blocks / SK; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kStage;
          uint8_t* sb = sa + kAB;
          const uint32_t leader_full = mapa_shared(smem_u32(&full_bar[stage]), 0);
          // b_is_a (gram X X^T, poly A A): on a diagonal tile CTA r's B half is its A half, so B
          // is not loaded (the MMA reads A's stage for both operands)
          const bool same = p.b_is_a && c.tm == c.tn;
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], same ? 2 * kAB : 2 * kStage);
          // sym_in: a k-block left of the diagonal tile is stored only as its transpose
          const bool at = kSymIn && ((kb * kBK) >> 8) < c.tm;
          const bool bt = kSymIn && ((kb * kBK) >> 8) < c.tn;
          // distributed owner gram: the K axis (q) runs over the P rank pieces of X0
          const int pr = G.pieces_load ? (kb * kBK) / G.pieces_qo : 0;
          const int pc = G.pieces_load ? kb * kBK - pr * G.pieces_qo : kb * kBK;
          const CUtensorMap* pmap = G.pieces_load ? &P.mapP[c.group][pr] : nullptr;
          if (!at) {
            tma_load_3d_pair(sa, pmap ? pmap : &P.mapA[c.group], leader_full, pc, c.tm * 256 + (int)rank * 128, c.z);
          } else {
#pragma unroll
            for (int j = 0; j < 2; ++j)
              tma_load_3d_pair(sa + j * 64 * kBK * 2, &P.mapAT[c.group], leader_full,
                               c.tm * 256 + (int)rank * 128 + j * 64, kb * kBK, c.z);
          }
          if (same) {
          } else if (p.b_kmajor && bt) {
#pragma unroll
            for (int j = 0; j < 2; ++j)
              tma_load_3d_pair(sb + j * 64 * kBK * 2, &P.mapBT[c.group], leader_full,
                               c.tn * 256 + (int)rank * 128 + j * 64, kb * kBK, c.z);
          } else if (p.b_kmajor) {
            tma_load_3d_pair(sb, pmap ? pmap : &P.mapB[c.group], leader_full, pc, c.tn * 256 + (int)rank * 128, c.z);
          } else {
#pragma unroll
            for (int j = 0; j < 2; ++j)
              tma_load_3d_pair(sb + j * 64 * kBK * 2, &P.mapB[c.group], leader_full,
                               c.tn * 256 + (int)rank * 128 + j * 64, kb * kBK, c.z);
          }
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---------------- MMA issuer (leader CTA; the whole warp runs the loop, one lane issues)
      const uint32_t idesc0 = (p.b_kmajor ? kIdescK : kIdescMN) & (p.in_f16 ? ~kIdescAbFmt : ~0u);
      // descriptors of the stage ring's offset 0 (K-major: 16 B LBO; MN-major: 64-column panels);
      // a stage / k-step adds its byte offset >> 4 to the 14-bit address field
      const uint32_t ring = smem_u32(smem);
      const uint64_t dK = umma_desc_sw128(ring, 16, 1024);
      const uint64_t dMN = umma_desc_sw128(ring, 64 * kBK * 2, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int w = cid; w < nwork; w += ncl, ++it) {
        const int t = w / SK, slice = w - (w / SK) * SK;
        const TileCoord c = decode_tile(p, t);
        const int kblocks = p.g[c.group].k_blocks;
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * 256;
        const int kb0 = slice * kblocks / SK, kb1 = (slice + 1) * kblocks / SK;
        const bool same = p.b_is_a && c.tm == c.tn;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_off = stage * kStage;
          const uint32_t b_off = same ? a_off : a_off + kAB;
          // sym_in: transposed (MN-major) operands of this k-block, as loaded by the producer
          const bool at = kSymIn && ((kb * kBK) >> 8) < c.tm;
          const bool bt = kSymIn ? (((kb * kBK) >> 8) < c.tn) : !p.b_kmajor;
          const uint32_t idesc = kSymIn ? (idesc0 | (at ? (1u << 15) : 0u) | (bt ? (1u << 16) : 0u)) : idesc0;
          if (elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t adesc = (at ? dMN : dK) + (uint64_t)((a_off + (at ? k * 2048 : k * 32)) >> 4);
              const uint64_t bdesc = (bt ? dMN : dK) + (uint64_t)((b_off + (bt ? k * 2048 : k * 32)) >> 4);
              umma_bf16_ss_pair(tmem_d, adesc, bdesc, idesc, (kb != kb0) || (k != 0));
            }
            umma_commit_pair(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        if (elect_one_sync()) umma_commit_pair(&tfull_bar[acc]);
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue (both CTAs; warps 2..9 -> TMEM lane groups 2,3,0,1,2,3,0,1;
    // warps 2..5 drain columns 0..127, warps 6..9 columns 128..255)
    const int ew = warp - 2;
    const int lg = warp & 3;
    const int c0 = (ew >> 2) * 4;  // first 32-column chunk of this warp
    const int row_in_tile = (int)rank * 128 + lg * 32 + lane;
    const uint32_t leader_tempty[2] = {mapa_shared(smem_u32(&tempty_bar[0]), 0),
                                       mapa_shared(smem_u32(&tempty_bar[1]), 0)};
    int sbuf = 0;
    int it = 0;
    for (int w = cid; w < nwork; w += ncl, ++it) {
      const int t = w / SK;
      const TileCoord c = decode_tile(p, t);
      const NsGroup& G = p.g[c.group];
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      if (SK > 1) {
        // split-K: raw fp32 partial of this slice (row row_in_tile, this warp's 128 columns)
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        float* dst = p.partial + ((int64_t)w * 256 + row_in_tile) * 256;
#pragma unroll 1
        for (int cc32 = c0; cc32 < c0 + 4; ++cc32) {
          float v[32];
          tmem_ld_32x32b_x32(tmem_base + acc * 256 + cc32 * 32 + ((uint32_t)(lg * 32) << 16), v);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            reinterpret_cast<float4*>(dst + cc32 * 32)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_tempty[acc]);
        continue;
      }
      float osc = 1.f;
      if (p.scale_sel) osc = p.ns_scale_all[4 * G.gmats[c.z] + (p.scale_sel - 1)];
      const float ca = p.cacc * osc, cc = p.cC * osc, dterm = p.diag * osc;
      const int64_t row = (int64_t)c.tm * 256 + row_in_tile;
      // cin holds 2-byte elements (bf16, or fp16 when in_f16)
      const uint16_t* cin =
          G.cin ? reinterpret_cast<const uint16_t*>(G.cin) + (int64_t)c.z * G.cin_mstride + row * G.cin_ld +
                      (int64_t)c.tn * 256
                : nullptr;
      uint4 craw[4] = {};
      if (cin) {
#pragma unroll
        for (int q = 0; q < 4; ++q) craw[q] = reinterpret_cast<const uint4*>(cin + c0 * 32)[q];
      }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int cc32 = c0; cc32 < c0 + 4; ++cc32) {
        float v[32];
        tmem_ld_32x32b_x32(tmem_base + acc * 256 + cc32 * 32 + ((uint32_t)(lg * 32) << 16), v);
        float cv[32];
        if (p.in_f16) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const __half2* h = reinterpret_cast<const __half2*>(&craw[q]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              cv[q * 8 + 2 * e] = __low2float(h[e]);
              cv[q * 8 + 2 * e + 1] = __high2float(h[e]);
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&craw[q]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              cv[q * 8 + 2 * e] = __low2float(h[e]);
              cv[q * 8 + 2 * e + 1] = __high2float(h[e]);
            }
          }
        }
        if (cin && cc32 + 1 < c0 + 4) {
#pragma unroll
          for (int q = 0; q < 4; ++q) craw[q] = reinterpret_cast<const uint4*>(cin + (cc32 + 1) * 32)[q];
        }
        const int dcol = (int)(row - ((int64_t)c.tn * 256 + cc32 * 32));
        float o[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = ca * v[e] + cc * cv[e] + (e == dcol ? dterm : 0.f);
        // 4 staging buffers per warp (SWIZZLE_64B layout: 16-B chunk q of row r at
        // q ^ ((r >> 1) & 3)); a buffer is rewritten once the store 4 commits back has read it
        const bool mirror = p.sym && !p.no_mirror && c.tm != c.tn;
        uint8_t* buf = stage_base + (ew * 4 + sbuf) * 2048;
        if (lane == 0) bulk_wait_read<3>();
        __syncwarp();
        uint32_t pk[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) pk[q] = p.out_f16 ? pack_f16x2(o[2 * q], o[2 * q + 1]) : pack_bf16x2(o[2 * q], o[2 * q + 1]);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          sts128(smem_u32(buf) + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4),
                 make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]));
        uint8_t* tbuf = stage_base + (ew * 4 + ((sbuf + 1) & 3)) * 2048;
        if (mirror) {
          // the transposed 32 x 32 chunk: element (row e, col lane) = o[e]; tbuf was used by
          // the 3rd most recent store (the current one is not issued yet)
          if (lane == 0) bulk_wait_read<2>();
          __syncwarp();
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const uint16_t h = p.out_f16 ? __half_as_ushort(__float2half_rn(o[e]))
                                         : __bfloat16_as_ushort(__float2bfloat16_rn(o[e]));
            sts16(smem_u32(tbuf) + e * 64 + ((((lane >> 3) ^ ((e >> 1) & 3))) << 4) + (lane & 7) * 2, h);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&P.mapD[c.group], buf, c.tn * 256 + cc32 * 32, c.tm * 256 + (int)rank * 128 + lg * 32, c.z);
          bulk_commit();
          if (mirror) {
            tma_store_3d(&P.mapD[c.group], tbuf, c.tm * 256 + (int)rank * 128 + lg * 32, c.tn * 256 + cc32 * 32,
                         c.z);
            bulk_commit();
          }
        }
        sbuf = (sbuf + (mirror ? 2 : 1)) & 3;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty[acc]);
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, kTmemCols);
  }
}

// Split-K reduction: block = 4 rows x 256 columns of one output tile; thread = 4 columns.
// Sums the slices in slice order (deterministic), applies the epilogue algebra of the pair
// kernel (oscale * cacc * acc + diag; split-K launches carry no cin) and writes the 2-byte
// output, plus the transposed copy of an off-diagonal symmetric tile unless no_mirror.
__global__ void __launch_bounds__(256) k_splitk_reduce(const NsParams p) {
  const int t = blockIdx.x >> 6;
  const int r = ((blockIdx.x & 63) << 2) + (threadIdx.x >> 6);
  const int c4 = (threadIdx.x & 63) << 2;
  const int S = p.splitk;
  const TileCoord c = decode_tile(p, t);
  const NsGroup& G = p.g[c.group];
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int sl = 0; sl < S; ++sl) {
    const float4 v = *reinterpret_cast<const float4*>(p.partial + (((int64_t)t * S + sl) * 256 + r) * 256 + c4);
    a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
  }
  float osc = 1.f;
  if (p.scale_sel) osc = p.ns_scale_all[4 * G.gmats[c.z] + (p.scale_sel - 1)];
  const float ca = p.cacc * osc, dterm = p.diag * osc;
  const int64_t row = (int64_t)c.tm * 256 + r, col = (int64_t)c.tn * 256 + c4;
  float o[4] = {ca * a.x, ca * a.y, ca * a.z, ca * a.w};
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (row == col + e) o[e] += dterm;
  uint16_t h[4];
#pragma unroll
  for (int e = 0; e < 4; ++e)
    h[e] = p.out_f16 ? __half_as_ushort(__float2half_rn(o[e])) : __bfloat16_as_ushort(__float2bfloat16_rn(o[e]));
  uint16_t* out = reinterpret_cast<uint16_t*>(G.out) + (int64_t)c.z * G.out_mstride;
  *reinterpret_cast<uint2*>(out + row * G.out_ld + col) =
      make_uint2((uint32_t)h[0] | ((uint32_t)h[1] << 16), (uint32_t)h[2] | ((uint32_t)h[3] << 16));
  if (p.sym && !p.no_mirror && c.tm != c.tn) {
#pragma unroll
    for (int e = 0; e < 4; ++e) out[(col + e) * G.out_ld + row] = h[e];
  }
}

void launch_splitk_reduce(cudaStream_t s, const NsParams& p) {
  k_splitk_reduce<<<p.total_tiles * 64, 256, 0, s>>>(p);
}

void ns_pair_set_attrs() {
  cudaFuncSetAttribute(k_ns_gemm_tc_pair<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, ns_pair_smem_bytes());
  cudaFuncSetAttribute(k_ns_gemm_tc_pair<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, ns_pair_smem_bytes());
}

void launch_ns_pair(int grid, cudaStream_t s, const NsTcParams& P) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kPairThreads);
  cfg.dynamicSmemBytes = ns_pair_smem_bytes();
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (P.p.sym_in)
    cudaLaunchKernelEx(&cfg, k_ns_gemm_tc_pair<true>, P);
  else
    cudaLaunchKernelEx(&cfg, k_ns_gemm_tc_pair<false>, P);
}

}  // namespace dion2
