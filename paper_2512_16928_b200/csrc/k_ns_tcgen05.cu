// K4-K6: the Newton-Schulz GEMMs on the 5th-generation tensor cores.
//
// Newton-Schulz "require[s] only matrix multiplications and additions"
// (PAPER.md P:65); per iteration t with coefficients (a, b, c) (reading R1-R5):
//   gram  : A  = s_t^2 * X X^T        (M = N = p, K = q; both operands K-major rows of X)
//   poly  : B  = b*A + c*A A^T        (A symmetric, so A A^T = A^2; K-major)
//   apply : X' = s_t * (a*X + B X)    (M = p, N = q, K = p; X is the MN-major B operand)
// with s_1 = 1/(||X||_F + eps) folding the pre-normalisation into the first
// iteration and s_t = 1 afterwards.  Each output is rounded once to fp16 (or bf16,
// p.in_f16 / p.out_f16; reading R24); the poly epilogue reuses the same 16-bit A for the
// b*A term as the MMA saw ("consistent A", SURVEY finding 3).
//
// Kernel: persistent, warp-specialised, one CTA per SM.
//   warp 0      TMA producer (one elected lane): A tile 128x64, B tile BNx64 per stage
//   warp 1      TMEM allocator + MMA issuer (one lane): tcgen05.mma 128xBNx16, fp32 in TMEM
//   warps 2-5   epilogue: tcgen05.ld -> combine with C -> bf16 -> global
// smem ring of S stages (full/empty mbarriers), TMEM double-buffered
// accumulators (tmem_full/tmem_empty) so the epilogue of tile i overlaps
// the mainloop of tile i+1.  A static round-robin tile schedule walks all
// matrices of up to kMaxGroups shape groups in one launch.
#include "kernels.cuh"

namespace dion2 {

constexpr int kBM = 128, kBK = 64;

struct TileCoord {
  int group, z, tm, tn;
};

__device__ __forceinline__ TileCoord decode_tile(const NsParams& p, int t) {
  int g = 0;
#pragma unroll
  for (int i = 1; i < kMaxGroups; ++i)
    if (i < p.ngroups && t >= p.g[i].tile_base) g = i;
  const NsGroup& G = p.g[g];
  const int local = t - G.tile_base;
  const int per = G.m_tiles * G.n_tiles;
  TileCoord c;
  c.group = g;
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
// a/b operand format fields of the instruction descriptor: 1 = bf16, 0 = fp16
constexpr uint32_t kIdescAbFmt1 = (7u << 7) | (7u << 10);

template <int BN>
__global__ void __launch_bounds__(192, 1) k_ns_gemm_tc(const __grid_constant__ NsTcParams P) {
  constexpr int S = ns_tc_stages<BN>();
  constexpr uint32_t kABytes = kBM * kBK * 2;
  constexpr uint32_t kBBytes = BN * kBK * 2;
  constexpr uint32_t kStageBytes = kABytes + kBBytes;
  constexpr uint32_t kTmemCols = 2 * BN;  // two accumulators (256 or 512 columns)
  constexpr uint32_t kIdescK = umma_idesc_bf16(kBM, BN, 0);
  constexpr uint32_t kIdescMN = umma_idesc_bf16(kBM, BN, 1);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * kStageBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const NsParams& p = P.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 128);
    }
    fence_mbar_init();
    for (int gi = 0; gi < p.ngroups; ++gi) {
      tma_prefetch_desc(&P.mapA[gi]);
      tma_prefetch_desc(&P.mapB[gi]);
      tma_prefetch_desc(&P.mapD[gi]);
    }
  }
  if (warp == 1) tmem_alloc(tmem_base_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  pdl_wait();               // the previous launch's outputs are complete and visible
  pdl_launch_dependents();  // the next NS launch may begin its prologue on SMs we free

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
        const TileCoord c = decode_tile(p, t);
        const NsGroup& G = p.g[c.group];
        for (int kb = 0; kb < G.k_blocks; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kStageBytes;
          uint8_t* sb = sa + kABytes;
          mbar_arrive_expect_tx(&full_bar[stage], kStageBytes);
          tma_load_3d(sa, &P.mapA[c.group], &full_bar[stage], kb * kBK, c.tm * kBM, c.z);
          if (p.b_kmajor) {
            tma_load_3d(sb, &P.mapB[c.group], &full_bar[stage], kb * kBK, c.tn * BN, c.z);
          } else if (G.pieces_load) {
            // distributed owner apply: the N axis (q) of X0 runs over the P rank pieces
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) {
              const int nn = c.tn * BN + j * 64, pr = nn / G.pieces_qo;
              tma_load_3d(sb + j * 64 * kBK * 2, &P.mapP[c.group][G.pieces_P + pr], &full_bar[stage],
                          nn - pr * G.pieces_qo, kb * kBK, c.z);
            }
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_3d(sb + j * 64 * kBK * 2, &P.mapB[c.group], &full_bar[stage], c.tn * BN + j * 64, kb * kBK, c.z);
          }
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    {
      // ---------------- MMA issuer (the whole warp runs the loop, one lane issues)
      const uint32_t idesc = (p.b_kmajor ? kIdescK : kIdescMN) & (p.in_f16 ? ~kIdescAbFmt1 : ~0u);
      const uint32_t ring = smem_u32(smem);
      const uint64_t dK = umma_desc_sw128(ring, 16, 1024);
      const uint64_t dMN = umma_desc_sw128(ring, 64 * kBK * 2, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++it) {
        const TileCoord c = decode_tile(p, t);
        const int kblocks = p.g[c.group].k_blocks;
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_off = stage * kStageBytes;
          const uint32_t b_off = a_off + kABytes;
          if (elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t adesc = dK + (uint64_t)((a_off + k * 32) >> 4);
              const uint64_t bdesc = p.b_kmajor ? dK + (uint64_t)((b_off + k * 32) >> 4)
                                                : dMN + (uint64_t)((b_off + k * 2048) >> 4);
              umma_bf16_ss(tmem_d, adesc, bdesc, idesc, (kb | k) != 0);
            }
            umma_commit(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        if (elect_one_sync()) umma_commit(&tfull_bar[acc]);
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue (warps 2..5 -> TMEM lane groups 2,3,0,1)
    const int lg = warp & 3;
    const int row_in_tile = lg * 32 + lane;
    uint8_t* stage_base = smem + S * kStageBytes + 1024;  // 1024-B aligned, after the barriers
    int sbuf = 0;
    int it = 0;
    for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++it) {
      const TileCoord c = decode_tile(p, t);
      const NsGroup& G = p.g[c.group];
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      float osc = 1.f;
      if (p.scale_sel) osc = p.ns_scale_all[4 * G.gmats[c.z] + (p.scale_sel - 1)];
      const float ca = p.cacc * osc, cc = p.cC * osc, dterm = p.diag * osc;
      const int64_t row = (int64_t)c.tm * kBM + row_in_tile;
      // cin holds 2-byte elements (bf16, or fp16 when in_f16)
      const uint16_t* cin =
          G.cin ? reinterpret_cast<const uint16_t*>(G.cin) + (int64_t)c.z * G.cin_mstride + row * G.cin_ld +
                      (int64_t)c.tn * BN
                : nullptr;
      // C-term (poly: b*A) for chunk 0 is fetched before the accumulator is ready,
      // then one chunk ahead: its latency hides under the MMA / the previous chunk.
      uint4 craw[4] = {};
      if (cin) {
#pragma unroll
        for (int q = 0; q < 4; ++q) craw[q] = reinterpret_cast<const uint4*>(cin)[q];
      }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int cc32 = 0; cc32 < BN / 32; ++cc32) {
        float v[32];
        tmem_ld_32x32b_x32(tmem_base + acc * BN + cc32 * 32 + ((uint32_t)(lg * 32) << 16), v);
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
        if (cin && cc32 + 1 < BN / 32) {
#pragma unroll
          for (int q = 0; q < 4; ++q) craw[q] = reinterpret_cast<const uint4*>(cin + (cc32 + 1) * 32)[q];
        }
        // diagonal term (poly phase: C = a*I + b*A + c*A*A): element e sits on the
        // global diagonal iff row == col0 + e
        const int dcol = (int)(row - ((int64_t)c.tn * BN + cc32 * 32));
        float o[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = ca * v[e] + cc * cv[e] + (e == dcol ? dterm : 0.f);
        // stage the 32x32 16-bit chunk in SWIZZLE_64B layout (row = lane, 16-B chunk
        // q stored at q ^ ((row >> 1) & 3): conflict-free) and TMA-store it
        uint8_t* buf = stage_base + (lg * 2 + sbuf) * 2048;
        if (lane == 0) bulk_wait_read<1>();  // the store that used this buffer two chunks ago is done reading
        __syncwarp();
        uint32_t pk[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) pk[q] = p.out_f16 ? pack2_h(o[2 * q], o[2 * q + 1]) : pack_bf16x2(o[2 * q], o[2 * q + 1]);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          sts128(smem_u32(buf) + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4),
                 make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]));
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const NsGroup& Gs = p.g[c.group];
          const int col = c.tn * BN + cc32 * 32;
          if (Gs.pieces_store) {  // X_T straight into the rank pieces of the exchange buffer
            const int pr = col / Gs.pieces_qo;
            tma_store_3d(&P.mapP[c.group][2 * Gs.pieces_P + pr], buf, col - pr * Gs.pieces_qo,
                         c.tm * kBM + lg * 32, c.z);
          } else {
            tma_store_3d(&P.mapD[c.group], buf, col, c.tm * kBM + lg * 32, c.z);
          }
          bulk_commit();
        }
        sbuf ^= 1;
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

void ns_tc_set_attrs() {
  cudaFuncSetAttribute(k_ns_gemm_tc<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, ns_tc_smem_bytes<128>());
  cudaFuncSetAttribute(k_ns_gemm_tc<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, ns_tc_smem_bytes<256>());
}

void launch_ns_tc(int bn, int grid, cudaStream_t s, const NsTcParams& P) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(192);
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (bn == 256) {
    cfg.dynamicSmemBytes = ns_tc_smem_bytes<256>();
    cudaLaunchKernelEx(&cfg, k_ns_gemm_tc<256>, P);
  } else {
    cfg.dynamicSmemBytes = ns_tc_smem_bytes<128>();
    cudaLaunchKernelEx(&cfg, k_ns_gemm_tc<128>, P);
  }
}

}  // namespace dion2
