// K6 apply on a CTA pair with the A operand resident in TENSOR MEMORY:
//   X' = oscale * (cacc * A X)        A = Q (Gram space, readings R23/R24) or C (direct form)
// M = p, N = q, K = p (p_pad <= 512), A [p x p] row-major (K-major), X [p x q] the MN-major B
// operand (Alg. 1 l.4).
//
// Why: X streams from DRAM at a rate set by the bytes in flight per SM (~3 us of latency under
// load: 64 KB in flight -> 3.2 TB/s, 128 KB -> 6 TB/s, profiles/r02_tma_box_microbench.txt),
// and the shared-memory resident A of k_ns_apply_pair leaves room for only 80 KB of X.  Here
// each CTA keeps its 128 rows of A in TMEM (lane = row, K packed two fp16 per 32-bit column:
// K / 2 <= 256 columns) and `tcgen05.mma ... [a_tmem]` reads A from there, so shared memory
// holds a 16-stage X ring (128 KB per CTA in flight) and the MMAs read only B from it.
//
// TMEM per CTA: columns [0, 256) A, [256, 384) and [384, 512) two 128-column accumulators
// (pair tile 256 x 128, tcgen05.mma.cta_group::2 256 x 128 x 16).
//
// Work unit = a chunk: one 256-row block tm of one matrix and a run of up to p.chunk_len
// 128-column blocks; chunks numbered (matrix, run, tm) with tm fastest and dealt round-robin to
// the CTA pairs (the pairs of one run read X together).  Per chunk the A rows are loaded into
// TMEM by four loader warps (global -> registers -> tcgen05.st), once the previous chunk's
// MMAs have completed.
//
// Roles per CTA (320 threads): warp 0 TMA producer (X ring), warp 1 TMEM allocator + MMA issuer
// (leader CTA, whole warp, one elected lane), warps 2-5 A loaders, warps 6-9 epilogue (one per
// TMEM lane group; TMEM -> scale -> 16-bit -> SWIZZLE_64B staging -> TMA store).
#include "kernels.cuh"

namespace dion2 {

namespace {

constexpr int kBK = 64;
constexpr int kStages = 16;
constexpr int kThreads = 64 + 128 + 128;
constexpr uint32_t kBB = 64 * kBK * 2;       // B per CTA and k-block: 64 columns x 64 k (8 KB)
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kAccCol0 = 256;           // accumulators at columns 256 and 384
constexpr uint32_t kIdescMN = umma_idesc_bf16(256, 128, 1);
constexpr uint32_t kIdescAbFmt = (7u << 7) | (7u << 10);
constexpr int kBarOff = kStages * (int)kBB;
constexpr int kStageOff = kBarOff + 1024;
constexpr int kSmem = 1024 + kStageOff + 4 * 2 * 2048;

struct Chunk {
  int group, z, tm, tn0, len;
};

// tile_base of a group = its first chunk; n_tiles counts 128-column blocks
__device__ __forceinline__ Chunk decode_chunk(const NsParams& p, int c) {
  int g = 0;
#pragma unroll
  for (int i = 1; i < kMaxGroups; ++i)
    if (i < p.ngroups && c >= p.g[i].tile_base) g = i;
  const NsGroup& G = p.g[g];
  const int L = p.chunk_len;
  const int runs = (G.n_tiles + L - 1) / L;
  const int per_z = runs * G.m_tiles;
  const int local = c - G.tile_base;
  Chunk k;
  k.group = g;
  k.z = local / per_z;
  const int r = local % per_z;
  k.tm = r % G.m_tiles;
  k.tn0 = (r / G.m_tiles) * L;
  k.len = min(L, G.n_tiles - k.tn0);
  return k;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// D[tmem] (+)= A[tmem] . B[smem], pair MMA
__device__ __forceinline__ void umma_ts_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// 32 lanes x 32 consecutive 32-bit columns from registers (thread t -> lane base + t)
__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_ns_apply_tmem(const __grid_constant__ NsTcParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = smem;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kBarOff);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* afull_bar = tempty_bar + 2;   // leader: A of a chunk in both CTAs' TMEM (8 loader warps)
  uint64_t* aempty_bar = afull_bar + 1;   // both: the previous chunk's MMAs are done with A
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(aempty_bar + 1);
  uint8_t* stage_base = smem + kStageOff;

  const NsParams& p = P.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();
  const int nchunks = p.total_tiles;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 2 * 4);  // the 4 epilogue warps of both CTAs
    }
    mbar_init(afull_bar, 2 * 4);          // the 4 loader warps of both CTAs
    mbar_init(aempty_bar, 1);
    fence_mbar_init();
    for (int gi = 0; gi < p.ngroups; ++gi) {
      tma_prefetch_desc(&P.mapB[gi]);
      tma_prefetch_desc(&P.mapD[gi]);
    }
  }
  if (warp == 1) tmem_alloc_pair(tmem_base_slot, kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: this CTA's 64 columns of every 128-column block of X
      int stage = 0;
      uint32_t phase = 0;
      for (int ci = cid; ci < nchunks; ci += ncl) {
        const Chunk k = decode_chunk(p, ci);
        const NsGroup& G = p.g[k.group];
        for (int tn = k.tn0; tn < k.tn0 + k.len; ++tn) {
          const int nn = tn * 128 + (int)rank * 64;
          for (int kb = 0; kb < G.k_blocks; ++kb) {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            const uint32_t leader_full = mapa_shared(smem_u32(&full_bar[stage]), 0);
            if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * kBB);
            uint8_t* sb = sB + stage * kBB;
            if (G.pieces_load) {  // distributed owner: the N axis (q) of X0 runs over the rank pieces
              const int pr = nn / G.pieces_qo;
              tma_load_3d_pair(sb, &P.mapP[k.group][G.pieces_P + pr], leader_full, nn - pr * G.pieces_qo, kb * kBK,
                               k.z);
            } else {
              tma_load_3d_pair(sb, &P.mapB[k.group], leader_full, nn, kb * kBK, k.z);
            }
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---------------- MMA issuer (leader CTA; whole warp, one elected lane issues)
      const uint32_t idesc = kIdescMN & (p.in_f16 ? ~kIdescAbFmt : ~0u);
      const uint64_t bdesc0 = umma_desc_sw128(smem_u32(sB), 64 * kBK * 2, 1024);
      int stage = 0, chunk = 0, it = 0;
      uint32_t phase = 0;
      for (int ci = cid; ci < nchunks; ci += ncl, ++chunk) {
        const Chunk k = decode_chunk(p, ci);
        const int kblocks = p.g[k.group].k_blocks;
        mbar_wait(afull_bar, chunk & 1);
        tc_fence_after();
        for (int tn = k.tn0; tn < k.tn0 + k.len; ++tn, ++it) {
          const int acc = it & 1;
          const uint32_t acc_phase = (it >> 1) & 1;
          mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t tmem_d = tmem_base + kAccCol0 + acc * 128;
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            if (elect_one_sync()) {
#pragma unroll
              for (int kk = 0; kk < kBK / 16; ++kk)
                umma_ts_pair(tmem_d, tmem_base + (uint32_t)(kb * (kBK / 2) + kk * 8),
                             bdesc0 + (uint64_t)((stage * kBB + kk * 2048) >> 4), idesc, (kb | kk) != 0);
              umma_commit_pair(&empty_bar[stage]);
            }
            __syncwarp();
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
          if (elect_one_sync()) umma_commit_pair(&tfull_bar[acc]);
          __syncwarp();
        }
        if (elect_one_sync()) umma_commit_pair(aempty_bar);  // this chunk's MMAs have read A
        __syncwarp();
      }
    }
  } else if (warp < 6) {
    // ---------------- A loaders: lane group lg = warp & 3 holds TMEM lanes 32 lg .. 32 lg + 31,
    // i.e. rows tm * 256 + rank * 128 + 32 lg + lane of A; K packed two fp16 per column
    const int lg = warp & 3;
    const uint32_t leader_afull = mapa_shared(smem_u32(afull_bar), 0);
    int chunk = 0;
    for (int ci = cid; ci < nchunks; ci += ncl, ++chunk) {
      const Chunk k = decode_chunk(p, ci);
      const NsGroup& G = p.g[k.group];
      mbar_wait(aempty_bar, (chunk & 1) ^ 1);  // the previous chunk's MMAs are done with A
      tc_fence_after();
      const int64_t row = (int64_t)k.tm * 256 + (int)rank * 128 + lg * 32 + lane;
      const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(G.a) +
                                                        (int64_t)k.z * G.a_mstride + row * G.lda);
      const int ncol32 = G.k_blocks;  // 64 k per block = 32 columns
      for (int c = 0; c < ncol32; ++c) {
        uint32_t r[32];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint4 v = __ldg(src + c * 8 + q);
          r[4 * q] = v.x; r[4 * q + 1] = v.y; r[4 * q + 2] = v.z; r[4 * q + 3] = v.w;
        }
        tmem_st_32x32b_x32(tmem_base + ((uint32_t)(lg * 32) << 16) + (uint32_t)(c * 32), r);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0)  // release: the tcgen05.st above are visible to the leader's MMAs
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(leader_afull) : "memory");
    }
  } else {
    // ---------------- epilogue (warps 6..9 -> TMEM lane groups 2,3,0,1; 4 x 32 columns each)
    const int lg = warp & 3;
    const int ew = warp - 6;
    const uint32_t leader_tempty[2] = {mapa_shared(smem_u32(&tempty_bar[0]), 0),
                                       mapa_shared(smem_u32(&tempty_bar[1]), 0)};
    int sbuf = 0, it = 0;
    for (int ci = cid; ci < nchunks; ci += ncl) {
      const Chunk k = decode_chunk(p, ci);
      const NsGroup& G = p.g[k.group];
      float osc = 1.f;
      if (p.scale_sel) osc = p.ns_scale_all[4 * G.gmats[k.z] + (p.scale_sel - 1)];
      const float ca = p.cacc * osc;
      const int row = k.tm * 256 + (int)rank * 128 + lg * 32;
      for (int tn = k.tn0; tn < k.tn0 + k.len; ++tn, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
#pragma unroll 1
        for (int cc32 = 0; cc32 < 4; ++cc32) {
          float v[32];
          tmem_ld_32x32b_x32(tmem_base + kAccCol0 + acc * 128 + cc32 * 32 + ((uint32_t)(lg * 32) << 16), v);
          uint8_t* buf = stage_base + (ew * 2 + sbuf) * 2048;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          uint32_t pk[16];
#pragma unroll
          for (int q = 0; q < 16; ++q)
            pk[q] = p.out_f16 ? pack2_h(ca * v[2 * q], ca * v[2 * q + 1]) : pack_bf16x2(ca * v[2 * q], ca * v[2 * q + 1]);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            sts128(smem_u32(buf) + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4),
                   make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]));
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int col = tn * 128 + cc32 * 32;
            if (G.pieces_store) {
              const int pr = col / G.pieces_qo;
              tma_store_3d(&P.mapP[k.group][2 * G.pieces_P + pr], buf, col - pr * G.pieces_qo, row, k.z);
            } else {
              tma_store_3d(&P.mapD[k.group], buf, col, row, k.z);
            }
            bulk_commit();
          }
          sbuf ^= 1;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_tempty[acc]);
      }
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

void ns_apply_tmem_set_attrs() {
  cudaFuncSetAttribute(k_ns_apply_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
}

void launch_ns_apply_tmem(int grid, cudaStream_t s, const NsTcParams& P) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_ns_apply_tmem, P);
}

}  // namespace dion2
