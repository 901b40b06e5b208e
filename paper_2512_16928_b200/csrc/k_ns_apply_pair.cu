// K6 apply on a CTA pair with the A operand resident in shared memory:
//   X' = oscale * (cacc * A X)        A = Q (Gram space, readings R23/R24) or C (direct form)
// M = p, N = q, K = p (p_pad <= 512), A [p x p] K-major, X [p x q] the MN-major B operand
// (Alg. 1 l.4).
//
// The apply's K is short (p = 512 at alpha = 1/4 on the 1B set) and its N long (q = 2048 ..
// 8192).  Work unit = a CHUNK: one 256-row block (tm) of one matrix and a run of up to
// p.chunk_len consecutive 256-column blocks.  The pair loads its 256 rows of A (128 per CTA,
// K x 128 fp16 <= 128 KB) once per chunk and keeps them in shared memory while it streams the
// chunk's X column blocks through a 4-stage ring (16 KB per CTA per k-block): per CTA and tile
// 128 KB of B, against 128 KB of A + 128 KB of B for the pair kernel and 384 KB for the 1-SM
// kernel.  Chunks are numbered (matrix, column run, tm) with tm fastest and dealt round-robin
// to the pairs, so the p / 256 chunks that read the same X column blocks run on neighbouring
// pairs at the same time and X comes from DRAM once (a pair-contiguous tile range read it
// twice: ncu 1.30 GB for 0.6 GB of X, 0.353 ms per launch).
//
// Roles per CTA (320 threads): warp 0 TMA producer (A blocks on a chunk change, then the B
// ring; completion counted on the leader's barriers), warp 1 TMEM allocator (both CTAs) + MMA
// issuer (leader: tcgen05.mma.cta_group::2 256 x 256 x 16, fp16/bf16 -> fp32), warps 2-9
// epilogue (TMEM -> scale -> 16-bit -> SWIZZLE_64B staging -> TMA store; two 256-column TMEM
// accumulators so the epilogue of one tile overlaps the next tile's MMAs).
#include "kernels.cuh"

namespace dion2 {

namespace {

constexpr int kBK = 64;
// 5 B stages (80 KB of X in flight per CTA) and one 2 KB epilogue staging buffer per warp: the
// resident A takes 128 KB, and X streams from DRAM at a rate set by the bytes in flight
// (profiles/r02_tma_box_microbench.txt: 64 KB per SM -> 3.2 TB/s, 128 KB -> 6 TB/s)
constexpr int kStages = 5;
constexpr int kStgBufs = 1;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr uint32_t kABlk = 128 * kBK * 2;    // one resident A k-block per CTA (128 rows x 64 k)
constexpr uint32_t kBB = 128 * kBK * 2;      // B half-tile per CTA and k-block (128 n x 64 k)
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kIdescMN = umma_idesc_bf16(256, 256, 1);
constexpr uint32_t kIdescAbFmt = (7u << 7) | (7u << 10);  // a/b format fields: 1 = bf16, 0 = fp16
constexpr int kAOff = 0;
constexpr int kBOff = kMaxResidentKB * (int)kABlk;
constexpr int kBarOff = kBOff + kStages * (int)kBB;
constexpr int kStageOff = kBarOff + 1024;
constexpr int kSmem = 1024 + kStageOff + kEpiWarps * kStgBufs * 2048;

struct Chunk {
  int group, z, tm, tn0, len;
};

// chunk index -> (group, z, tm, first column block, column blocks); NsGroup::tile_base holds
// the group's first chunk index here
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

}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_ns_apply_pair(const __grid_constant__ NsTcParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem + kAOff;
  uint8_t* sB = smem + kBOff;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kBarOff);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* afull_bar = tempty_bar + 2;
  uint64_t* aempty_bar = afull_bar + 1;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(aempty_bar + 1);
  uint8_t* stage_base = smem + kStageOff;

  const NsParams& p = P.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();
  const int nchunks = p.total_tiles;  // kind 5 launches count chunks

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 2 * kEpiWarps);
    }
    mbar_init(afull_bar, 1);
    mbar_init(aempty_bar, 1);
    fence_mbar_init();
    for (int gi = 0; gi < p.ngroups; ++gi) {
      tma_prefetch_desc(&P.mapA[gi]);
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
      // ---------------- TMA producer (both CTAs)
      int stage = 0, chunk = 0;
      uint32_t phase = 0;
      const uint32_t leader_afull = mapa_shared(smem_u32(afull_bar), 0);
      for (int ci = cid; ci < nchunks; ci += ncl, ++chunk) {
        const Chunk k = decode_chunk(p, ci);
        const NsGroup& G = p.g[k.group];
        // reload the resident A rows once the previous chunk's MMAs have read them (the first
        // wait passes on the fresh barrier's preceding phase)
        mbar_wait(aempty_bar, (chunk & 1) ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(afull_bar, 2 * kABlk * G.k_blocks);
        for (int kb = 0; kb < G.k_blocks; ++kb)
          tma_load_3d_pair(sA + kb * kABlk, &P.mapA[k.group], leader_afull, kb * kBK, k.tm * 256 + (int)rank * 128, k.z);
        for (int tn = k.tn0; tn < k.tn0 + k.len; ++tn) {
          // L2 prefetch of the next column block's B (this CTA's half): the ring holds only
          // 4 k-blocks (~1.6 us of MMA), less than a DRAM round trip under load, so the loads
          // of the next tile should hit L2 (ncu: the MMA waited on its full barriers while the
          // producer sat on a full ring, DRAM at 49%)
          if (tn + 1 < k.tn0 + k.len && !G.pieces_load) {
            for (int kb = 0; kb < G.k_blocks; ++kb)
#pragma unroll
              for (int j = 0; j < 2; ++j)
                tma_prefetch_3d(&P.mapB[k.group], (tn + 1) * 256 + (int)rank * 128 + j * 64, kb * kBK, k.z);
          }
          for (int kb = 0; kb < G.k_blocks; ++kb) {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            uint8_t* sb = sB + stage * kBB;
            const uint32_t leader_full = mapa_shared(smem_u32(&full_bar[stage]), 0);
            if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * kBB);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int nn = tn * 256 + (int)rank * 128 + j * 64;
              if (G.pieces_load) {  // distributed owner: the N axis (q) of X0 runs over the rank pieces
                const int pr = nn / G.pieces_qo;
                tma_load_3d_pair(sb + j * 64 * kBK * 2, &P.mapP[k.group][G.pieces_P + pr], leader_full,
                                 nn - pr * G.pieces_qo, kb * kBK, k.z);
              } else {
                tma_load_3d_pair(sb + j * 64 * kBK * 2, &P.mapB[k.group], leader_full, nn, kb * kBK, k.z);
              }
            }
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---------------- MMA issuer (leader CTA; the whole warp runs the loop, one lane issues)
      const uint32_t idesc = kIdescMN & (p.in_f16 ? ~kIdescAbFmt : ~0u);
      // descriptors of offset 0; a k-step / stage adds its byte offset >> 4 to the address field
      const uint64_t adesc0 = umma_desc_sw128(smem_u32(sA), 16, 1024);
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
          const uint32_t tmem_d = tmem_base + acc * 256;
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            if (elect_one_sync()) {
#pragma unroll
              for (int kk = 0; kk < kBK / 16; ++kk)
                umma_bf16_ss_pair(tmem_d, adesc0 + (uint64_t)((kb * kABlk + kk * 32) >> 4),
                                  bdesc0 + (uint64_t)((stage * kBB + kk * 2048) >> 4), idesc, (kb | kk) != 0);
              umma_commit_pair(&empty_bar[stage]);
            }
            __syncwarp();
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
          if (elect_one_sync()) umma_commit_pair(&tfull_bar[acc]);
          __syncwarp();
        }
        if (elect_one_sync()) umma_commit_pair(aempty_bar);  // this chunk's MMAs have read the resident A
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue (both CTAs; warps 2..9 -> TMEM lane groups 2,3,0,1,2,3,0,1;
    // warps 2..5 drain columns 0..127, warps 6..9 columns 128..255)
    const int ew = warp - 2;
    const int lg = warp & 3;
    const int c0 = (ew >> 2) * 4;
    const uint32_t leader_tempty[2] = {mapa_shared(smem_u32(&tempty_bar[0]), 0),
                                       mapa_shared(smem_u32(&tempty_bar[1]), 0)};
    int sbuf = 0, it = 0;
    for (int ci = cid; ci < nchunks; ci += ncl) {
     const Chunk k = decode_chunk(p, ci);
     const NsGroup& G = p.g[k.group];
     float osc = 1.f;
     if (p.scale_sel) osc = p.ns_scale_all[4 * G.gmats[k.z] + (p.scale_sel - 1)];
     const float ca = p.cacc * osc;
     for (int tn = k.tn0; tn < k.tn0 + k.len; ++tn, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int cc32 = c0; cc32 < c0 + 4; ++cc32) {
        float v[32];
        tmem_ld_32x32b_x32(tmem_base + acc * 256 + cc32 * 32 + ((uint32_t)(lg * 32) << 16), v);
        uint8_t* buf = stage_base + (ew * kStgBufs + sbuf) * 2048;
        if (lane == 0) bulk_wait_read<kStgBufs - 1>();  // the store that last used this buffer has read it
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
          const int col = tn * 256 + cc32 * 32, row = k.tm * 256 + (int)rank * 128 + lg * 32;
          if (G.pieces_store) {  // X_T straight into the rank pieces of the exchange buffer
            const int pr = col / G.pieces_qo;
            tma_store_3d(&P.mapP[k.group][2 * G.pieces_P + pr], buf, col - pr * G.pieces_qo, row, k.z);
          } else {
            tma_store_3d(&P.mapD[k.group], buf, col, row, k.z);
          }
          bulk_commit();
        }
        sbuf = (sbuf + 1) % kStgBufs;
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

void ns_apply_pair_set_attrs() {
  cudaFuncSetAttribute(k_ns_apply_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
}

void launch_ns_apply_pair(int grid, cudaStream_t s, const NsTcParams& P) {
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
  cudaLaunchKernelEx(&cfg, k_ns_apply_pair, P);
}

}  // namespace dion2
