// K5 chain: the p x p products of the Gram-space Newton-Schulz form (reading R23,
// include/dion2.h dion2_ns_form) in ONE persistent launch.
//
// Per matrix the recursion is a fixed list of ops on five p x p buffers (A, C, Q0, Q1, B):
//   poly  C_t = a_t I + b_t A + c_t A A      (A-term read by the epilogue)
//   C.A   B   = C_t A
//   C.Q   Q'  = C_t Q
//   C.B   A   = C_t B
// Every product is symmetric (a polynomial in A_0), so only upper-triangle 256 x 256 tiles
// are computed and mirrored, as in k_ns_tcgen05_pair.cu.  Launching each op over all
// matrices (the flat kernel) streams every buffer of every matrix through HBM per op: the
// 1B set's 144 x 5 x 512 KiB does not fit the 126 MB L2.  Here one CTA pair owns one matrix
// at a time and runs its whole op list back to back, so an op's operands were written a
// few microseconds earlier by the same pair and are L2-resident.
//
// Dependencies: op j may start its TMA loads once the ops that last wrote its operands (and
// last read its output buffer) have completed -- the host computes that index (ChainOp::dep,
// dion2_api.cu append_gram_space_launches).  Completion is a monotonic
// counter per CTA: every epilogue warp of the pair, after its last tile of an op, waits for
// its bulk stores to complete, fences the async proxy and adds 1 with release semantics to
// the counter of both CTAs (8 per op).  The producer (and the epilogue, before reading the
// A-term) spins with acquire semantics until the counter reaches 8 x (ops to wait for).
#include "kernels.cuh"

namespace dion2 {

namespace {

constexpr int kBK = 64;
constexpr int kStagesC = 6;
constexpr uint32_t kAB = 128 * kBK * 2;
constexpr uint32_t kBB = 128 * kBK * 2;
constexpr uint32_t kStage = kAB + kBB;
constexpr uint32_t kTmemCols = 512;
// fp16 x fp16 -> fp32, K-major A and B, 256 x 256
constexpr uint32_t kIdescF16 = umma_idesc_bf16(256, 256, 0) & ~((7u << 7) | (7u << 10));

__device__ __forceinline__ void sym_tile(int r, int T, int& tm, int& tn) {
  int m = 0;
  while (r >= T - m) {
    r -= T - m;
    ++m;
  }
  tm = m;
  tn = m + r;
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi, int f16) {
  if (f16) {
    __half2 v = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
  }
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void red_release_cluster_add(uint32_t cluster_addr, uint32_t v) {
  asm volatile("red.release.cluster.shared::cluster.add.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_cluster(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

// wait until `target` op completions (x 8 epilogue warps) have been counted
__device__ __forceinline__ void wait_done(const uint32_t* counter, uint32_t target) {
  if (ld_acquire_cluster(counter) >= target) return;
  const long long t0 = clock64();
  while (ld_acquire_cluster(counter) < target) {
    if (clock64() - t0 > DION2_WATCHDOG_CYCLES) __trap();
  }
}

}  // namespace

constexpr int ns_chain_smem_bytes() { return 1024 + kStagesC * (int)kStage + 1024 + 4 * 4 * 2048; }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    k_ns_chain_pair(const __grid_constant__ NsChainParams P) {
  constexpr int S = kStagesC;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * kStage);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  uint32_t* done_ctr = tmem_base_slot + 1;  // op completions x 8 (this CTA's copy)
  uint8_t* stage_base = smem + S * kStage + 1024;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();
  const int nops = P.nops;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 8);
    }
    *done_ctr = 0;
    fence_mbar_init();
    for (int gi = 0; gi < P.ngroups; ++gi)
      for (int b = 0; b < kChainBufs; ++b) {
        tma_prefetch_desc(&P.ld[gi][b]);
        tma_prefetch_desc(&P.st[gi][b]);
      }
  }
  if (warp == 1) tmem_alloc_pair(tmem_base_slot, kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      uint32_t base = 0;  // ops of earlier matrices (this pair)
      for (int e = cid; e < P.n_entries; e += ncl, base += nops) {
        const int ent = P.entries[e];
        const int g = ent >> 24, z = ent & 0xFFFFFF;
        const int T = P.p_pad[g] >> 8, per = T * (T + 1) / 2, kblocks = P.p_pad[g] / kBK;
        for (int op = 0; op < nops; ++op) {
          const ChainOp& o = P.ops[op];
          if (o.dep >= 0) {
            wait_done(done_ctr, 8u * (base + (uint32_t)o.dep + 1u));
            fence_proxy_async_global();
          }
          const CUtensorMap* ma = &P.ld[g][o.a];
          const CUtensorMap* mb = &P.ld[g][o.b];
          for (int r = 0; r < per; ++r) {
            int tm, tn;
            sym_tile(r, T, tm, tn);
            for (int kb = 0; kb < kblocks; ++kb) {
              mbar_wait(&empty_bar[stage], phase ^ 1);
              uint8_t* sa = smem + stage * kStage;
              const uint32_t leader_full = mapa_shared(smem_u32(&full_bar[stage]), 0);
              if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * kStage);
              tma_load_3d_pair(sa, ma, leader_full, kb * kBK, tm * 256 + (int)rank * 128, z);
              tma_load_3d_pair(sa + kAB, mb, leader_full, kb * kBK, tn * 256 + (int)rank * 128, z);
              if (++stage == S) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------- MMA issuer (leader CTA)
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int e = cid; e < P.n_entries; e += ncl) {
        const int g = P.entries[e] >> 24;
        const int T = P.p_pad[g] >> 8, per = T * (T + 1) / 2, kblocks = P.p_pad[g] / kBK;
        const int tiles = nops * per;
        for (int i = 0; i < tiles; ++i, ++it) {
          const int acc = it & 1;
          const uint32_t acc_phase = (it >> 1) & 1;
          mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t tmem_d = tmem_base + acc * 256;
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            const uint32_t a_addr = smem_u32(smem + stage * kStage);
            const uint32_t b_addr = a_addr + kAB;
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              umma_bf16_ss_pair(tmem_d, umma_desc_sw128(a_addr + k * 32, 16, 1024),
                                umma_desc_sw128(b_addr + k * 32, 16, 1024), kIdescF16, (kb | k) != 0);
            umma_commit_pair(&empty_bar[stage]);
            if (++stage == S) { stage = 0; phase ^= 1; }
          }
          umma_commit_pair(&tfull_bar[acc]);
        }
      }
    }
  } else {
    // ---------------- epilogue (both CTAs; warps 2..5 -> TMEM lane groups 2,3,0,1)
    const int lg = warp & 3;
    const int row_in_tile = (int)rank * 128 + lg * 32 + lane;
    const uint32_t leader_tempty[2] = {mapa_shared(smem_u32(&tempty_bar[0]), 0),
                                       mapa_shared(smem_u32(&tempty_bar[1]), 0)};
    const uint32_t ctr_remote[2] = {mapa_shared(smem_u32(done_ctr), 0), mapa_shared(smem_u32(done_ctr), 1)};
    int sbuf = 0;
    int it = 0;
    uint32_t base = 0;
    for (int e = cid; e < P.n_entries; e += ncl, base += nops) {
      const int ent = P.entries[e];
      const int g = ent >> 24, z = ent & 0xFFFFFF;
      const int T = P.p_pad[g] >> 8, per = T * (T + 1) / 2;
      const int ld = P.p_pad[g];
      for (int op = 0; op < nops; ++op) {
        const ChainOp& o = P.ops[op];
        const CUtensorMap* md = &P.st[g][o.out];
        const uint16_t* cbase = nullptr;
        if (o.cin >= 0) {
          // the A-term was written by an earlier op of this pair: wait for it
          if (o.cin_dep >= 0) {
            wait_done(done_ctr, 8u * (base + (uint32_t)o.cin_dep + 1u));
            fence_proxy_async_global();
          }
          cbase = reinterpret_cast<const uint16_t*>(P.buf[g][o.cin]) + (int64_t)z * P.mstride[g];
        }
        for (int r = 0; r < per; ++r, ++it) {
          int tm, tn;
          sym_tile(r, T, tm, tn);
          const int acc = it & 1;
          const uint32_t acc_phase = (it >> 1) & 1;
          const int64_t row = (int64_t)tm * 256 + row_in_tile;
          const uint16_t* cin = cbase ? cbase + row * ld + (int64_t)tn * 256 : nullptr;
          uint4 craw[4] = {};
          if (cin) {
#pragma unroll
            for (int q = 0; q < 4; ++q) craw[q] = __ldcg(reinterpret_cast<const uint4*>(cin) + q);
          }
          mbar_wait(&tfull_bar[acc], acc_phase);
          tc_fence_after();
#pragma unroll 1
          for (int cc32 = 0; cc32 < 8; ++cc32) {
            float v[32];
            tmem_ld_32x32b_x32(tmem_base + acc * 256 + cc32 * 32 + ((uint32_t)(lg * 32) << 16), v);
            float cv[32];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const __half2* h = reinterpret_cast<const __half2*>(&craw[q]);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                cv[q * 8 + 2 * k] = __low2float(h[k]);
                cv[q * 8 + 2 * k + 1] = __high2float(h[k]);
              }
            }
            if (cin && cc32 + 1 < 8) {
#pragma unroll
              for (int q = 0; q < 4; ++q) craw[q] = __ldcg(reinterpret_cast<const uint4*>(cin + (cc32 + 1) * 32) + q);
            }
            const int dcol = (int)(row - ((int64_t)tn * 256 + cc32 * 32));
            float out[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) out[k] = o.cacc * v[k] + o.cC * cv[k] + (k == dcol ? o.diag : 0.f);
            const bool mirror = tm != tn;
            uint8_t* buf = stage_base + (lg * 4 + sbuf) * 2048;
            if (lane == 0) bulk_wait_read<3>();
            __syncwarp();
            uint32_t pk[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) pk[q] = pack2(out[2 * q], out[2 * q + 1], o.out_f16);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              sts128(smem_u32(buf) + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4),
                 make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]));
            uint8_t* tbuf = stage_base + (lg * 4 + ((sbuf + 1) & 3)) * 2048;
            if (mirror) {
              if (lane == 0) bulk_wait_read<2>();
              __syncwarp();
#pragma unroll
              for (int k = 0; k < 32; ++k) {
                const uint16_t h = o.out_f16 ? __half_as_ushort(__float2half_rn(out[k]))
                                             : __bfloat16_as_ushort(__float2bfloat16_rn(out[k]));
                sts16(smem_u32(tbuf) + k * 64 + ((((lane >> 3) ^ ((k >> 1) & 3))) << 4) + (lane & 7) * 2, h);
              }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_3d(md, buf, tn * 256 + cc32 * 32, tm * 256 + (int)rank * 128 + lg * 32, z);
              bulk_commit();
              if (mirror) {
                tma_store_3d(md, tbuf, tm * 256 + (int)rank * 128 + lg * 32, tn * 256 + cc32 * 32, z);
                bulk_commit();
              }
            }
            sbuf = (sbuf + (mirror ? 2 : 1)) & 3;
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(leader_tempty[acc]);
        }
        // op complete for this warp: its stores are globally performed before the count
        if (lane == 0) {
          bulk_wait_all();
          fence_proxy_async_global();
          red_release_cluster_add(ctr_remote[0], 1);
          red_release_cluster_add(ctr_remote[1], 1);
        }
        __syncwarp();
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

void ns_chain_set_attrs() {
  cudaFuncSetAttribute(k_ns_chain_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, ns_chain_smem_bytes());
}

void launch_ns_chain(int grid, cudaStream_t s, const NsChainParams& P) {
  k_ns_chain_pair<<<grid, 192, ns_chain_smem_bytes(), s>>>(P);
}

}  // namespace dion2
