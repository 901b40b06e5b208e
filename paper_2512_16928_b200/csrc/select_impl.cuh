// select_impl.cuh -- K2 body: top-k selection of one matrix by one CTA (Alg. 1 l.3,
// PAPER.md P:184).  Default rule: the k rows/columns with the largest l1 norm;
// ties go to the lower index (reading R9); K is emitted in ascending index order.
//
// Scores are non-negative fp32, so their bit patterns order like the values: a
// 4 x 8-bit MSB-first radix select finds the k-th largest key T exactly; then elements
// > T are taken, and of the elements == T the lowest-index ones, via two block-wide
// prefix sums in index order.  Integer-only after the scores exist: bit-exact and
// deterministic for any block size (a multiple of 32, at most 1024).
//
// Used by k_topk_select (one CTA per matrix); scores are read with ld.global.cg (L2).
#pragma once
#include "common.cuh"

namespace dion2 {

struct SelectSmem {
  uint32_t hist[256];
  int warp_tot[33];
  uint32_t s_prefix, s_remaining;
  uint32_t smax;  // bits of the largest score (non-negative floats order like their bits)
};


__device__ __forceinline__ int block_exclusive_scan(int v, int* warp_tot, int* total_out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = (lane < (int)(blockDim.x >> 5)) ? warp_tot[lane] : 0;
    int s = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    warp_tot[lane] = s - w;  // exclusive warp offsets
    if (lane == 31) warp_tot[32] = s;
  }
  __syncthreads();
  const int res = warp_tot[wid] + x - v;
  *total_out = warp_tot[32];
  __syncthreads();
  return res;
}

__device__ __forceinline__ void select_matrix(const MatDesc& md, int mi, uint32_t* __restrict__ keys,
                                              SelectSmem& sh, int32_t* __restrict__ bad,
                                              int32_t* __restrict__ status, int random_sel, uint64_t seed,
                                              uint64_t step) {
  uint32_t* hist = sh.hist;
  int* warp_tot = sh.warp_tot;
  uint32_t& s_prefix = sh.s_prefix;
  uint32_t& s_remaining = sh.s_remaining;
  const int d = md.d, k = md.k;
  const int tid = threadIdx.x;

  // 1. scores -> keys (cols mode: fixed-order sum of the K1 row-block partials)
  int nonfinite = 0;
  uint32_t smax = 0u;
  if (tid == 0) sh.smax = 0u;
  __syncthreads();
#pragma unroll 4
  for (int i = tid; i < d; i += blockDim.x) {
    float s;
    if (md.axis == kAxisCols && !md.scores_final) {
      s = 0.f;
      for (int rb = 0; rb < md.rowblocks; ++rb) s += __ldcg(md.col_partials + (int64_t)rb * md.cols + i);
      md.scores[i] = s;
    } else {
      s = __ldcg(md.scores + i);
    }
    if (!(s <= 3.402823466e38f)) nonfinite = 1;  // NaN or +Inf
    smax = max(smax, __float_as_uint(s));
    // Random rule: the k SMALLEST Philox keys = the k largest complemented keys;
    // ties (p ~ 2^-32) go to the lower index exactly as for the l1 rule.
    keys[i] = random_sel ? ~philox_word0((uint32_t)i, (uint32_t)step, (uint32_t)(step >> 32), (uint32_t)md.mid,
                                         (uint32_t)seed, (uint32_t)(seed >> 32))
                         : __float_as_uint(s);
  }
  smax = __reduce_max_sync(0xffffffffu, smax);
  if ((tid & 31) == 0) atomicMax(&sh.smax, smax);
  nonfinite = __syncthreads_or(nonfinite);
  if (tid == 0 && md.ns_scale) {
    md.ns_scale[2] = (md.x16 && !nonfinite) ? x16_prescale(__uint_as_float(sh.smax)) : 1.f;
    md.ns_scale[3] = __uint_as_float(sh.smax);  // the bound itself (compressed DP-sync combines it)
  }
  if (nonfinite) {
    if (tid == 0) {
      bad[mi] = 1;
      set_status_bad(status, md.mid);
    }
    for (int i = tid; i < k; i += blockDim.x) {
      md.sel[i] = i;
      if (md.sel_out) md.sel_out[i] = i;
    }
    return;
  }
  if (tid == 0) bad[mi] = 0;

  // 2. radix select of the k-th largest key
  uint32_t prefix = 0, mask = 0;
  uint32_t remaining = (uint32_t)k;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    // warp-aggregated: lanes sharing a bin add once (scores of similar magnitude share
    // their top bits, so unaggregated shared atomics serialise on one bin)
    for (int base = 0; base < d; base += blockDim.x) {
      const int i = base + tid;
      uint32_t bin = 256u;  // 256: not counted
      if (i < d) {
        const uint32_t key = keys[i];
        if ((key & mask) == prefix) bin = (key >> shift) & 255u;
      }
      const unsigned peers = __match_any_sync(0xffffffffu, bin);
      if (bin < 256u && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
    }
    __syncthreads();
    if (tid < 32) {
      // warp-parallel scan from the top bin down: lane l owns bins 255-8l .. 248-8l
      uint32_t c[8], tot = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        c[e] = hist[255 - 8 * tid - e];
        tot += c[e];
      }
      uint32_t incl = tot;  // inclusive prefix over lanes (higher bins first)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += y;
      }
      const uint32_t excl = incl - tot;
      // the lane whose range contains the k-th largest key
      const unsigned hit = __ballot_sync(0xffffffffu, excl < remaining && incl >= remaining);
      if (tid == __ffs(hit) - 1) {
        uint32_t above = excl;
        int e = 0;
        for (; e < 7; ++e) {
          if (above + c[e] >= remaining) break;
          above += c[e];
        }
        s_prefix = prefix | ((uint32_t)(255 - 8 * tid - e) << shift);
        s_remaining = remaining - above;
      }
    }
    __syncthreads();
    prefix = s_prefix;
    remaining = s_remaining;
    mask |= 255u << shift;
    __syncthreads();
  }
  const uint32_t T = prefix;  // k-th largest key; `remaining` of the keys == T are taken

  // 3. stable compaction in index order: thread t owns the chunk [t*c, (t+1)*c)
  const int chunk = (d + blockDim.x - 1) / blockDim.x;
  const int i0 = min(d, tid * chunk), i1 = min(d, i0 + chunk);
  int n_eq = 0;
  for (int i = i0; i < i1; ++i) n_eq += (keys[i] == T);
  int tot;
  int eq_base = block_exclusive_scan(n_eq, warp_tot, &tot);
  int n_sel = 0;
  {
    int e = eq_base;
    for (int i = i0; i < i1; ++i) {
      const uint32_t key = keys[i];
      if (key > T) ++n_sel;
      else if (key == T) { if ((uint32_t)e < remaining) ++n_sel; ++e; }
    }
  }
  int pos = block_exclusive_scan(n_sel, warp_tot, &tot);
  {
    int e = eq_base;
    for (int i = i0; i < i1; ++i) {
      const uint32_t key = keys[i];
      bool take = false;
      if (key > T) take = true;
      else if (key == T) { take = (uint32_t)e < remaining; ++e; }
      if (take) {
        md.sel[pos] = i;
        if (md.sel_out) md.sel_out[pos] = i;
        ++pos;
      }
    }
  }
}


}  // namespace dion2
