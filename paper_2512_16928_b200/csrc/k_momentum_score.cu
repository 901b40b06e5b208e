// K1: fused momentum accumulation + l1 scoring.
//   Alg. 1 l.2  M <- M + G
//   Alg. 1 l.3  score = l1 norm of every row / column of the updated M
// HBM-bound single pass: read G, read M, write M (12 B per fp32 parameter).
#include "kernels.cuh"

namespace dion2 {

// ------------------------------------------------------------------ rows mode
// One warp per row; a persistent grid strides over the flattened rows of all
// row-mode matrices.  Score = per-lane sequential sum, then a fixed xor-tree:
// deterministic run to run.
template <bool kBf16G>
__device__ __forceinline__ float row_pass(const MatDesc& md, int64_t r, int lane) {
  float* __restrict__ Mrow = md.M + r * md.ld;
  const int64_t n = md.cols;
  float acc = 0.f;
  if (md.vec4) {
    const int64_t n4 = n >> 2;
    float4* M4 = reinterpret_cast<float4*>(Mrow);
    constexpr int U = 4;
    int64_t j = lane;
    for (; j + 32 * (U - 1) < n4; j += 32 * U) {
      float4 m[U], g[U];
#pragma unroll
      for (int u = 0; u < U; ++u) m[u] = M4[j + 32 * u];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if constexpr (kBf16G) {
          const uint2 raw = __ldg(reinterpret_cast<const uint2*>(
                                      reinterpret_cast<const __nv_bfloat16*>(md.G) + r * md.ld) +
                                  (j + 32 * u));
          const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(&raw.x);
          const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&raw.y);
          g[u] = make_float4(__low2float(lo), __high2float(lo), __low2float(hi), __high2float(hi));
        } else {
          g[u] = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(md.G) + r * md.ld) + (j + 32 * u));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        m[u].x += g[u].x; m[u].y += g[u].y; m[u].z += g[u].z; m[u].w += g[u].w;
        M4[j + 32 * u] = m[u];
        acc += fabsf(m[u].x) + fabsf(m[u].y) + fabsf(m[u].z) + fabsf(m[u].w);
      }
    }
    for (; j < n4; j += 32) {
      float4 m = M4[j];
      float4 g;
      if constexpr (kBf16G) {
        const __nv_bfloat16* gr = reinterpret_cast<const __nv_bfloat16*>(md.G) + r * md.ld + 4 * j;
        g = make_float4(bf16_to_f(gr[0]), bf16_to_f(gr[1]), bf16_to_f(gr[2]), bf16_to_f(gr[3]));
      } else {
        g = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(md.G) + r * md.ld) + j);
      }
      m.x += g.x; m.y += g.y; m.z += g.z; m.w += g.w;
      M4[j] = m;
      acc += fabsf(m.x) + fabsf(m.y) + fabsf(m.z) + fabsf(m.w);
    }
    for (int64_t t = 4 * n4 + lane; t < n; t += 32) {
      float g = kBf16G ? bf16_to_f(reinterpret_cast<const __nv_bfloat16*>(md.G)[r * md.ld + t])
                       : reinterpret_cast<const float*>(md.G)[r * md.ld + t];
      float m = Mrow[t] + g;
      Mrow[t] = m;
      acc += fabsf(m);
    }
  } else {
    for (int64_t t = lane; t < n; t += 32) {
      float g = kBf16G ? bf16_to_f(reinterpret_cast<const __nv_bfloat16*>(md.G)[r * md.ld + t])
                       : reinterpret_cast<const float*>(md.G)[r * md.ld + t];
      float m = Mrow[t] + g;
      Mrow[t] = m;
      acc += fabsf(m);
    }
  }
  return warp_sum(acc);
}

__global__ void __launch_bounds__(256) k_momentum_score_rows(const MatDesc* __restrict__ mats,
                                                             const int32_t* __restrict__ row_mats,
                                                             const int64_t* __restrict__ row_prefix, int n_row_mats,
                                                             int64_t total_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t gr = warp; gr < total_rows; gr += nwarps) {
    // locate the matrix: largest i with row_prefix[i] <= gr
    int lo = 0, hi = n_row_mats - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (row_prefix[mid] <= gr) lo = mid; else hi = mid - 1;
    }
    const MatDesc& md = mats[row_mats[lo]];
    const int64_t r = gr - row_prefix[lo];
    float s = md.grad_bf16 ? row_pass<true>(md, r, lane) : row_pass<false>(md, r, lane);
    if (lane == 0) md.scores[r] = s;
  }
}

// ------------------------------------------------------------------ cols mode
// Block = kColRB (256) rows x 256 columns; thread (ty in [0,4), tx in [0,64)) owns 4
// column slots and rows ty, ty+4, ...; a fixed-order smem reduce over ty gives
// one partial per (row block, column).  K2 sums the partials in row-block
// order: no float atomics anywhere.
constexpr int kColRB = kColRowBlock;
constexpr int kColCB = 256;

template <bool kBf16G>
__device__ __forceinline__ void col_tile(const MatDesc& md, int rb, int cb, float (*red)[kColCB]) {
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const int64_t r0 = (int64_t)rb * kColRB;
  const int64_t c0 = (int64_t)cb * kColCB;
  const int64_t rend = md.rows < r0 + kColRB ? md.rows : r0 + kColRB;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  const bool full4 = md.vec4 && (c0 + tx * 4 + 3 < md.cols);
  if (full4) {
    const int64_t c = c0 + tx * 4;
#pragma unroll 4
    for (int64_t r = r0 + ty; r < rend; r += 4) {
      float4* mp = reinterpret_cast<float4*>(md.M + r * md.ld + c);
      float4 m = *mp, g;
      if constexpr (kBf16G) {
        const uint2 raw = __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(md.G) + r * md.ld + c));
        const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(&raw.x);
        const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&raw.y);
        g = make_float4(__low2float(lo), __high2float(lo), __low2float(hi), __high2float(hi));
      } else {
        g = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(md.G) + r * md.ld + c));
      }
      m.x += g.x; m.y += g.y; m.z += g.z; m.w += g.w;
      *mp = m;
      acc[0] += fabsf(m.x); acc[1] += fabsf(m.y); acc[2] += fabsf(m.z); acc[3] += fabsf(m.w);
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) red[ty][tx * 4 + s] = acc[s];
  } else {
    // scalar slots: column c0 + tx*4 + s (same slot map as above)
    for (int64_t r = r0 + ty; r < rend; r += 4) {
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int64_t c = c0 + tx * 4 + s;
        if (c < md.cols) {
          float g = kBf16G ? bf16_to_f(reinterpret_cast<const __nv_bfloat16*>(md.G)[r * md.ld + c])
                           : reinterpret_cast<const float*>(md.G)[r * md.ld + c];
          float m = md.M[r * md.ld + c] + g;
          md.M[r * md.ld + c] = m;
          acc[s] += fabsf(m);
        }
      }
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) red[ty][tx * 4 + s] = acc[s];
  }
  __syncthreads();
  {
    const int c = threadIdx.x;  // 256 threads cover the 256 columns of the tile
    const int64_t col = c0 + c;
    if (col < md.cols) {
      float v = ((red[0][c] + red[1][c]) + red[2][c]) + red[3][c];
      md.col_partials[(int64_t)rb * md.cols + col] = v;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_momentum_score_cols(const MatDesc* __restrict__ mats,
                                                             const int32_t* __restrict__ col_mats,
                                                             const int64_t* __restrict__ tile_prefix, int n_col_mats,
                                                             int64_t total_tiles) {
  __shared__ float red[4][kColCB];
  for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
    int lo = 0, hi = n_col_mats - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (tile_prefix[mid] <= t) lo = mid; else hi = mid - 1;
    }
    const MatDesc& md = mats[col_mats[lo]];
    const int64_t local = t - tile_prefix[lo];
    const int cbs = (int)((md.cols + kColCB - 1) / kColCB);
    const int rb = (int)(local / cbs), cb = (int)(local % cbs);
    if (md.grad_bf16) col_tile<true>(md, rb, cb, red);
    else col_tile<false>(md, rb, cb, red);
  }
}

// ------------------------------------------------------------------ cols mode, M stored transposed
// M^T (cols x rows) += G^T through a 32 x 32 shared-memory transpose of the row-major G;
// the column l1 score of M is the row sum of M^T.  Unit = (block of kColRB rows of M,
// 32 columns): warp w owns columns j0 + 4w .. 4w+3 and accumulates their |M| over the
// block; one partial per (row block, column) exactly like the row-major kernel.
template <bool kBf16G>
__device__ __forceinline__ float load_g(const MatDesc& md, int64_t i, int64_t j) {
  if constexpr (kBf16G) return bf16_to_f(reinterpret_cast<const __nv_bfloat16*>(md.G)[i * md.ld + j]);
  else return __ldg(reinterpret_cast<const float*>(md.G) + i * md.ld + j);
}

template <bool kBf16G>
__device__ __forceinline__ void col_tile_mt(const MatDesc& md, int rb, int cb, float (*gs)[33]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t j0 = (int64_t)cb * 32;
  const int64_t ib = (int64_t)rb * kColRB;
  const int64_t ie = md.rows < ib + kColRB ? md.rows : ib + kColRB;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t i0 = ib; i0 < ie; i0 += 32) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t gi = i0 + 4 * w + r, gj = j0 + lane;
      gs[4 * w + r][lane] = (gi < ie && gj < md.cols) ? load_g<kBf16G>(md, gi, gj) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t j = j0 + 4 * w + r, i = i0 + lane;
      if (j < md.cols && i < ie) {
        float* p = md.M + j * md.ldm + i;
        const float m = *p + gs[lane][4 * w + r];
        *p = m;
        acc[r] += fabsf(m);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const float s = warp_sum(acc[r]);
    const int64_t j = j0 + 4 * w + r;
    if (lane == 0 && j < md.cols) md.col_partials[(int64_t)rb * md.cols + j] = s;
  }
}

// Vectorised variant (16-B aligned rows): 64 x 64 tiles through a [64][65] shared transpose.
// Lane = (g = lane / 8, c8 = lane % 8) in both phases: warp w moves rows 8 w + 4 jg + g
// (jg = 0, 1) and float4 chunks c8 + 8 h (h = 0, 1), so every instruction covers 4 rows x
// 128 contiguous bytes, and the shared accesses (row + column) mod 32 hit 32 distinct banks
// (scalar stores of G rows, column reads for M^T rows).  All loads of a tile are issued
// before the barrier.
template <bool kBf16G>
__device__ __forceinline__ float4 load_g4(const MatDesc& md, int64_t i, int64_t j) {
  if constexpr (kBf16G) {
    const uint2 raw = __ldcs(reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(md.G) + i * md.ld + j));
    const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(&raw.x);
    const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&raw.y);
    return make_float4(__low2float(lo), __high2float(lo), __low2float(hi), __high2float(hi));
  } else {
    return __ldcs(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(md.G) + i * md.ld + j));
  }
}

template <bool kBf16G>
__device__ __forceinline__ void col_tile_mt_v4(const MatDesc& md, int rb, int cb, float (*gs)[65]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 3, c8 = lane & 7;
  const int64_t j0 = (int64_t)cb * 64;
  const int64_t ib = (int64_t)rb * kColRB;
  const int64_t ie = md.rows < ib + kColRB ? md.rows : ib + kColRB;
  float acc[2] = {0.f, 0.f};  // |M| over the block's rows, M^T rows j0 + 8w + 4jg + g
  // bf16 G with 16-B aligned rows: each thread loads 8 consecutive columns (8 c8 .. +7) of a
  // row instead of two 4-column chunks 32 apart; the G tile column of slot u follows
  const bool g16 = kBf16G && (reinterpret_cast<uintptr_t>(md.G) % 16 == 0) && (md.ld % 8 == 0);
  auto gcol = [&](int u) { return g16 ? 8 * c8 + 4 * (u & 1) : 4 * (c8 + 8 * (u & 1)); };
  for (int64_t i0 = ib; i0 < ie; i0 += 64) {
    float4 gv[4], mv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // G row i0 + 8w + 4(u>>1) + g, columns gcol(u) .. +3
      const int64_t i = i0 + 8 * w + 4 * (u >> 1) + g, j = j0 + gcol(u);
      if (kBf16G && g16 && (u & 1)) continue;  // loaded with its even partner below
      if (kBf16G && g16 && i < ie && j + 7 < md.cols) {
        // bf16 G: one 16-B load = 8 columns (both halves), 128 contiguous bytes per row per warp
        const uint4 raw = __ldcs(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(md.G) +
                                                                i * md.ld + j));
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
        gv[u] = make_float4(__low2float(h[0]), __high2float(h[0]), __low2float(h[1]), __high2float(h[1]));
        gv[u + 1] = make_float4(__low2float(h[2]), __high2float(h[2]), __low2float(h[3]), __high2float(h[3]));
      } else if (!(kBf16G && g16) && i < ie && j + 3 < md.cols) {
        gv[u] = load_g4<kBf16G>(md, i, j);
      } else {
        const int nh = (kBf16G && g16) ? 2 : 1;  // bf16 16-B path: this slot covers both halves
        for (int hh = 0; hh < nh; ++hh) {
          float4& t = gv[u + hh];
          t = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int e = 0; e < 4; ++e)
            if (i < ie && j + 4 * hh + e < md.cols) (&t.x)[e] = load_g<kBf16G>(md, i, j + 4 * hh + e);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // M^T row j0 + 8w + 4(u>>1) + g, columns i0 + 4(c8 + 8(u&1)) .. +3
      const int64_t j = j0 + 8 * w + 4 * (u >> 1) + g, i = i0 + 4 * (c8 + 8 * (u & 1));
      mv[u] = (j < md.cols && i + 3 < ie) ? *reinterpret_cast<const float4*>(md.M + j * md.ldm + i)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
      if (j < md.cols && i < ie && i + 3 >= ie)
        for (int e = 0; e < 4; ++e)
          if (i + e < ie) (&mv[u].x)[e] = md.M[j * md.ldm + i + e];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = 8 * w + 4 * (u >> 1) + g, c = gcol(u);
      gs[r][c + 0] = gv[u].x;
      gs[r][c + 1] = gv[u].y;
      gs[r][c + 2] = gv[u].z;
      gs[r][c + 3] = gv[u].w;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int jl = 8 * w + 4 * (u >> 1) + g, il = 4 * (c8 + 8 * (u & 1));
      const int64_t j = j0 + jl, i = i0 + il;
      float* e = &mv[u].x;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        e[q] += gs[il + q][jl];  // G^T element (j, i + q)
        acc[u >> 1] += (i + q < ie) ? fabsf(e[q]) : 0.f;
      }
      if (j < md.cols) {
        if (i + 3 < ie) *reinterpret_cast<float4*>(md.M + j * md.ldm + i) = mv[u];
        else
          for (int q = 0; q < 4; ++q)
            if (i + q < ie) md.M[j * md.ldm + i + q] = e[q];
      }
    }
    __syncthreads();
  }
  // reduce the 8 lanes (c8) that share an M^T row, in a fixed xor-tree order
#pragma unroll
  for (int jg = 0; jg < 2; ++jg) {
    float s = acc[jg];
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const int64_t j = j0 + 8 * w + 4 * jg + g;
    if (c8 == 0 && j < md.cols) md.col_partials[(int64_t)rb * md.cols + j] = s;
  }
}

__global__ void __launch_bounds__(256, 4) k_momentum_score_cols_mt(const MatDesc* __restrict__ mats,
                                                                const int32_t* __restrict__ col_mats,
                                                                const int64_t* __restrict__ tile_prefix,
                                                                int n_col_mats, int64_t total_tiles) {
  __shared__ float gs[64][65];
  for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
    int lo = 0, hi = n_col_mats - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (tile_prefix[mid] <= t) lo = mid; else hi = mid - 1;
    }
    const MatDesc& md = mats[col_mats[lo]];
    const int64_t local = t - tile_prefix[lo];
    // units: (row block, 64 columns); unaligned rows take two scalar 32-column halves
    // column-block-major: consecutive blocks take consecutive row blocks of the same 64
    // columns, so together they stream whole M^T rows (2/3 of the traffic) page by page
    const int rbs = (int)((md.rows + kColRB - 1) / kColRB);
    const int cb = (int)(local / rbs), rb = (int)(local % rbs);
    if (md.vec4) {
      if (md.grad_bf16) col_tile_mt_v4<true>(md, rb, cb, gs);
      else col_tile_mt_v4<false>(md, rb, cb, gs);
    } else {
      float(*g33)[33] = reinterpret_cast<float(*)[33]>(&gs[0][0]);
      for (int h = 0; h < 2; ++h) {
        if (md.grad_bf16) col_tile_mt<true>(md, rb, 2 * cb + h, g33);
        else col_tile_mt<false>(md, rb, 2 * cb + h, g33);
      }
    }
  }
}

// ------------------------------------------------------------------ cols mode, M^T, cp.async pipeline
// Same unit decomposition and column-block-major order as k_momentum_score_cols_mt (unit =
// 256 rows of M x 64 columns = four 64 x 64 sub-tiles), for fp32 G on aligned, whole tiles.
// Every sub-tile's G tile and M^T tile (16 KB each) are copied global -> shared with 16-byte
// cp.async S - 1 sub-tiles ahead (across unit boundaries), so loads stay in flight while the
// CTA transposes and stores: one barrier per sub-tile, no registers held by loads.
// G's 16-byte chunk cj of tile row r sits at chunk cj ^ ((r >> 2) & 7): the transposed reads
// (lane = (g, c8) -> G rows 4 c8 + q, column 4 jb + g) then hit 32 distinct banks.
namespace {
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

struct MtUnit {
  const MatDesc* md;
  int64_t i0, j0;  // first row of M (column of M^T), first column of M (row of M^T)
  int rb;
};

__device__ __forceinline__ MtUnit mt_unit(const MatDesc* __restrict__ mats, const int32_t* __restrict__ col_mats,
                                          const int64_t* __restrict__ tile_prefix, int n_col_mats, int64_t u) {
  int lo = 0, hi = n_col_mats - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tile_prefix[mid] <= u) lo = mid; else hi = mid - 1;
  }
  MtUnit r;
  r.md = &mats[col_mats[lo]];
  const int64_t local = u - tile_prefix[lo];
  const int rbs = (int)(r.md->rows / kColRB);
  const int cb = (int)(local / rbs);
  r.rb = (int)(local % rbs);
  r.i0 = (int64_t)r.rb * kColRB;
  r.j0 = (int64_t)cb * 64;
  return r;
}
}  // namespace

// bf16 G: the G tile is 64 x 64 bf16 (8 KB, 8 chunks of 8 columns per row), chunk cj of row r
// at cj ^ ((r >> 2) & 7): a warp's transposed reads then touch 16 distinct words, two lanes each.
template <int S, bool kBf16>
__global__ void __launch_bounds__(256) k_momentum_score_cols_mt_pipe(const MatDesc* __restrict__ mats,
                                                                     const int32_t* __restrict__ col_mats,
                                                                     const int64_t* __restrict__ tile_prefix,
                                                                     int n_col_mats, int64_t total_units) {
  constexpr int kGB = kBf16 ? 8192 : 16384;  // G tile bytes
  constexpr int kStageB = kGB + 16384;       // + M^T tile
  extern __shared__ float4 sm4[];
  uint8_t* sm = reinterpret_cast<uint8_t*>(sm4);  // [S][G tile | M^T 64 x 64 fp32]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 3, c8 = lane & 7;
  if (blockIdx.x >= total_units) return;
  const int64_t my_units = (total_units - 1 - blockIdx.x) / gridDim.x + 1;
  const int64_t n_st = my_units * 4;

  MtUnit iu = mt_unit(mats, col_mats, tile_prefix, n_col_mats, blockIdx.x);  // issue cursor's unit
  int64_t iu_idx = 0;
  auto issue = [&](int64_t st) {
    const int64_t ui = st >> 2;
    if (ui != iu_idx) {
      iu = mt_unit(mats, col_mats, tile_prefix, n_col_mats, blockIdx.x + ui * gridDim.x);
      iu_idx = ui;
    }
    const MatDesc& md = *iu.md;
    const int64_t i0 = iu.i0 + (st & 3) * 64;
    uint8_t* gdst = sm + (int)(st % S) * kStageB;
    float* mdst = reinterpret_cast<float*>(gdst + kGB);
    if constexpr (kBf16) {
      const __nv_bfloat16* G = reinterpret_cast<const __nv_bfloat16*>(md.G);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int c = tid + 256 * q, r = c >> 3, cj = c & 7;
        cp_async16(reinterpret_cast<float*>(gdst + r * 128 + ((cj ^ ((r >> 2) & 7)) << 4)),
                   reinterpret_cast<const float*>(G + (i0 + r) * md.ld + iu.j0 + 8 * cj));
      }
    } else {
      const float* G = reinterpret_cast<const float*>(md.G);
      float* gf = reinterpret_cast<float*>(gdst);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = tid + 256 * q, r = c >> 4, cj = c & 15;
        cp_async16(gf + r * 64 + ((cj ^ ((r >> 2) & 7)) << 2), G + (i0 + r) * md.ld + iu.j0 + 4 * cj);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = tid + 256 * q, r = c >> 4, cj = c & 15;
      cp_async16(mdst + r * 64 + 4 * cj, md.M + (iu.j0 + r) * md.ldm + i0 + 4 * cj);
    }
  };
#pragma unroll
  for (int s0 = 0; s0 < S - 1; ++s0) {
    if (s0 < n_st) issue(s0);
    cp_async_commit();
  }
  MtUnit cu = mt_unit(mats, col_mats, tile_prefix, n_col_mats, blockIdx.x);  // compute cursor's unit
  float acc[2] = {0.f, 0.f};
  for (int64_t st = 0; st < n_st; ++st) {
    cp_async_wait<S - 2>();
    __syncthreads();
    if (st + S - 1 < n_st) issue(st + S - 1);
    cp_async_commit();
    if ((st & 3) == 0 && st) cu = mt_unit(mats, col_mats, tile_prefix, n_col_mats, blockIdx.x + (st >> 2) * gridDim.x);
    const MatDesc& md = *cu.md;
    const int64_t i0 = cu.i0 + (st & 3) * 64;
    const uint8_t* gs = sm + (int)(st % S) * kStageB;
    const float* ms = reinterpret_cast<const float*>(gs + kGB);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int jl = 8 * w + 4 * (u >> 1) + g, il = 4 * (c8 + 8 * (u & 1));
      float4 m = *reinterpret_cast<const float4*>(ms + jl * 64 + il);
      float e[4];
      if constexpr (kBf16) {
        // (il + q) >> 2 == il >> 2; chunk jl >> 3, element jl & 7
        const int off = (((jl >> 3) ^ ((il >> 2) & 7)) << 4) + (jl & 7) * 2;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          e[q] = __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(gs + (il + q) * 128 + off));
      } else {
        const float* gf = reinterpret_cast<const float*>(gs);
        const int off = (((jl >> 2) ^ ((il >> 2) & 7)) << 2) + (jl & 3);
#pragma unroll
        for (int q = 0; q < 4; ++q) e[q] = gf[(il + q) * 64 + off];
      }
      m.x += e[0];
      m.y += e[1];
      m.z += e[2];
      m.w += e[3];
      *reinterpret_cast<float4*>(md.M + (cu.j0 + jl) * md.ldm + i0 + il) = m;
      acc[u >> 1] += fabsf(m.x) + fabsf(m.y) + fabsf(m.z) + fabsf(m.w);
    }
    if ((st & 3) == 3) {
      // unit done: reduce the 8 lanes (c8) sharing an M^T row in a fixed xor-tree order
#pragma unroll
      for (int jg = 0; jg < 2; ++jg) {
        float v = acc[jg];
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (c8 == 0) md.col_partials[(int64_t)cu.rb * md.cols + cu.j0 + 8 * w + 4 * jg + g] = v;
        acc[jg] = 0.f;
      }
    }
  }
  cp_async_wait<0>();
}

template <int S, bool kBf16>
constexpr size_t mt_pipe_smem() { return (size_t)S * ((kBf16 ? 8192 : 16384) + 16384); }

template <int S, bool B>
static void mt_pipe_launch(int blocks, cudaStream_t s, const MatDesc* mats, const int32_t* col_mats,
                           const int64_t* tile_prefix, int n_col_mats, int64_t total_units) {
  k_momentum_score_cols_mt_pipe<S, B><<<blocks, 256, mt_pipe_smem<S, B>(), s>>>(mats, col_mats, tile_prefix,
                                                                                n_col_mats, total_units);
}
template <int S, bool B>
static int mt_pipe_attr() {
  cudaFuncSetAttribute(k_momentum_score_cols_mt_pipe<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)mt_pipe_smem<S, B>());
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_momentum_score_cols_mt_pipe<S, B>, 256, mt_pipe_smem<S, B>());
  return nb;
}

void launch_momentum_score_cols_mt_pipe(int stages, bool bf16, int blocks, cudaStream_t s, const MatDesc* mats,
                                        const int32_t* col_mats, const int64_t* tile_prefix, int n_col_mats,
                                        int64_t total_units) {
  switch (stages * 2 + (bf16 ? 1 : 0)) {
    case 4: mt_pipe_launch<2, false>(blocks, s, mats, col_mats, tile_prefix, n_col_mats, total_units); break;
    case 5: mt_pipe_launch<2, true>(blocks, s, mats, col_mats, tile_prefix, n_col_mats, total_units); break;
    case 8: mt_pipe_launch<4, false>(blocks, s, mats, col_mats, tile_prefix, n_col_mats, total_units); break;
    case 9: mt_pipe_launch<4, true>(blocks, s, mats, col_mats, tile_prefix, n_col_mats, total_units); break;
    case 7: mt_pipe_launch<3, true>(blocks, s, mats, col_mats, tile_prefix, n_col_mats, total_units); break;
    default: mt_pipe_launch<3, false>(blocks, s, mats, col_mats, tile_prefix, n_col_mats, total_units); break;
  }
}

int momentum_score_cols_mt_pipe_attrs(int stages, bool bf16) {
  switch (stages * 2 + (bf16 ? 1 : 0)) {
    case 4: return mt_pipe_attr<2, false>();
    case 5: return mt_pipe_attr<2, true>();
    case 8: return mt_pipe_attr<4, false>();
    case 9: return mt_pipe_attr<4, true>();
    case 7: return mt_pipe_attr<3, true>();
    default: return mt_pipe_attr<3, false>();
  }
}

}  // namespace dion2
