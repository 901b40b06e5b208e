// dion2_api.cu -- host runtime of the Dion2 step: config validation, the
// per-(shapes, config, workspace) plan (axis/k resolution, wide orientation,
// NS shape groups, workspace carve-up, TMA tensor maps, launch list), and the
// C ABI declared in include/dion2.h.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "runtime.h"

using namespace dion2;
using namespace dion2rt;

namespace dion2rt {

const char* kPhaseNames[kNumPhases] = {"momentum_score", "select",       "gather",       "norm",
                                       "ns_gram",        "ns_poly",      "ns_apply",     "scatter",
                                       "full_decay",     "gather_rows",  "gather_cols",  "scatter_rows",
                                       "scatter_cols",   "ns_mul",       "momentum_score_mt"};

std::mutex g_mu;
int g_sm_count = 0;

int sm_count() {
  if (g_sm_count <= 0) {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      g_sm_count = v;
    else
      cudaGetLastError();  // no device visible (host-only size query): assume B200's 148
  }
  return g_sm_count > 0 ? g_sm_count : 148;
}
bool g_attr_done = false;
int32_t g_last_launches = 0;

// ------------------------------------------------------------------ phase timing
bool g_timing = false;
std::vector<TimedLaunch> g_timed;
std::vector<cudaEvent_t> g_event_pool;
cudaEvent_t take_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// ------------------------------------------------------------------ helpers

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D bf16 tensor map over [count][rows][cols] (row-major), SWIZZLE_128B, box {64, box_rows, 1}.
bool make_map(CUtensorMap* m, const void* base, int64_t cols, int64_t rows, int64_t count, int box_cols, int box_rows,
              CUtensorMapSwizzle swz) {
  auto enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)count};
  cuuint64_t strides[2] = {(cuuint64_t)(cols * 2), (cuuint64_t)(cols * rows * 2)};
  cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3-D bf16 tensor map over `count` row-major [rows][cols] arrays spaced zstride_bytes apart
// (the distributed step's rank pieces: piece size rounded up to 256 B).
bool make_map_strided(CUtensorMap* m, const void* base, int64_t cols, int64_t rows, int64_t count,
                      int64_t zstride_bytes, int box_cols, int box_rows, CUtensorMapSwizzle swz) {
  auto enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)count};
  cuuint64_t strides[2] = {(cuuint64_t)(cols * 2), (cuuint64_t)zstride_bytes};
  cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

std::vector<dion2_matrix> storage_view(const dion2_matrix* mats, int n) {
  std::vector<dion2_matrix> v(mats, mats + n);
  for (auto& m : v)
    if (m.storage_transposed == 1) std::swap(m.rows, m.cols);
  return v;
}

int validate_config(const dion2_config* c) {
  if (!c) return DION2_EINVAL_CONFIG;
  if (!(c->alpha > 0.f && c->alpha <= 1.f)) return DION2_EINVAL_CONFIG;
  if (!(c->mu >= 0.f && c->mu < 1.f)) return DION2_EINVAL_CONFIG;
  if (!(c->lr >= 0.f) || !std::isfinite(c->lr)) return DION2_EINVAL_CONFIG;
  if (c->ns_steps < 1 || c->ns_steps > DION2_MAX_NS_STEPS) return DION2_EINVAL_CONFIG;
  if (!(c->ns_eps > 0.f)) return DION2_EINVAL_CONFIG;
  for (int t = 0; t < c->ns_steps; ++t)
    for (int j = 0; j < 3; ++j)
      if (!std::isfinite(c->ns_coeffs[t][j])) return DION2_EINVAL_CONFIG;
  if (c->axis < 0 || c->axis > 2) return DION2_EINVAL_CONFIG;
  if (c->select != DION2_SELECT_L1 && c->select != DION2_SELECT_RANDOM) return DION2_EINVAL_CONFIG;
  if (c->precision != DION2_NS_BF16 && c->precision != DION2_NS_FP32) return DION2_EINVAL_CONFIG;
  if (c->grad_dtype != DION2_DT_F32 && c->grad_dtype != DION2_DT_BF16) return DION2_EINVAL_CONFIG;
  if (c->w_dtype != DION2_DT_F32 && c->w_dtype != DION2_DT_BF16) return DION2_EINVAL_CONFIG;
  if (c->decay_mode < 0 || c->decay_mode > 1) return DION2_EINVAL_CONFIG;
  if (c->scale_mode < 0 || c->scale_mode > 1) return DION2_EINVAL_CONFIG;
  if (c->ns_form < DION2_NS_FORM_AUTO || c->ns_form > DION2_NS_FORM_GRAM || (c->reserved0 & ~(DION2_FLAG_LR_DEVICE | DION2_FLAG_DIST_DIRECT)) != 0)
    return DION2_EINVAL_CONFIG;
  return DION2_OK;
}

int validate_shape(const dion2_matrix& m, bool need_ptrs) {
  if (m.rows < 1 || m.cols < 1 || m.ld < m.cols) return DION2_EINVAL_SHAPE;
  if (m.rows > (1ll << 31) - 1 || m.cols > (1ll << 31) - 1) return DION2_EINVAL_SHAPE;
  if (need_ptrs && (!m.W || !m.M || !m.G)) return DION2_EINVAL_SHAPE;
  if ((m.storage_transposed != 0 && m.storage_transposed != 1) || (m.m_transposed != 0 && m.m_transposed != 1))
    return DION2_EINVAL_SHAPE;
  if (m.m_transposed && m.ldm < m.rows) return DION2_EINVAL_SHAPE;
  return DION2_OK;
}

// ------------------------------------------------------------------ plan

std::map<std::string, std::unique_ptr<Plan>> g_plans;
uint64_t g_next_plan_id = 1;

std::string plan_key(const dion2_matrix* mats, int n, const dion2_config* c, void* ws) {
  std::string k;
  auto put = [&](const void* p, size_t s) { k.append(reinterpret_cast<const char*>(p), s); };
  put(&n, sizeof n);
  put(&ws, sizeof ws);
  for (int i = 0; i < n; ++i) {
    put(&mats[i].rows, 8);
    put(&mats[i].cols, 8);
    put(&mats[i].ld, 8);
    put(&mats[i].m_transposed, 4);  // selects the gather / K1 paths and the sum-of-squares layout
    put(&mats[i].storage_transposed, 4);
  }
  put(&c->alpha, 4);
  put(&c->ns_steps, 4);
  put(c->ns_coeffs, sizeof(float) * 3 * c->ns_steps);
  put(&c->axis, 4);
  put(&c->select, 4);
  put(&c->precision, 4);
  put(&c->grad_dtype, 4);
  put(&c->w_dtype, 4);
  put(&c->decay_mode, 4);
  put(&c->scale_mode, 4);
  put(&c->ns_form, 4);
  k += env_key();
  return k;
}

// kernel-variant switches read at plan build (tests and measurements flip them): part of
// every plan-cache key
std::string env_key() {
  std::string k;
  for (const char* v : {"DION2_NS_PAIR", "DION2_NS_SYM", "DION2_NS_SERPENTINE", "DION2_NS_UPPER",
                        "DION2_GRAM_SPLITK", "DION2_DIST_CHUNKS"}) {
    const char* e = getenv(v);
    k.append(e ? e : "-");
    k.push_back('|');
  }
  return k;
}

// Build the plan layout (no device work).  ws may be null (size query).
int build_layout(Plan& P, const dion2_matrix* mats, int n, const dion2_config* c) {
  P.n = n;
  P.bf16_ns = c->precision == DION2_NS_BF16;
  P.ns_steps = c->ns_steps;
  P.mp.resize(n);
  const size_t xel = P.bf16_ns ? 2 : 4;
  std::map<std::tuple<int, int, int>, int> gidx;
  for (int i = 0; i < n; ++i) {
    const dion2_matrix& m = mats[i];
    MatPlan& q = P.mp[i];
    // m is the storage view (storage_view()); the paper's rules apply to the LOGICAL matrix
    const int64_t rows = m.rows, cols = m.cols;
    const bool st = m.storage_transposed == 1;
    const int64_t lrows = st ? cols : rows, lcols = st ? rows : cols;
    int laxis = c->axis == DION2_AXIS_AUTO ? (lrows <= lcols ? DION2_AXIS_ROWS : DION2_AXIS_COLS) : c->axis;
    int axis = st ? (laxis == DION2_AXIS_ROWS ? DION2_AXIS_COLS : DION2_AXIS_ROWS) : laxis;
    q.axis = axis;
    q.d = (int)(axis == DION2_AXIS_ROWS ? rows : cols);
    q.o = (int)(axis == DION2_AXIS_ROWS ? cols : rows);
    if (q.d > DION2_MAX_SELECT_DIM) return DION2_EINVAL_SHAPE;
    int64_t k = (int64_t)std::floor((double)c->alpha * (double)q.d + 0.5);  // reading R7
    k = std::max<int64_t>(1, std::min<int64_t>(k, q.d));
    q.k = (int)k;
    q.sr = axis == DION2_AXIS_ROWS ? q.k : (int)rows;
    q.sc = axis == DION2_AXIS_ROWS ? (int)cols : q.k;
    q.transposed = q.sr > q.sc;  // wide orientation (reading R4)
    q.p = std::min(q.sr, q.sc);
    q.q = std::max(q.sr, q.sc);
    q.p_pad = (int)align_up(q.p, 256);  // 256-row CTA-pair tiles
    q.q_pad = (int)align_up(q.q, 256);
    if (c->scale_mode == 0) q.fan_sqrt = (float)std::sqrt((double)lrows / (double)lcols);  // Alg. 1 l.6
    else q.fan_sqrt = (float)(st ? std::sqrt((double)q.sc / (double)q.sr) : std::sqrt((double)q.sr / (double)q.sc));
    q.rowblocks = (int)ceil_div(rows, kColRowBlock);
    // gather tiles cover the padded extent of S (wide(S_pad) = X_pad) so K3 also
    // rewrites X's zero padding every step
    q.sa_pad = q.transposed ? q.q_pad : q.p_pad;
    q.sb_pad = q.transposed ? q.p_pad : q.q_pad;
    // gather/scatter path: streaming kernels for the two orientations auto mode produces
    if (axis == DION2_AXIS_ROWS && !q.transposed && P.bf16_ns) q.path = 1;
    else if (axis == DION2_AXIS_COLS && q.transposed && P.bf16_ns && q.k <= kMaxColKFast) q.path = 2;
    else q.path = 0;
    q.mt = m.m_transposed ? 1 : 0;
    // transposed M: column mode with X = S^T (k <= rows), bf16; the gather is the row path on M^T
    if (q.mt && !(axis == DION2_AXIS_COLS && q.transposed && P.bf16_ns)) return DION2_EUNSUPPORTED;
    // the cols streaming scatter takes larger k than the gather (8-row O tiles above k = 1024)
    q.spath = (axis == DION2_AXIS_COLS && q.transposed && P.bf16_ns && q.k <= kMaxColKScatter) ? 2 : q.path;
    const bool generic = (q.path == 0 && !q.mt) || q.spath == 0;  // a generic gather or scatter needs tiles
    q.ga = generic ? (int)ceil_div(q.sa_pad, kTileA) : 0;
    q.gb = generic ? (int)ceil_div(q.sb_pad, kTileB) : 0;
    q.n_sumsq = (q.path == 1 || q.mt) ? q.p_pad : (q.path == 0 ? q.ga * q.gb : q.q_pad / 32);
    // reading R25 / k_ns_small.cu: a short X (p <= kTinyP = 128 rows) under AUTO is evaluated in high precision
    q.tiny = (!P.no_tiny && P.bf16_ns && c->ns_form == DION2_NS_FORM_AUTO && q.p <= kTinyP) ? 1 : 0;
    auto key = std::make_tuple(q.p_pad, q.q_pad, q.tiny);
    auto it = gidx.find(key);
    if (it == gidx.end()) {
      Group g{};
      g.p_pad = q.p_pad;
      g.q_pad = q.q_pad;
      g.tiny = q.tiny;
      g.count = 0;
      gidx[key] = (int)P.groups.size();
      P.groups.push_back(g);
      it = gidx.find(key);
    }
    q.group = it->second;
    q.zi = P.groups[q.group].count++;
    P.groups[q.group].mats.push_back(i);
    P.max_d = std::max(P.max_d, q.d);
  }
  // ---- workspace carve-up
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 1), 256);
    return o;
  };
  P.off_status = take(16);
  P.off_bad = take(4 * (size_t)n);
  P.off_desc = take(sizeof(MatDesc) * n);
  P.off_rowmats = take(4 * (size_t)n);
  P.off_rowprefix = take(8 * (size_t)n);
  P.off_colmats = take(4 * (size_t)n);
  P.off_colprefix = take(8 * (size_t)n);
  P.off_mtmats = take(4 * (size_t)n);
  P.off_mtprefix = take(8 * (size_t)n);
  P.off_gprefix = take(4 * (size_t)n);
  for (int l = 0; l < 2; ++l) {
    P.off_flg_mats[l] = take(4 * (size_t)n);
    P.off_fls_mats[l] = take(4 * (size_t)n);
    P.off_fl_gprefix[l] = take(4 * (size_t)n);
    P.off_fl_sprefix[l] = take(4 * (size_t)n);
  }
  for (auto& g : P.groups) g.off_gmats = take(4 * (size_t)g.count);
  P.off_cf_mats = take(4 * (size_t)n);
  P.off_cf_prefix = take(8 * (size_t)n);
  P.off_tiny_list = take(4 * (size_t)n);
  P.off_nsscale = take(16 * (size_t)n);
  for (int i = 0; i < n; ++i) {
    MatPlan& q = P.mp[i];
    q.off_scores = take(4 * (size_t)q.d);
    q.off_partials = q.axis == DION2_AXIS_COLS ? take(4 * (size_t)q.rowblocks * (size_t)mats[i].cols) : 0;
    q.off_sel = take(4 * (size_t)q.k);
    q.off_sumsq = take(4 * (size_t)q.n_sumsq);
  }
  off = align_up(off, 4096);
  P.off_ns_begin = off;
  for (auto& g : P.groups) {
    const size_t xb = (size_t)g.count * g.p_pad * g.q_pad * xel;
    const size_t ab = (size_t)g.count * g.p_pad * g.p_pad * xel;
    g.off_X0 = off; off = align_up(off + xb, 4096);
    g.off_X1 = off; off = align_up(off + xb, 4096);
    g.off_A = off;  off = align_up(off + ab, 4096);
    g.off_B = off;  off = align_up(off + ab, 4096);
    // Gram-space form (reading R23): 16-bit hot path, wide X with q >= 2p (AUTO) or forced.
    // AUTO: fewer FLOPs on the padded shapes (q_pad >= 2 p_pad), or every member has q >= 2p;
    // and every member has p >= kGramMinP (R25: with fp16 X the direct form is the accurate one
    // for short X, 0.2-0.9% against up to 3.5% emulated at p <= 32)
    bool all_wide = true, all_tall_enough = true;
    for (int i : g.mats) {
      all_wide = all_wide && P.mp[i].q >= 2 * P.mp[i].p;
      // reading R25: the fp16 Gram matrix of a short X (p < 64 rows) carries too much of each
      // eigenvalue per entry -- AUTO keeps the direct form there
      all_tall_enough = all_tall_enough && P.mp[i].p >= kGramMinP;
    }
    g.gs = P.bf16_ns && !g.tiny && (c->ns_form == DION2_NS_FORM_GRAM ||
                         (c->ns_form == DION2_NS_FORM_AUTO && all_tall_enough &&
                          (g.q_pad >= 2 * g.p_pad || all_wide)));
    g.off_C = g.off_Q0 = g.off_Q1 = 0;
    if (g.gs) {
      g.off_C = off;  off = align_up(off + ab, 4096);
      g.off_Q0 = off; off = align_up(off + ab, 4096);
      g.off_Q1 = off; off = align_up(off + ab, 4096);
    }
  }
  // split-K for the gram launches (K = q_pad) when all their upper-triangle pair tiles
  // together cover at most half of the CTA pairs (few, large matrices: configs[4]); each
  // slice keeps >= 4 k-blocks.  The fp32 partials live after the NS buffers.
  P.gram_splitk = 1;
  P.off_splitk = 0;
  const char* pe = getenv("DION2_NS_PAIR");
  const char* se = getenv("DION2_GRAM_SPLITK");
  if (P.bf16_ns && !(pe && strcmp(pe, "none") == 0) && !(se && atoi(se) == 1)) {
    int64_t tt = 0;
    int min_kb = 1 << 30;
    for (auto& g : P.groups) {
      const int T = g.p_pad / 256;
      tt += (int64_t)g.count * T * (T + 1) / 2;
      min_kb = std::min(min_kb, g.q_pad / 64);
    }
    const int pairs = sm_count() / 2;  // the same value the size query and the step see
    if (tt > 0 && 2 * tt <= pairs) {
      int S = (int)std::min<int64_t>((pairs + tt - 1) / tt, min_kb / 4);
      if (se && atoi(se) > 1) S = std::min(atoi(se), min_kb);
      if (S > 1) {
        P.gram_splitk = S;
        P.off_splitk = off;
        off = align_up(off + (size_t)tt * S * 256 * 256 * 4, 4096);
      }
    }
  }
  P.off_ns_end = off;
  P.total = off + 4096;  // slack for base alignment
  return DION2_OK;
}



// Kind-5 launches (resident-A pair apply) count work in chunks of up to L consecutive 256-column
// blocks of one 256-row block: L = 8, halved while the launch has fewer than two chunks per CTA pair.
static void apply_chunks(NsParams& np) {
  const int pairs = sm_count() / 2;
  auto count = [&](int L) {
    int n = 0;
    for (int j = 0; j < np.ngroups; ++j) n += np.g[j].count * ((np.g[j].n_tiles + L - 1) / L) * np.g[j].m_tiles;
    return n;
  };
  int L = 8;
  while (L > 1 && count(L) < 2 * pairs) L /= 2;
  np.chunk_len = L;
  int base = 0;
  for (int j = 0; j < np.ngroups; ++j) {
    np.g[j].tile_base = base;
    base += np.g[j].count * ((np.g[j].n_tiles + L - 1) / L) * np.g[j].m_tiles;
  }
  np.total_tiles = base;
}

// Restart segments of the Gram-space form (reading R24): consecutive iterations [t0, t1) whose
// growth prod |a_t| stays <= kRestartGrowth share one p x p recursion; each later segment
// restarts from its X, formed explicitly by the previous segment's apply.  The default
// quintic (a = 3.4445) gives [0, 3) + [3, 5): Q's eigenvalues span at most a^3 / 0.68 ~ 60
// instead of a^5 / 0.68 ~ 700.
constexpr double kRestartGrowth = 64.0;
std::vector<std::pair<int, int>> ns_segments(const dion2_config* c, int T) {
  std::vector<std::pair<int, int>> v;
  int t0 = 0;
  double prod = 1.0;
  for (int t = 0; t < T; ++t) {
    const double a = std::max(1.0, std::fabs((double)c->ns_coeffs[t][0]));
    if (t > t0 && prod * a > kRestartGrowth) {
      v.push_back({t0, t});
      t0 = t;
      prod = 1.0;
    }
    prod *= a;
  }
  v.push_back({t0, T});
  return v;
}

// Launch list of the Gram-space Newton-Schulz form (readings R23, R24) for the groups with
// g.gs, per restart segment j (iterations t0 .. t1-1, Ts = t1 - t0) on Xin = X_{t0}:
//   gram   A   = s_j^2 Xin Xin^T                     (s_0 = s' of the prescaled X0; s_j = 1 after)
//   tl = 0 .. Ts-1 (t = t0 + tl):
//     poly   C   = a_t I + b_t A + c_t A A            (C of tl = 0 doubles as Q_1)
//     mul    Q_{tl+1} = C Q_tl (tl >= 1),  B = C A (tl < Ts-1)
//     mul    A   = C B                                (tl < Ts-1)
//   apply  Xout = s_j Q_Ts Xin                         (X_{t1}; the last segment's is X_T = O)
// Xin / Xout alternate between the X0 and X1 buffers.  Every p x p product is a polynomial in
// the segment's A, hence symmetric: upper-triangle pair tiles.  All operands and outputs are
// fp16 with fp32 accumulation; Q_Ts is written mirrored (the 1-SM apply reads it whole).
static int append_gram_space_launches(Plan& P, const dion2_config* c, void* ws, int pair_mode) {
  std::vector<int> gl;
  for (int gi = 0; gi < (int)P.groups.size(); ++gi)
    if (P.groups[gi].gs) gl.push_back(gi);
  if (gl.empty()) return DION2_OK;
  const float* scale_all = (const float*)at(ws, P.off_nsscale);
  const int T = P.ns_steps;
  struct Entry {
    int gi;
    void *a, *b, *out, *cin;
  };
  // one launch per kMaxGroups entries; kind: 3 = pair (sym p x p products, or apply under
  // DION2_NS_PAIR=all), 1 = 1-SM BN 256 (apply)
  const bool sym_on = !(getenv("DION2_NS_SYM") && atoi(getenv("DION2_NS_SYM")) == 0);
  const char* serp_env = getenv("DION2_NS_SERPENTINE");
  const bool serpentine = !serp_env || atoi(serp_env) != 0;
  unsigned flip = 0;
  // p x p buffers hold only their upper 256 x 256 tiles (the kernel reads lower k-blocks
  // transposed); Q_T, read by the 1-SM apply, is written mirrored.  DION2_NS_UPPER=0: mirror all.
  const bool upper_only = !(getenv("DION2_NS_UPPER") && atoi(getenv("DION2_NS_UPPER")) == 0) && sym_on;
  auto emit = [&](int phase, const std::vector<Entry>& es, float cacc, float cC, float diag, int scale_sel,
                  int in_f16, int out_f16, bool mirror_out = false) -> int {
    const bool apply = phase == PH_APPLY;
    for (size_t s0 = 0; s0 < es.size(); s0 += kMaxGroups) {
      const size_t s1 = std::min(es.size(), s0 + kMaxGroups);
      bool res_ok = apply && pair_mode == 1;
      for (size_t e = s0; e < s1; ++e) res_ok = res_ok && P.groups[es[e].gi].p_pad <= 64 * kMaxResidentKB;
      const bool pair = !apply || pair_mode == 2 || res_ok;
      const int MT = pair ? 256 : 128, BN = 256;
      Launch L{};
      L.phase = phase;
      L.bn = BN;
      L.kind = res_ok ? 5 : (pair ? 3 : 1);
      NsParams& np = L.tc.p;
      np.ngroups = (int)std::min<size_t>(kMaxGroups, es.size() - s0);
      np.ns_scale_all = scale_all;
      np.cacc = cacc; np.cC = cC; np.diag = diag; np.scale_sel = scale_sel;
      np.sym = (apply || !sym_on) ? 0 : 1;
      np.b_kmajor = apply ? 0 : 1;
      np.in_f16 = in_f16; np.out_f16 = out_f16;
      np.sym_in = (upper_only && !apply && phase != PH_GRAM) ? 1 : 0;
      np.no_mirror = (upper_only && !apply && !mirror_out) ? 1 : 0;
      // alternate the walk direction between consecutive p x p launches: a launch starts on the
      // matrices the previous one wrote last (still in L2)
      np.reverse = (!apply && serpentine) ? (int)(flip++ & 1) : 0;
      if (phase == PH_GRAM && pair && np.sym && P.gram_splitk > 1) {  // partials sized for sym tiles
        np.splitk = P.gram_splitk;
        np.partial = (float*)at(ws, P.off_splitk);
      }
      int tiles = 0;
      for (int j = 0; j < np.ngroups; ++j) {
        const Entry& e = es[s0 + j];
        const Group& g = P.groups[e.gi];
        const long long xs = (long long)g.p_pad * g.q_pad, as = (long long)g.p_pad * g.p_pad;
        const int K = phase == PH_GRAM ? g.q_pad : g.p_pad;
        NsGroup& G = np.g[j];
        G.count = g.count;
        G.gmats = (const int32_t*)tab(P, g.off_gmats);
        G.m_tiles = g.p_pad / MT;
        G.n_tiles = apply ? g.q_pad / BN : g.p_pad / BN;
        G.k_blocks = K / 64;
        G.a = e.a; G.a_mstride = phase == PH_GRAM ? xs : as; G.lda = K;
        G.b = e.b; G.b_mstride = (phase == PH_GRAM || apply) ? xs : as; G.ldb = apply ? g.q_pad : K;
        G.out = e.out; G.out_mstride = apply ? xs : as; G.out_ld = apply ? g.q_pad : g.p_pad;
        G.cin = e.cin; G.cin_mstride = e.cin ? as : 0; G.cin_ld = e.cin ? g.p_pad : 0;
        if (!make_map(&L.tc.mapA[j], e.a, K, g.p_pad, g.count, 64, 128)) return DION2_ECUDA;
        if (apply) {
          if (!make_map(&L.tc.mapB[j], e.b, g.q_pad, g.p_pad, g.count, 64, 64)) return DION2_ECUDA;
        } else {
          if (!make_map(&L.tc.mapB[j], e.b, K, g.p_pad, g.count, 64, 128)) return DION2_ECUDA;
        }
        if (!make_map(&L.tc.mapD[j], e.out, G.out_ld, g.p_pad, g.count, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
          return DION2_ECUDA;
        if (np.sym_in) {
          if (!make_map(&L.tc.mapAT[j], e.a, g.p_pad, g.p_pad, g.count, 64, 64)) return DION2_ECUDA;
          if (!make_map(&L.tc.mapBT[j], e.b, g.p_pad, g.p_pad, g.count, 64, 64)) return DION2_ECUDA;
        }
        G.tile_base = tiles;
        tiles += G.count * (np.sym ? G.m_tiles * (G.m_tiles + 1) / 2 : G.m_tiles * G.n_tiles);
      }
      np.total_tiles = tiles;
      np.b_is_a = np.b_kmajor ? 1 : 0;
      for (int j = 0; j < np.ngroups; ++j) np.b_is_a &= np.g[j].a == np.g[j].b ? 1 : 0;
      if (L.kind == 5) apply_chunks(np);
      P.ns_launches.push_back(L);
    }
    return DION2_OK;
  };
  auto X0 = [&](int gi) { return at(ws, P.groups[gi].off_X0); };
  auto X1 = [&](int gi) { return at(ws, P.groups[gi].off_X1); };
  auto Ab = [&](int gi) { return at(ws, P.groups[gi].off_A); };
  auto Bb = [&](int gi) { return at(ws, P.groups[gi].off_B); };
  auto Cb = [&](int gi, int t) { return t == 0 ? at(ws, P.groups[gi].off_Q0) : at(ws, P.groups[gi].off_C); };
  auto Qb = [&](int gi, int j) { return at(ws, (j & 1) ? P.groups[gi].off_Q0 : P.groups[gi].off_Q1); };  // Q_j, j >= 1
  int rc;
  std::vector<Entry> es;
  const std::vector<std::pair<int, int>> segs = ns_segments(c, T);
  for (size_t sg = 0; sg < segs.size(); ++sg) {
    const int t0 = segs[sg].first, Ts = segs[sg].second - t0;
    auto Xin = [&](int gi) { return (sg & 1) ? X1(gi) : X0(gi); };
    auto Xout = [&](int gi) { return (sg & 1) ? X0(gi) : X1(gi); };
    es.clear();
    for (int gi : gl) es.push_back({gi, Xin(gi), Xin(gi), Ab(gi), nullptr});
    if ((rc = emit(PH_GRAM, es, 1.f, 0.f, 0.f, sg == 0 ? 2 : 0, 1, 1))) return rc;
    // p x p products: one flat launch per op over all matrices
    for (int tl = 0; tl < Ts; ++tl) {
      const int t = t0 + tl;
      const float a = c->ns_coeffs[t][0], b = c->ns_coeffs[t][1], cc = c->ns_coeffs[t][2];
      const bool last = tl == Ts - 1;
      es.clear();
      for (int gi : gl) es.push_back({gi, Ab(gi), Ab(gi), Cb(gi, tl), Ab(gi)});
      if ((rc = emit(PH_POLY, es, cc, b, a, 0, 1, 1, Ts == 1))) return rc;
      es.clear();
      for (int gi : gl) {
        if (tl >= 1) es.push_back({gi, Cb(gi, tl), Qb(gi, tl), Qb(gi, tl + 1), nullptr});
        if (!last) es.push_back({gi, Cb(gi, tl), Ab(gi), Bb(gi), nullptr});
      }
      if (!es.empty() && (rc = emit(PH_NSMUL, es, 1.f, 0.f, 0.f, 0, 1, 1, last))) return rc;
      if (!last) {
        es.clear();
        for (int gi : gl) es.push_back({gi, Cb(gi, tl), Bb(gi), Ab(gi), nullptr});
        if ((rc = emit(PH_NSMUL, es, 1.f, 0.f, 0.f, 0, 1, 1))) return rc;
      }
    }
    es.clear();
    for (int gi : gl) es.push_back({gi, Qb(gi, Ts), Xin(gi), Xout(gi), nullptr});
    if ((rc = emit(PH_APPLY, es, 1.f, 0.f, 0.f, sg == 0 ? 1 : 0, 1, 1))) return rc;
  }
  return DION2_OK;
}

// Fill host tables and NS launches for a concrete workspace.
int build_device_plan(Plan& P, const dion2_matrix* mats, const dion2_config* c, void* ws) {
  P.ws = ws;
  const int n = P.n;
  P.host_tables.assign(P.off_nsscale - P.off_desc, 0);
  if (!P.dtab && cudaMalloc(&P.dtab, P.host_tables.size()) != cudaSuccess) return DION2_ECUDA;
  auto H = [&](size_t off) { return P.host_tables.data() + (off - P.off_desc); };
  MatDesc* D = reinterpret_cast<MatDesc*>(H(P.off_desc));
  std::vector<int32_t> rowmats, colmats;
  std::vector<int64_t> rowprefix, colprefix;
  std::vector<int32_t> gprefix(n);
  std::vector<int32_t> flg_mats[2], fls_mats[2], fl_gp[2], fl_sp[2], mtmats;
  std::vector<int64_t> mtprefix;
  int64_t mt_acc = 0;
  std::vector<int32_t> cf_mats;
  std::vector<int64_t> cf_prefix;
  P.cf_total = 0;
  P.fl_gunits[0] = P.fl_gunits[1] = P.fl_sunits[0] = P.fl_sunits[1] = 0;
  P.fl_maxk = 0;
  P.fl_smaxk = 0;
  P.fl_maxn = 0;
  int64_t rows_acc = 0, ctiles_acc = 0;
  int gt_acc = 0;
  P.generic_gather_mats = 0;
  P.generic_scatter_mats = 0;
  for (int i = 0; i < n; ++i) {
    const MatPlan& q = P.mp[i];
    const Group& g = P.groups[q.group];
    MatDesc& d = D[i];
    d.rows = mats[i].rows;
    d.cols = mats[i].cols;
    d.ld = mats[i].ld;
    d.axis = q.axis;
    d.d = q.d; d.o = q.o; d.k = q.k; d.sr = q.sr; d.sc = q.sc; d.transposed = q.transposed;
    d.p = q.p; d.q = q.q; d.p_pad = q.p_pad; d.q_pad = q.q_pad;
    d.grad_bf16 = c->grad_dtype == DION2_DT_BF16;
    d.update_scale = q.fan_sqrt;
    d.scores = (float*)at(ws, q.off_scores);
    d.col_partials = q.axis == DION2_AXIS_COLS ? (float*)at(ws, q.off_partials) : nullptr;
    d.sel = (int32_t*)at(ws, q.off_sel);
    d.sumsq_partials = (float*)at(ws, q.off_sumsq);
    d.ns_scale = (float*)at(ws, P.off_nsscale) + 4 * i;
    d.x16 = P.bf16_ns ? 1 : 0;
    const size_t xel = P.bf16_ns ? 2 : 4;
    d.X0 = at(ws, g.off_X0 + (size_t)q.zi * g.p_pad * g.q_pad * xel);
    d.X1 = at(ws, g.off_X1 + (size_t)q.zi * g.p_pad * g.q_pad * xel);
    // X_T lands in X1 after an odd number of applies (direct: T; Gram space: one per segment)
    d.final_in_x1 = g.tiny ? 1 : (g.gs ? (int)(ns_segments(c, P.ns_steps).size() & 1) : (P.ns_steps & 1));
    d.gather_tile_base = gt_acc;
    d.gather_tiles_a = q.ga;
    d.gather_tiles_b = q.gb;
    d.sa_pad = q.sa_pad;
    d.sb_pad = q.sb_pad;
    d.rowblocks = q.rowblocks;
    // cols mode: the column sums of the K1 row-block partials are finalised by a grid-wide
    // kernel before K2 (one K2 CTA summing m / 256 partials per column is latency-bound: 112
    // partials on 28672 rows; even the 1B set's 32 gain, select 0.038 -> 0.029 ms);
    // DION2_CF_MIN_RB = r: only matrices with >= r row blocks (the rest are summed by K2)
    static const int cf_min = getenv("DION2_CF_MIN_RB") ? atoi(getenv("DION2_CF_MIN_RB")) : 1;
    const bool cf = q.axis == DION2_AXIS_COLS && q.rowblocks >= cf_min;
    d.scores_final = cf ? 1 : 0;
    if (cf) {
      cf_mats.push_back(i);
      cf_prefix.push_back(P.cf_total);
      P.cf_total += mats[i].cols;
    }
    d.mid = i;
    d.path = q.path;
    d.spath = q.spath;
    d.n_sumsq = q.n_sumsq;
    d.mt = q.mt;
    d.ldm = q.mt ? mats[i].ldm : 0;
    gprefix[i] = gt_acc;
    gt_acc += q.ga * q.gb;
    if (q.ga * q.gb > 0 && !q.mt && q.path == 0) P.generic_gather_mats++;  // transposed-M matrices: row gather
    if (q.ga * q.gb > 0 && q.spath == 0) P.generic_scatter_mats++;
    // gather: rows streaming (path 1, or transposed-M columns = rows of M^T), cols streaming
    // (path 2) or generic tiles; scatter: by path (generic tiles for path 0)
    const int lg = (q.path == 1 || q.mt) ? 0 : (q.path == 2 ? 1 : -1);
    const int ls = q.spath - 1;
    if (lg >= 0) {
      flg_mats[lg].push_back(i);
      fl_gp[lg].push_back(P.fl_gunits[lg]);
      P.fl_gunits[lg] += lg == 0 ? q.p_pad : q.q_pad / 32;
    }
    if (ls >= 0) {
      fls_mats[ls].push_back(i);
      fl_sp[ls].push_back(P.fl_sunits[ls]);
      P.fl_sunits[ls] += ls == 0 ? q.k : q.q_pad / 32;
    }
    if (lg == 1 || ls == 1) P.fl_maxn = std::max<int64_t>(P.fl_maxn, mats[i].cols);
    if (lg == 1) P.fl_maxk = std::max(P.fl_maxk, q.k);
    if (ls == 1) P.fl_smaxk = std::max(P.fl_smaxk, q.k);
    if (q.axis == DION2_AXIS_ROWS) {
      rowmats.push_back(i);
      rowprefix.push_back(rows_acc);
      rows_acc += mats[i].rows;
    } else if (q.mt) {
      mtmats.push_back(i);
      mtprefix.push_back(mt_acc);
      mt_acc += (int64_t)q.rowblocks * ceil_div(mats[i].cols, 64);
    } else {
      colmats.push_back(i);
      colprefix.push_back(ctiles_acc);
      ctiles_acc += (int64_t)q.rowblocks * ceil_div(mats[i].cols, 256);
    }
  }
  P.total_rows = rows_acc;
  P.total_col_tiles = ctiles_acc;
  P.n_row_mats = (int)rowmats.size();
  P.n_col_mats = (int)colmats.size();
  P.total_gather_tiles = gt_acc;
  for (int l = 0; l < 2; ++l) {
    P.fl_gn[l] = (int)flg_mats[l].size();
    P.fl_sn[l] = (int)fls_mats[l].size();
    if (P.fl_gn[l]) {
      memcpy(H(P.off_flg_mats[l]), flg_mats[l].data(), 4 * flg_mats[l].size());
      memcpy(H(P.off_fl_gprefix[l]), fl_gp[l].data(), 4 * fl_gp[l].size());
    }
    if (P.fl_sn[l]) {
      memcpy(H(P.off_fls_mats[l]), fls_mats[l].data(), 4 * fls_mats[l].size());
      memcpy(H(P.off_fl_sprefix[l]), fl_sp[l].data(), 4 * fl_sp[l].size());
    }
  }
  P.n_mt_mats = (int)mtmats.size();
  P.total_mt_tiles = mt_acc;
  if (!mtmats.empty()) {
    memcpy(H(P.off_mtmats), mtmats.data(), 4 * mtmats.size());
    memcpy(H(P.off_mtprefix), mtprefix.data(), 8 * mtprefix.size());
  }
  if (!rowmats.empty()) {
    memcpy(H(P.off_rowmats), rowmats.data(), 4 * rowmats.size());
    memcpy(H(P.off_rowprefix), rowprefix.data(), 8 * rowprefix.size());
  }
  if (!colmats.empty()) {
    memcpy(H(P.off_colmats), colmats.data(), 4 * colmats.size());
    memcpy(H(P.off_colprefix), colprefix.data(), 8 * colprefix.size());
  }
  memcpy(H(P.off_gprefix), gprefix.data(), 4 * n);
  P.cf_n = (int)cf_mats.size();
  if (P.cf_n) {
    memcpy(H(P.off_cf_mats), cf_mats.data(), 4 * cf_mats.size());
    memcpy(H(P.off_cf_prefix), cf_prefix.data(), 8 * cf_prefix.size());
  }
  for (auto& g : P.groups) memcpy(H(g.off_gmats), g.mats.data(), 4 * g.mats.size());
  {
    std::vector<int32_t> tiny;
    for (int i = 0; i < n; ++i)
      if (P.mp[i].tiny && P.mp[i].p <= 64) tiny.push_back(i);
    P.n_tiny64 = (int)tiny.size();
    for (int i = 0; i < n; ++i)
      if (P.mp[i].tiny && P.mp[i].p > 64) tiny.push_back(i);
    P.n_tiny = (int)tiny.size();
    if (P.n_tiny) memcpy(H(P.off_tiny_list), tiny.data(), 4 * tiny.size());
  }

  // ---- Newton-Schulz launch list: per iteration t: gram, poly, apply; per phase the
  // groups are batched (<= kMaxGroups per launch, one BN class per launch).
  P.ns_launches.clear();
  const float* scale_all = (const float*)at(ws, P.off_nsscale);
  // bf16 path: 2-SM (cta_group::2) 256 x 256 tiles; DION2_NS_1SM=1 selects the 1-SM 128 x 256 kernel
  // (measured: the pair kernel wins on the long-K gram, the 1-SM kernel on the
  // short-K poly and the MN-major apply; DION2_NS_PAIR=all|none overrides)
  // DION2_NS_PAIR (A/B only): unset = pair kernel for gram / poly / products and the resident-A
  // pair apply; "all" = the streaming pair kernel for the apply too; "1sm_apply" = the 1-SM
  // apply (round 1's default); "none" = the 1-SM kernel everywhere
  const char* pair_env = getenv("DION2_NS_PAIR");
  const int pair_mode = !pair_env ? 1
                                  : (strcmp(pair_env, "all") == 0 ? 2
                                                                  : (strcmp(pair_env, "none") == 0 ? 0
                                                                                                   : (strcmp(pair_env, "1sm_apply") == 0 ? 3 : 1)));
  for (int t = 0; t < P.ns_steps; ++t) {
    const float a = c->ns_coeffs[t][0], b = c->ns_coeffs[t][1], cc = c->ns_coeffs[t][2];
    for (int ph = PH_GRAM; ph <= PH_APPLY; ++ph) {
      // apply: the 2-SM kernel with A resident for p_pad <= 512 (k_ns_apply_pair.cu)
      bool res_all = P.bf16_ns && ph == PH_APPLY && pair_mode == 1;  // (3: the 1-SM apply)
      for (const Group& g : P.groups)
        if (!g.gs) res_all = res_all && g.p_pad <= 64 * kMaxResidentKB;
      const bool pair = P.bf16_ns && (pair_mode == 2 || ((pair_mode == 1 || pair_mode == 3) && (ph != PH_APPLY || res_all)));
      // gram and poly outputs are symmetric: the pair kernel computes upper-triangle tiles
      // only and mirrors them (DION2_NS_SYM=0 disables)
      const bool sym = pair && ph != PH_APPLY && !(getenv("DION2_NS_SYM") && atoi(getenv("DION2_NS_SYM")) == 0);
      const int MT = pair ? 256 : 128;
      // bucket groups by BN class
      std::vector<int> by_bn[2];
      for (int gi = 0; gi < (int)P.groups.size(); ++gi) {
        const Group& g = P.groups[gi];
        if (g.gs || g.tiny) continue;  // Gram-space groups: append_gram_space_launches; tiny: k_ns_small
        int bn256 = ph == PH_APPLY ? 1 : (g.p_pad % 256 == 0);
        by_bn[bn256].push_back(gi);
      }
      for (int cls = 0; cls < 2; ++cls) {
        const int BN = cls ? 256 : 128;
        auto& gl = by_bn[cls];
        for (size_t s0 = 0; s0 < gl.size(); s0 += kMaxGroups) {
          Launch L{};
          L.phase = ph;
          L.bn = BN;
          L.kind = P.bf16_ns ? (res_all ? 5 : (pair ? 3 : cls)) : 2;
          NsParams& np = L.tc.p;
          np.ngroups = (int)std::min<size_t>(kMaxGroups, gl.size() - s0);
          np.ns_scale_all = scale_all;
          np.in_f16 = np.out_f16 = P.bf16_ns ? 1 : 0;  // fp16 X / A / C (reading R24)
          // gram: A = s^2 X X^T; poly: C = a I + b A + c A A^T (consistent 16-bit A);
          // apply: X' = s C X (the linear term a X is folded into C: no epilogue read)
          np.diag = 0.f;
          np.sym = sym ? 1 : 0;
          if (ph == PH_GRAM) { np.cacc = 1.f; np.cC = 0.f; np.scale_sel = t == 0 ? 2 : 0; np.b_kmajor = 1; }
          if (ph == PH_GRAM && pair && sym && P.gram_splitk > 1) {  // partials sized for sym tiles
            np.splitk = P.gram_splitk;
            np.partial = (float*)at(ws, P.off_splitk);
          }
          if (ph == PH_POLY) { np.cacc = cc; np.cC = b; np.diag = a; np.scale_sel = 0; np.b_kmajor = 1; }
          if (ph == PH_APPLY) { np.cacc = 1.f; np.cC = 0.f; np.scale_sel = t == 0 ? 1 : 0; np.b_kmajor = 0; }
          int tiles = 0;
          for (int j = 0; j < np.ngroups; ++j) {
            const Group& g = P.groups[gl[s0 + j]];
            const size_t xel = P.bf16_ns ? 2 : 4;
            void* Xc = at(ws, (t & 1) ? g.off_X1 : g.off_X0);
            void* Xn = at(ws, (t & 1) ? g.off_X0 : g.off_X1);
            void* A = at(ws, g.off_A);
            void* Bm = at(ws, g.off_B);
            NsGroup& G = np.g[j];
            G.count = g.count;
            G.gmats = (const int32_t*)tab(P, g.off_gmats);
            const long long xs = (long long)g.p_pad * g.q_pad, as = (long long)g.p_pad * g.p_pad;
            if (ph == PH_GRAM) {
              G.m_tiles = g.p_pad / MT; G.n_tiles = g.p_pad / BN; G.k_blocks = g.q_pad / 64;
              G.a = Xc; G.a_mstride = xs; G.lda = g.q_pad;
              G.b = Xc; G.b_mstride = xs; G.ldb = g.q_pad;
              G.out = A; G.out_mstride = as; G.out_ld = g.p_pad;
              G.cin = nullptr; G.cin_mstride = 0; G.cin_ld = 0;
              if (P.bf16_ns) {
                if (!make_map(&L.tc.mapA[j], Xc, g.q_pad, g.p_pad, g.count, 64, 128)) return DION2_ECUDA;
                if (!make_map(&L.tc.mapB[j], Xc, g.q_pad, g.p_pad, g.count, 64, pair ? 128 : BN)) return DION2_ECUDA;
              }
            } else if (ph == PH_POLY) {
              G.m_tiles = g.p_pad / MT; G.n_tiles = g.p_pad / BN; G.k_blocks = g.p_pad / 64;
              G.a = A; G.a_mstride = as; G.lda = g.p_pad;
              G.b = A; G.b_mstride = as; G.ldb = g.p_pad;
              G.out = Bm; G.out_mstride = as; G.out_ld = g.p_pad;
              G.cin = A; G.cin_mstride = as; G.cin_ld = g.p_pad;
              if (P.bf16_ns) {
                if (!make_map(&L.tc.mapA[j], A, g.p_pad, g.p_pad, g.count, 64, 128)) return DION2_ECUDA;
                if (!make_map(&L.tc.mapB[j], A, g.p_pad, g.p_pad, g.count, 64, pair ? 128 : BN)) return DION2_ECUDA;
              }
            } else {
              G.m_tiles = g.p_pad / MT; G.n_tiles = g.q_pad / BN; G.k_blocks = g.p_pad / 64;
              G.a = Bm; G.a_mstride = as; G.lda = g.p_pad;
              G.b = Xc; G.b_mstride = xs; G.ldb = g.q_pad;
              G.out = Xn; G.out_mstride = xs; G.out_ld = g.q_pad;
              G.cin = nullptr; G.cin_mstride = 0; G.cin_ld = 0;
              if (P.bf16_ns) {
                if (!make_map(&L.tc.mapA[j], Bm, g.p_pad, g.p_pad, g.count, 64, 128)) return DION2_ECUDA;
                // MN-major B operand: box = 64 columns of X (N) x 64 rows of X (K)
                if (!make_map(&L.tc.mapB[j], Xc, g.q_pad, g.p_pad, g.count, 64, 64)) return DION2_ECUDA;
              }
            }
            (void)xel;
            if (P.bf16_ns &&
                !make_map(&L.tc.mapD[j], G.out, G.out_ld, g.p_pad, g.count, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
              return DION2_ECUDA;
            G.tile_base = tiles;
            tiles += G.count * (sym ? G.m_tiles * (G.m_tiles + 1) / 2 : G.m_tiles * G.n_tiles);
          }
          np.total_tiles = tiles;
          np.b_is_a = np.b_kmajor ? 1 : 0;
          for (int j = 0; j < np.ngroups; ++j) np.b_is_a &= np.g[j].a == np.g[j].b ? 1 : 0;
          if (L.kind == 5) apply_chunks(np);
          if (P.bf16_ns) {
            P.ns_launches.push_back(L);
          } else {
            // SIMT path: one launch per group
            for (int j = 0; j < np.ngroups; ++j) {
              Launch L2 = L;
              L2.simt_group = j;
              P.ns_launches.push_back(L2);
            }
          }
        }
      }
    }
  }
  return append_gram_space_launches(P, c, ws, pair_mode);
}

void ensure_device_attrs() {
  if (g_attr_done) return;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
  ns_tc_set_attrs();
  launch_fast_paths_attrs();
  ns_pair_set_attrs();
  ns_apply_pair_set_attrs();
  cudaFuncSetAttribute(k_topk_select, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * DION2_MAX_SELECT_DIM);
  cudaFuncSetAttribute(k_full_decay, cudaFuncAttributeMaxDynamicSharedMemorySize, DION2_MAX_SELECT_DIM);
  g_attr_done = true;
}


// norm finalize (optional) + the Newton-Schulz launch list of a plan.
int run_ns(Plan& P, const dion2_config* c, Launcher& L, cudaStream_t s, bool do_norm) {
  const int sms = g_sm_count > 0 ? g_sm_count : 148;
  const MatDesc* dmats = (const MatDesc*)tab(P, P.off_desc);
  if (do_norm) {
    L.begin(PH_NORM);
    k_norm_finalize<<<(unsigned)ceil_div(P.n, 8), 256, 0, s>>>(dmats, P.n, c->ns_eps);
    L.end();
  }
  for (const Launch& ln : P.ns_launches) {
    L.begin(ln.phase);
    if (ln.kind == 5) {
      launch_ns_apply_pair(std::min(2 * ln.tc.p.total_tiles, sms & ~1), s, ln.tc);
    } else if (ln.kind == 3) {
      const int sk = ln.tc.p.splitk > 1 ? ln.tc.p.splitk : 1;
      launch_ns_pair(std::min(2 * ln.tc.p.total_tiles * sk, sms & ~1), s, ln.tc);
      if (sk > 1) launch_splitk_reduce(s, ln.tc.p);
    } else if (ln.kind == 0 || ln.kind == 1) {
      launch_ns_tc(ln.bn, std::min(ln.tc.p.total_tiles, sms), s, ln.tc);
    } else {
      const NsGroup& G = ln.tc.p.g[ln.simt_group];
      const int Mdim = G.m_tiles * 128;
      const int Ndim = G.n_tiles * ln.bn;
      dim3 grid(Ndim / 64, Mdim / 64, G.count);
      k_ns_gemm_simt_f32<<<grid, 256, 0, s>>>(ln.tc.p, ln.simt_group);
    }
    L.end();
  }
  return L.err;
}

// Upload the caller's W/M/G/sel_out/O_out pointers into the plan-owned descriptor
// table when they changed (the workspace itself is pure scratch).
int refresh_tables(Plan& P, const dion2_matrix* mats, const dion2_config* c, cudaStream_t s) {
  const int n = P.n;
  bool upload = false;
  if ((int)P.last_ptrs.size() != 6 * n) {
    P.last_ptrs.assign(6 * n, nullptr);
    upload = true;
  }
  MatDesc* D = reinterpret_cast<MatDesc*>(P.host_tables.data());
  for (int i = 0; i < n; ++i) {
    const void* ptrs[6] = {mats[i].W, mats[i].M, mats[i].G, mats[i].sel_out, mats[i].O_out,
                           reinterpret_cast<const void*>((uintptr_t)(mats[i].m_transposed ? mats[i].ldm : 0))};
    for (int j = 0; j < 6; ++j)
      if (P.last_ptrs[6 * i + j] != ptrs[j]) { upload = true; P.last_ptrs[6 * i + j] = ptrs[j]; }
    D[i].ldm = mats[i].m_transposed ? mats[i].ldm : 0;
    D[i].W = mats[i].W;
    D[i].M = mats[i].M;
    D[i].G = mats[i].G;
    D[i].sel_out = mats[i].sel_out;
    D[i].O_out = mats[i].O_out;
    const size_t gel = c->grad_dtype == DION2_DT_BF16 ? 2 : 4;
    const size_t wal = c->w_dtype == DION2_DT_BF16 ? 8 : 16;  // 4 W elements per vector access
    const bool al = ((uintptr_t)mats[i].W % wal == 0) && ((uintptr_t)mats[i].M % 16 == 0) &&
                    ((uintptr_t)mats[i].G % (gel == 4 ? 16 : 8) == 0) && (mats[i].ld % 4 == 0) &&
                    (!mats[i].m_transposed || mats[i].ldm % 4 == 0);
    D[i].vec4 = al ? 1 : 0;
  }
  if (upload &&
      cudaMemcpyAsync(P.dtab, P.host_tables.data(), P.host_tables.size(), cudaMemcpyHostToDevice, s) != cudaSuccess)
    return DION2_ECUDA;
  return DION2_OK;
}

int reset_status(int32_t* status, cudaStream_t s) {
  // status[0] = flags (0), status[1] = first bad matrix (atomicMin from 0x7f7f7f7f)
  if (cudaMemsetAsync(status, 0, 4, s) != cudaSuccess) return DION2_ECUDA;
  if (cudaMemsetAsync(status + 1, 0x7f, 4, s) != cudaSuccess) return DION2_ECUDA;
  return DION2_OK;
}

// grid of a streaming kernel: `persistent` caps it at a few CTAs per SM (grid-stride
// loops); otherwise one CTA per work chunk, so CTAs retire quickly and a concurrently
// launched (higher-priority) NS kernel can take SM slots as they free up.
inline int stream_grid(int64_t units, int per_sm, bool persistent) {
  const int sms = g_sm_count > 0 ? g_sm_count : 148;
  const int64_t cap = persistent ? (int64_t)sms * per_sm : (int64_t)1 << 30;
  return (int)std::max<int64_t>(1, std::min<int64_t>(units, cap));
}

// K1 momentum + score, K2 select, K3 gather + decay (Alg. 1 l.2-5)
void stage_pre(Plan& P, const dion2_config* c, void* ws, int32_t* status, Launcher& L, cudaStream_t s,
               bool persistent) {
  stage_k1_select(P, c, ws, status, L, s, persistent);
  stage_gather(P, c, ws, L, s, persistent);
}

// Transposed-M K1 over a list of column-mode matrices: the cp.async-pipelined kernel when
// every transposed-M matrix of the host descriptor table has fp32 G and aligned whole
// 256 x 64 units (DION2_K1MT_PIPE=0: the register-staged kernel; =2/3/4: stages; 3 = two
// 96 KB CTAs per SM measured best: 0.93 -> 0.76 ms on the 1B set), else the register-staged
// kernel on `legacy_grid` blocks.
void launch_k1_mt(const MatDesc* host_desc, int n_desc, int grad_dtype, int64_t total_tiles, int legacy_grid,
                  cudaStream_t s, const MatDesc* dmats, const int32_t* list, const int64_t* prefix, int n_list) {
  const char* pe = getenv("DION2_K1MT_PIPE");  // read per call (tests flip it)
  int pipe_stages = pe ? atoi(pe) : 3;
  if (pipe_stages != 0 && (pipe_stages < 2 || pipe_stages > 4)) pipe_stages = 3;
  const bool bf16 = grad_dtype == DION2_DT_BF16;
  bool pipe = pipe_stages != 0;
  for (int i = 0; i < n_desc && pipe; ++i)
    if (host_desc[i].mt && host_desc[i].axis == kAxisCols)
      pipe = (host_desc[i].grad_bf16 != 0) == bf16 && host_desc[i].vec4 && host_desc[i].rows % kColRowBlock == 0 &&
             host_desc[i].cols % 64 == 0 && host_desc[i].ldm % 4 == 0 &&
             (!bf16 || (host_desc[i].ld % 8 == 0 && (uintptr_t)host_desc[i].G % 16 == 0));
  if (pipe) {
    static int per_sm[5][2] = {{-1, -1}, {-1, -1}, {-1, -1}, {-1, -1}, {-1, -1}};
    int& nb = per_sm[pipe_stages][bf16];
    if (nb < 0) nb = std::max(1, momentum_score_cols_mt_pipe_attrs(pipe_stages, bf16));
    const int sms = g_sm_count > 0 ? g_sm_count : 148;
    launch_momentum_score_cols_mt_pipe(pipe_stages, bf16, (int)std::min<int64_t>(total_tiles, (int64_t)nb * sms), s,
                                       dmats, list, prefix, n_list, total_tiles);
  } else {
    k_momentum_score_cols_mt<<<legacy_grid, 256, 0, s>>>(dmats, list, prefix, n_list, total_tiles);
  }
}

// K1 momentum + score, K2 select (Alg. 1 l.2-3)
void stage_k1_select(Plan& P, const dion2_config* c, void* ws, int32_t* status, Launcher& L, cudaStream_t s,
                     bool persistent) {
  const int n = P.n;
  const MatDesc* dmats = (const MatDesc*)tab(P, P.off_desc);
  int32_t* bad = (int32_t*)at(ws, P.off_bad);
  if (P.n_row_mats) {
    L.begin(PH_K1);
    const int blocks = stream_grid(ceil_div(P.total_rows, 8), 8, persistent);
    k_momentum_score_rows<<<blocks, 256, 0, s>>>(dmats, (const int32_t*)tab(P, P.off_rowmats),
                                                 (const int64_t*)tab(P, P.off_rowprefix), P.n_row_mats, P.total_rows);
    L.end();
  }
  if (P.n_col_mats) {
    L.begin(PH_K1);
    const int blocks = stream_grid(P.total_col_tiles, 8, persistent);
    k_momentum_score_cols<<<blocks, 256, 0, s>>>(dmats, (const int32_t*)tab(P, P.off_colmats),
                                                 (const int64_t*)tab(P, P.off_colprefix), P.n_col_mats,
                                                 P.total_col_tiles);
    L.end();
  }
  if (P.n_mt_mats) {
    L.begin(PH_K1_MT);
    launch_k1_mt(reinterpret_cast<const MatDesc*>(P.host_tables.data()), n, c->grad_dtype, P.total_mt_tiles,
                 stream_grid(P.total_mt_tiles, 8, persistent), s, dmats, (const int32_t*)tab(P, P.off_mtmats),
                 (const int64_t*)tab(P, P.off_mtprefix), P.n_mt_mats);
    L.end();
  }
  const int n_sel = n;
  if (P.cf_n) {
    L.begin(PH_SELECT);
    k_col_scores_finalize<<<(unsigned)ceil_div(P.cf_total, 32), 256, 0, s>>>(
        dmats, (const int32_t*)tab(P, P.off_cf_mats), (const int64_t*)tab(P, P.off_cf_prefix), P.cf_n, P.cf_total);
    L.end();
  }
  if (n_sel) {
    L.begin(PH_SELECT);
    const int32_t* list = nullptr;
    k_topk_select<<<n_sel, kSelectThreads, 4 * P.max_d, s>>>(dmats, list, bad, status,
                                                             c->select == DION2_SELECT_RANDOM, c->seed, c->step);
    L.end();
  }
}

// K3 gather + selective decay (Alg. 1 l.4-5); first the fp64 NS of short X (k_ns_small.cu), which
// reads the pre-decay M[K]
void stage_gather(Plan& P, const dion2_config* c, void* ws, Launcher& L, cudaStream_t s, bool persistent) {
  const int n = P.n;
  const MatDesc* dmats = (const MatDesc*)tab(P, P.off_desc);
  int32_t* bad = (int32_t*)at(ws, P.off_bad);
  if (P.n_tiny) {
    NsSmallCoeffs cs{};
    for (int t = 0; t < c->ns_steps && t < 16; ++t)
      for (int e = 0; e < 3; ++e) cs.c[t][e] = c->ns_coeffs[t][e];
    cs.T = c->ns_steps;
    cs.eps = c->ns_eps;
    L.begin(PH_NSMUL);
    const int32_t* tl = (const int32_t*)tab(P, P.off_tiny_list);
    launch_ns_small(s, dmats, tl, P.n_tiny64, bad, cs, false);
    launch_ns_small(s, dmats, tl + P.n_tiny64, P.n_tiny - P.n_tiny64, bad, cs, true);
    L.end();
  }
  if (P.total_gather_tiles > 0 && P.generic_gather_mats > 0) {
    L.begin(PH_GATHER);
    launch_gather_decay(P.bf16_ns, stream_grid(P.total_gather_tiles, 8, persistent), s, dmats,
                        (const int32_t*)tab(P, P.off_gprefix), n, P.total_gather_tiles, bad, 1, c->mu);
    L.end();
  }
  if (P.fl_gn[0]) {
    // TMA-staged rows gather when every listed matrix has 16-B aligned rows with n % 8 == 0
    // (DION2_GATHER_TMA=0: the register-streaming kernel; =4/6: ring stages; 6 = 0.496 ms vs
    // 0.500 for the register kernel on the 1B set, 4 = 0.52)
    const char* ge = getenv("DION2_GATHER_TMA");
    const int gstages = ge ? atoi(ge) : 6;
    bool tma = gstages != 0;
    const MatDesc* hd = reinterpret_cast<const MatDesc*>(P.host_tables.data());
    const int32_t* lm = reinterpret_cast<const int32_t*>(P.host_tables.data() + (P.off_flg_mats[0] - P.off_desc));
    for (int j = 0; j < P.fl_gn[0] && tma; ++j) {
      const MatDesc& m = hd[lm[j]];
      tma = m.vec4 && ((m.mt ? m.rows : m.cols) % 8 == 0) && (!m.mt || m.ldm % 4 == 0);
    }
    L.begin(PH_GATHER_ROWS);
    if (tma) {
      launch_gather_rows_tma(gstages, 16, s, dmats, (const int32_t*)tab(P, P.off_flg_mats[0]),
                             (const int32_t*)tab(P, P.off_fl_gprefix[0]), P.fl_gn[0], P.fl_gunits[0], bad, c->mu,
                             g_sm_count > 0 ? g_sm_count : 148);
    } else {
      launch_gather_rows(stream_grid(ceil_div(P.fl_gunits[0], 8), 8, persistent), s, dmats,
                         (const int32_t*)tab(P, P.off_flg_mats[0]), (const int32_t*)tab(P, P.off_fl_gprefix[0]),
                         P.fl_gn[0], P.fl_gunits[0], bad, c->mu);
    }
    L.end();
  }
  if (P.fl_gn[1]) {
    L.begin(PH_GATHER_COLS);
    launch_gather_cols_t(stream_grid(P.fl_gunits[1], 6, persistent), P.fl_maxk, P.fl_maxn, s, dmats,
                         (const int32_t*)tab(P, P.off_flg_mats[1]), (const int32_t*)tab(P, P.off_fl_gprefix[1]),
                         P.fl_gn[1], P.fl_gunits[1], bad, c->mu);
    L.end();
  }
}

// K7 scatter (Alg. 1 l.6) and the full-decay ablation
void stage_post(Plan& P, const dion2_matrix* mats, const dion2_config* c, void* ws, Launcher& L, cudaStream_t s,
                bool persistent) {
  const int n = P.n;
  const MatDesc* dmats = (const MatDesc*)tab(P, P.off_desc);
  int32_t* bad = (int32_t*)at(ws, P.off_bad);
  // DION2_FLAG_LR_DEVICE: eta is the fp32 word at workspace byte 8 (written by the caller)
  const float* lr_dev = (c->reserved0 & DION2_FLAG_LR_DEVICE) ? (const float*)at(ws, P.off_status + 8) : nullptr;
  if (P.total_gather_tiles > 0 && P.generic_scatter_mats > 0) {
    L.begin(PH_SCATTER);
    launch_scatter_update(P.bf16_ns, c->w_dtype == DION2_DT_BF16, stream_grid(P.total_gather_tiles, 8, persistent), s, dmats,
                          (const int32_t*)tab(P, P.off_gprefix), n, P.total_gather_tiles, bad, c->lr, lr_dev);
    L.end();
  }
  if (P.fl_sn[0]) {
    L.begin(PH_SCATTER_ROWS);
    launch_scatter_rows(c->w_dtype == DION2_DT_BF16, stream_grid(ceil_div(P.fl_sunits[0], 8), 8, persistent), s, dmats,
                        (const int32_t*)tab(P, P.off_fls_mats[0]), (const int32_t*)tab(P, P.off_fl_sprefix[0]),
                        P.fl_sn[0], P.fl_sunits[0], bad, c->lr, lr_dev);
    L.end();
  }
  if (P.fl_sn[1]) {
    L.begin(PH_SCATTER_COLS);
    launch_scatter_cols_t(c->w_dtype == DION2_DT_BF16, stream_grid(P.fl_sunits[1], 6, persistent), P.fl_smaxk, P.fl_maxn, s, dmats,
                          (const int32_t*)tab(P, P.off_fls_mats[1]), (const int32_t*)tab(P, P.off_fl_sprefix[1]),
                          P.fl_sn[1], P.fl_sunits[1], bad, c->lr, lr_dev);
    L.end();
  }
  if (c->decay_mode == 1) {
    L.begin(PH_FULLDECAY);
    int64_t maxrows = 0;
    for (int i = 0; i < n; ++i) maxrows = std::max<int64_t>(maxrows, mats[i].rows);
    dim3 grid((unsigned)ceil_div(maxrows, 64), n);
    k_full_decay<<<grid, 256, P.max_d, s>>>(dmats, n, bad, c->mu);
    L.end();
  }
}

int run_step(Plan& P, const dion2_matrix* mats, const dion2_config* c, void* ws, cudaStream_t s) {
  int rc = refresh_tables(P, mats, c, s);
  if (rc) return rc;
  int32_t* status = (int32_t*)at(ws, P.off_status);
  if ((rc = reset_status(status, s))) return rc;
  Launcher L{s};
  stage_pre(P, c, ws, status, L, s, true);
  run_ns(P, c, L, s, true);  // norm finalize + K4-K6 Newton-Schulz (Alg. 1 l.4)
  stage_post(P, mats, c, ws, L, s, true);
  g_last_launches = L.count;
  return L.err;
}

}  // namespace dion2rt

// ============================================================================ C ABI

extern "C" {

int dion2_config_init(dion2_config* cfg) {
  if (!cfg) return DION2_EINVAL_CONFIG;
  memset(cfg, 0, sizeof(*cfg));
  cfg->alpha = 0.25f;
  cfg->mu = 0.95f;
  cfg->lr = 0.02f;
  cfg->ns_steps = 5;
  for (int t = 0; t < DION2_MAX_NS_STEPS; ++t) {
    cfg->ns_coeffs[t][0] = 3.4445f;
    cfg->ns_coeffs[t][1] = -4.7750f;
    cfg->ns_coeffs[t][2] = 2.0315f;
  }
  cfg->ns_eps = 1e-7f;
  cfg->axis = DION2_AXIS_AUTO;
  cfg->select = DION2_SELECT_L1;
  cfg->precision = DION2_NS_BF16;
  cfg->grad_dtype = DION2_DT_F32;
  cfg->decay_mode = 0;
  cfg->scale_mode = 0;
  return DION2_OK;
}

int dion2_workspace_size(const dion2_matrix* user_mats, int32_t n, const dion2_config* cfg, size_t* bytes_out) {
  if (!bytes_out) return DION2_EINVAL_CONFIG;
  int rc = validate_config(cfg);
  if (rc) return rc;
  if (n < 1 || !user_mats) return DION2_EINVAL_SHAPE;
  const std::vector<dion2_matrix> sv = storage_view(user_mats, n);
  const dion2_matrix* mats = sv.data();
  for (int i = 0; i < n; ++i)
    if ((rc = validate_shape(mats[i], false))) return rc;
  Plan P;
  rc = build_layout(P, mats, n, cfg);
  if (rc) return rc;
  *bytes_out = P.total;
  return DION2_OK;
}

int dion2_step_batched(const dion2_matrix* user_mats, int32_t n, const dion2_config* cfg, void* workspace,
                       size_t ws_bytes, void* stream) {
  int rc = validate_config(cfg);
  if (rc) return rc;
  if (n < 1 || !user_mats) return DION2_EINVAL_SHAPE;
  const std::vector<dion2_matrix> sv = storage_view(user_mats, n);
  const dion2_matrix* mats = sv.data();
  for (int i = 0; i < n; ++i)
    if ((rc = validate_shape(mats[i], true))) return rc;
  if (!workspace) return DION2_EWORKSPACE;
  std::lock_guard<std::mutex> lock(g_mu);
  ensure_device_attrs();
  // align the usable workspace base to 4 KiB (TMA / swizzle alignment)
  void* ws = reinterpret_cast<void*>(align_up(reinterpret_cast<uintptr_t>(workspace), 4096));
  const size_t slack = (uintptr_t)ws - (uintptr_t)workspace;
  std::string key = plan_key(mats, n, cfg, ws);
  auto it = g_plans.find(key);
  Plan* P;
  if (it == g_plans.end()) {
    auto np = std::make_unique<Plan>();
    rc = build_layout(*np, mats, n, cfg);
    if (rc) return rc;
    if (np->total - 4096 + slack > ws_bytes) return DION2_EWORKSPACE;
    rc = build_device_plan(*np, mats, cfg, ws);
    if (rc) return rc;
    np->id = g_next_plan_id++;
    P = np.get();
    g_plans[key] = std::move(np);
  } else {
    P = it->second.get();
    if (P->total - 4096 + slack > ws_bytes) return DION2_EWORKSPACE;
  }
  return run_step(*P, mats, cfg, ws, reinterpret_cast<cudaStream_t>(stream));
}

int dion2_step(const dion2_matrix* mat, const dion2_config* cfg, void* workspace, size_t ws_bytes, void* stream) {
  return dion2_step_batched(mat, 1, cfg, workspace, ws_bytes, stream);
}

int dion2_get_status(const void* workspace, void* stream, int32_t* first_bad_matrix) {
  if (!workspace) return DION2_EWORKSPACE;
  const void* ws = reinterpret_cast<const void*>(align_up(reinterpret_cast<uintptr_t>(workspace), 4096));
  int32_t st[2] = {0, 0};
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // pageable destination: the copy is stream-ordered and returns once it has completed
  if (cudaMemcpyAsync(st, ws, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess) return DION2_ECUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return DION2_ECUDA;
  if (first_bad_matrix) *first_bad_matrix = st[0] ? st[1] : -1;
  return st[0] ? DION2_ENONFINITE : DION2_OK;
}

int32_t dion2_release_workspace(const void* workspace, size_t bytes) {
  std::lock_guard<std::mutex> lock(g_mu);
  const uintptr_t lo = reinterpret_cast<uintptr_t>(workspace), hi = lo + bytes;
  cudaDeviceSynchronize();
  int dropped = 0;
  for (auto it = g_plans.begin(); it != g_plans.end();) {
    const uintptr_t w = reinterpret_cast<uintptr_t>(it->second->ws);
    if (w >= lo && w < hi) {
      it = g_plans.erase(it);
      ++dropped;
    } else {
      ++it;
    }
  }
  return dropped + release_dist_plans(lo, hi);
}

const char* dion2_strerror(int code) {
  switch (code) {
    case DION2_OK: return "ok";
    case DION2_EINVAL_CONFIG: return "invalid configuration";
    case DION2_EINVAL_SHAPE: return "invalid matrix shape or pointer";
    case DION2_EWORKSPACE: return "workspace missing or too small";
    case DION2_EUNSUPPORTED: return "unsupported configuration";
    case DION2_ECUDA: return "CUDA error";
    case DION2_ENCCL: return "NCCL error";
    case DION2_ENONFINITE: return "non-finite scores (matrix skipped)";
    default: return "unknown status";
  }
}

int dion2_set_phase_timing(int32_t enable) {
  std::lock_guard<std::mutex> lock(g_mu);
  g_timing = enable != 0;
  return DION2_OK;
}

int dion2_get_phase_times(float* ms_out, int32_t* launches_out, int32_t cap, int32_t* n_phases_out) {
  std::lock_guard<std::mutex> lock(g_mu);
  std::vector<float> ms(kNumPhases, 0.f);
  std::vector<int32_t> cnt(kNumPhases, 0);
  int rc = DION2_OK;
  for (auto& t : g_timed) {
    if (cudaEventSynchronize(t.b) != cudaSuccess) rc = DION2_ECUDA;
    float e = 0.f;
    cudaEventElapsedTime(&e, t.a, t.b);
    ms[t.phase] += e;
    cnt[t.phase] += 1;
    g_event_pool.push_back(t.a);
    g_event_pool.push_back(t.b);
  }
  g_timed.clear();
  for (int i = 0; i < std::min<int>(cap, kNumPhases); ++i) {
    if (ms_out) ms_out[i] = ms[i];
    if (launches_out) launches_out[i] = cnt[i];
  }
  if (n_phases_out) *n_phases_out = kNumPhases;
  return rc;
}

const char* dion2_phase_name(int32_t i) { return (i >= 0 && i < kNumPhases) ? kPhaseNames[i] : "?"; }

int32_t dion2_last_launch_count(void) { return g_last_launches; }

int32_t dion2_abi_version(void) { return DION2_ABI_VERSION; }

}  // extern "C"
