// dion2_dist.cu -- owner-compute distributed Dion2 step (include/dion2.h).
//
// Layout (per rank): every matrix j is sharded along its NON-selection axis, so the rank
// holds a slice of every selectable row (column).  The rank's piece of X_j = wide(M[K])
// is the column block X_j[:, rank*o/P : (rank+1)*o/P] (k x o/P), produced by the same
// streaming gather kernels as the single-GPU step (with X pointing into the send buffer),
// and consumed by the same scatter kernels (with the final X pointing into the receive
// buffer).  The owner of j assembles X_j from the P blocks, runs the tcgen05 NS engine
// of a regular single-GPU plan over its owned matrices, and splits X_T back.
//
// Transport: NCCL (ncclAllGather + grouped ncclSend/ncclRecv on the caller's stream,
// resolved with dlsym from the process's libnccl -- torch's), or "loopback" (all ranks in
// one process on one device; exchanges are device copies) for tests.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "runtime.h"
#include "symm.h"

using namespace dion2;

namespace dion2rt {
namespace {

// ------------------------------------------------------------------ NCCL (dlsym)
typedef int ncclResult_t;
typedef void* ncclComm_t;
constexpr int kNcclChar = 0, kNcclFloat32 = 7;
struct NcclApi {
  ncclResult_t (*allgather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*allreduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  bool ok = false;
};
NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.allgather = reinterpret_cast<decltype(a.allgather)>(dlsym(h, "ncclAllGather"));
    a.send = reinterpret_cast<decltype(a.send)>(dlsym(h, "ncclSend"));
    a.recv = reinterpret_cast<decltype(a.recv)>(dlsym(h, "ncclRecv"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
    a.allreduce = reinterpret_cast<decltype(a.allreduce)>(dlsym(h, "ncclAllReduce"));
    a.ok = a.allgather && a.send && a.recv && a.group_start && a.group_end && a.allreduce;
    return a;
  }();
  return api;
}

// ------------------------------------------------------------------ plan
struct DistMat {
  int64_t m, n;            // global shape
  int axis, d, o, k, qo;   // selection axis, its length, other length, selected, block width o/P
  int64_t srows, scols;    // local shard shape
  int owner;
  int chunk;               // owner chunk (C2 / NS / C3 rounds overlap by chunk)
  int64_t piece;           // bytes of one k x qo fp16 piece (256-B aligned)
  int64_t soff;            // offset of this matrix's piece inside its owner's section
  double flops;
  int path, ga, gb;
  int n_sumsq;
  int mt;                  // local M shard stored transposed (cols mode): K1 transpose-add, row gather
  size_t off_partials, off_sel, off_sumsq;
  // short X under AUTO (k <= kTinyP, reading R25): no pieces and no owner; every rank sums the
  // partial Gram matrices of its column block and applies the exact NS to it locally
  int tiny = 0;
  size_t off_tx = 0, off_to = 0;  // local scratch for K3's X store and the local X_T
};

struct DistPlan {
  DistPlan() = default;
  DistPlan(const DistPlan&) = delete;
  DistPlan& operator=(const DistPlan&) = delete;
  ~DistPlan() {
    if (dtab) cudaFree(dtab);
  }
  void* ws = nullptr;  // aligned workspace base of the plan (dion2_release_workspace)
  int n = 0, world = 1, rank = 0;
  std::vector<DistMat> dm;
  int64_t total_d = 0;
  // workspace offsets
  size_t off_status, off_bad, off_scores, off_scores_all, off_sumsq_local, off_sumsq_all, off_nsscale, off_send,
      off_recv, off_osend, off_orecv, off_owner, total;
  std::vector<int64_t> sdispl, scount;  // per owner: my send section
  int64_t R = 0;                         // bytes per rank section of my recv / osend buffers
  // device tables (plan-owned)
  std::vector<uint8_t> htab;
  void* dtab = nullptr;
  // streaming lists: gather and scatter membership differ for transposed-M column matrices
  // (row gather on M^T, column scatter on W)
  size_t t_desc, t_rowmats, t_rowprefix, t_colmats, t_colprefix, t_mtmats, t_mtprefix, t_allcols, t_flgm[2],
      t_flsm[2], t_flg[2], t_fls[2], t_gprefix;
  int n_row_mats = 0, n_col_mats = 0, n_mt_mats = 0, n_allcols = 0, fl_gn[2] = {0, 0}, fl_sn[2] = {0, 0},
      fl_gunits[2] = {0, 0}, fl_sunits[2] = {0, 0}, fl_maxk = 0, max_d = 0, total_gather_tiles = 0;
  int64_t total_rows = 0, total_col_tiles = 0, total_mt_tiles = 0, max_cols_col = 0;
  std::vector<const void*> last_ptrs;
  bool uploaded = false;
  // owner side, in chunks: the exchange to the owners (C2), the owner's NS and the exchange
  // back (C3) run chunk by chunk on two streams, so C2 of chunk c + 1 and C3 of chunk c - 1
  // overlap the NS of chunk c.  Every owner's send section is ordered by (chunk, NS shape group,
  // index); cdispl[o][c] is chunk c's offset inside owner o's section (same on every rank).
  int nchunks = 1;
  std::vector<std::vector<int64_t>> cdispl;
  struct OwnerChunk {
    std::vector<int> owned;        // global matrix indices (index order)
    std::unique_ptr<Plan> plan;    // NS plan over their global shapes
    size_t off = 0;                // workspace offset of the plan
    PieceTable ptab{};
    size_t t_gidx = 0, t_roff = 0, t_inpl = 0, t_pmaps = 0;
    int max_p_pad = 0, max_k = 0;
    bool all_inplace = false;      // every matrix's NS reads and writes the exchange pieces in place
    bool all_inplace_in = false;   // ... reads them in place
  };
  std::vector<OwnerChunk> oc;
  // Direct peer exchange (DION2_FLAG_DIST_DIRECT, k_symm.cu): K3 pushes each piece straight into
  // its owner's receive buffer and K7 pulls its piece of O straight from the owner's outgoing
  // buffer (peer_recv / peer_osend: every rank's buffers as addressable here -- NCCL symmetric
  // windows, or the other loopback ranks' workspaces); recv_base / osend_base are this rank's
  // own (owner-side) buffers in either mode.
  int direct = 0;
  int64_t win_bytes = 0;  // max over owners of scount * world (same on every rank)
  uint8_t* recv_base = nullptr;
  uint8_t* osend_base = nullptr;
  std::vector<uint8_t*> peer_recv, peer_osend;
  SymmState* symm = nullptr;  // NCCL windows; kept for the process lifetime (collective teardown)
  // short X (DistMat::tiny): the p <= 64 matrices first, then 64 < p <= 128
  std::vector<int32_t> tiny_list;
  int n_tiny64 = 0;
  size_t off_tiny_a = 0, t_tiny = 0;
};

void* dt(DistPlan& D, size_t off) { return static_cast<uint8_t*>(D.dtab) + off; }

int resolve(DistPlan& D, const dion2_shard* sh, int n, const dion2_config* c, int world, int rank) {
  if (world < 1 || rank < 0 || rank >= world || n < 1 || !sh) return DION2_EINVAL_SHAPE;
  if (c->precision != DION2_NS_BF16 || c->decay_mode != 0) return DION2_EUNSUPPORTED;
  D.n = n;
  D.world = world;
  D.rank = rank;
  D.dm.assign(n, DistMat{});
  for (int j = 0; j < n; ++j) {
    DistMat& q = D.dm[j];
    q.m = sh[j].rows;
    q.n = sh[j].cols;
    if (q.m < 1 || q.n < 1) return DION2_EINVAL_SHAPE;
    q.axis = c->axis == DION2_AXIS_AUTO ? (q.m <= q.n ? DION2_AXIS_ROWS : DION2_AXIS_COLS) : c->axis;
    q.d = (int)(q.axis == DION2_AXIS_ROWS ? q.m : q.n);
    q.o = (int)(q.axis == DION2_AXIS_ROWS ? q.n : q.m);
    if (q.d > DION2_MAX_SELECT_DIM) return DION2_EINVAL_SHAPE;
    int64_t k = (int64_t)std::floor((double)c->alpha * (double)q.d + 0.5);  // reading R7
    q.k = (int)std::max<int64_t>(1, std::min<int64_t>(k, q.d));
    if (q.k > q.o || q.o % world) return DION2_EUNSUPPORTED;
    q.qo = q.o / world;
    if (q.axis == DION2_AXIS_ROWS) {
      if (q.qo % 8) return DION2_EUNSUPPORTED;
      q.srows = q.m;
      q.scols = q.qo;
    } else {
      if (q.qo % 8) return DION2_EUNSUPPORTED;
      q.srows = q.qo;
      q.scols = q.n;
    }
    if (sh[j].ld < q.scols) return DION2_EINVAL_SHAPE;
    if (sh[j].reserved != 0 || (sh[j].m_transposed != 0 && sh[j].m_transposed != 1)) return DION2_EINVAL_SHAPE;
    q.mt = sh[j].m_transposed;
    if (q.mt && q.axis != DION2_AXIS_COLS) return DION2_EUNSUPPORTED;
    if (q.mt && sh[j].ldm < q.srows) return DION2_EINVAL_SHAPE;
    q.piece = (int64_t)align_up((size_t)q.k * q.qo * 2, 256);
    q.tiny = (c->ns_form == DION2_NS_FORM_AUTO && c->precision == DION2_NS_BF16 && q.k <= kTinyP) ? 1 : 0;
    if (q.tiny) q.piece = 0;
    const double p = q.k, qq = q.o;
    q.flops = c->ns_steps * (4.0 * p * p * qq + 2.0 * p * p * p);
    // gather/scatter path: streaming rows (1), streaming cols (2), generic tiles (0)
    q.path = q.axis == DION2_AXIS_ROWS ? 1 : ((q.qo % 32 == 0 && q.k <= kMaxColKFast) ? 2 : 0);
    q.ga = q.path == 0 ? (int)ceil_div(q.srows, kTileA) : 0;
    q.gb = q.path == 0 ? (int)ceil_div(q.k, kTileB) : 0;
    q.n_sumsq = (q.path == 1 || q.mt) ? q.k : (q.path == 2 ? q.qo / 32 : q.ga * q.gb);
  }
  // owners: LPT on NS FLOPs (descending, ties -> lower index), least-loaded rank (ties -> lower rank)
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return D.dm[a].flops > D.dm[b].flops; });
  std::vector<double> load(world, 0.0);
  for (int j : order) {
    int best = 0;
    for (int r = 1; r < world; ++r)
      if (load[r] < load[best]) best = r;
    D.dm[j].owner = best;
    load[best] += D.dm[j].flops;
  }
  // owner chunks (DION2_DIST_CHUNKS, default 1): each owner's matrices in descending NS FLOPs
  // (ties -> lower index) dealt round-robin to the chunks.  Measured in loopback on the 1B set
  // (scripts/ab_dist_chunks.sh): 1 / 2 / 3 chunks -> 3.14 / 3.37 / 3.48 ms per rank at P = 2,
  // 1.26 / 1.48 / 1.64 at P = 8 -- half-size NS batches (9 matrices per chunk at P = 8, under
  // one wave) lose more than the overlapped exchange can win (~0.15 ms of NVLink per rank at
  // P = 8), so the overlap is opt-in.
  const char* ce = getenv("DION2_DIST_CHUNKS");
  D.direct = (c->reserved0 & DION2_FLAG_DIST_DIRECT) ? 1 : 0;
  D.nchunks = (world > 1 && !D.direct) ? std::max(1, ce ? atoi(ce) : 1) : 1;
  for (int o = 0; o < world; ++o) {
    int t = 0;
    for (int j : order)
      if (D.dm[j].owner == o) D.dm[j].chunk = (t++) % D.nchunks;
  }
  // send sections (by owner) and my recv section size
  D.sdispl.assign(world, 0);
  D.scount.assign(world, 0);
  D.cdispl.assign(world, std::vector<int64_t>(D.nchunks + 1, 0));
  // Inside an owner's section the pieces are ordered by chunk, then by the owner chunk plan's NS
  // shape groups ((p_pad, q_pad) in first-appearance order, members in index order), so a
  // group's pieces from one rank form a uniform [matrix][k][qo] array the owner's NS kernels can
  // address with one tensor map per rank (in-place pieces, build_tables).  Shapes only: the
  // same on every rank.
  int64_t run = 0;
  for (int o = 0; o < world; ++o) {
    D.sdispl[o] = run;
    for (int ch = 0; ch < D.nchunks; ++ch) {
      D.cdispl[o][ch] = run - D.sdispl[o];
      std::vector<int> mine;
      std::vector<std::pair<int64_t, int64_t>> keys;
      std::vector<int> key_of;
      for (int j = 0; j < n; ++j)
        if (D.dm[j].owner == o && D.dm[j].chunk == ch && !D.dm[j].tiny) {
          const std::pair<int64_t, int64_t> key((int64_t)align_up(D.dm[j].k, 256), (int64_t)align_up(D.dm[j].o, 256));
          int ki = (int)(std::find(keys.begin(), keys.end(), key) - keys.begin());
          if (ki == (int)keys.size()) keys.push_back(key);
          mine.push_back(j);
          key_of.push_back(ki);
        }
      std::vector<int> ord(mine.size());
      std::iota(ord.begin(), ord.end(), 0);
      std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return key_of[a] < key_of[b]; });
      for (int t : ord) {
        const int j = mine[t];
        D.dm[j].soff = run - D.sdispl[o];
        run += D.dm[j].piece;
      }
    }
    D.cdispl[o][D.nchunks] = run - D.sdispl[o];
    D.scount[o] = run - D.sdispl[o];
  }
  D.R = D.scount[rank];
  D.win_bytes = 0;
  for (int o = 0; o < world; ++o) D.win_bytes = std::max<int64_t>(D.win_bytes, D.scount[o] * world);
  D.oc.clear();
  D.oc.resize(D.nchunks);
  for (int j = 0; j < n; ++j)
    if (D.dm[j].owner == rank && !D.dm[j].tiny) D.oc[D.dm[j].chunk].owned.push_back(j);
  // workspace
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 1), 256);
    return o;
  };
  D.total_d = 0;
  for (auto& q : D.dm) D.total_d += q.d;
  D.off_status = take(16);
  D.off_bad = take(4 * (size_t)n);
  D.off_scores = take(4 * (size_t)D.total_d);
  D.off_scores_all = take(4 * (size_t)D.total_d * world);
  D.off_sumsq_local = take(4 * (size_t)n);
  D.off_sumsq_all = take(4 * (size_t)n * world);
  D.off_nsscale = take(16 * (size_t)n);  // per matrix: word 2 = the fp16 prescale K2 writes (R24)
  D.tiny_list.clear();
  for (int pass = 0; pass < 2; ++pass)
    for (int j = 0; j < n; ++j)
      if (D.dm[j].tiny && ((D.dm[j].k <= 64) == (pass == 0))) D.tiny_list.push_back(j);
  D.n_tiny64 = 0;
  for (int j : D.tiny_list) D.n_tiny64 += D.dm[j].k <= 64 ? 1 : 0;
  D.off_tiny_a = take(8 * (size_t)kTinyP * kTinyP * std::max<size_t>(1, D.tiny_list.size()));
  for (auto& q : D.dm)
    if (q.tiny) {
      q.off_tx = take((size_t)q.k * q.qo * 2);
      q.off_to = take((size_t)q.k * q.qo * 2);
    }
  for (auto& q : D.dm) {
    q.off_partials = q.axis == DION2_AXIS_COLS ? take(4 * (size_t)ceil_div(q.srows, kColRowBlock) * q.scols) : 0;
    q.off_sel = take(4 * (size_t)q.k);
    q.off_sumsq = take(4 * (size_t)q.n_sumsq);
  }
  D.off_send = take((size_t)run);
  D.off_orecv = take((size_t)run);
  D.off_recv = take((size_t)D.R * world);
  D.off_osend = take((size_t)D.R * world);
  off = align_up(off, 4096);
  D.off_owner = off;
  // one owner plan per chunk over its matrices' GLOBAL shapes (NS only)
  size_t owner_bytes = 0;
  for (auto& ch : D.oc) {
    ch.off = D.off_owner + owner_bytes;
    if (ch.owned.empty()) continue;
    std::vector<dion2_matrix> om(ch.owned.size());
    for (size_t i = 0; i < ch.owned.size(); ++i) {
      memset(&om[i], 0, sizeof(om[i]));
      om[i].rows = D.dm[ch.owned[i]].m;
      om[i].cols = D.dm[ch.owned[i]].n;
      om[i].ld = D.dm[ch.owned[i]].n;
    }
    ch.plan = std::make_unique<Plan>();
    ch.plan->no_tiny = true;  // the owner's X arrives as fp16 pieces: the tensor-core NS handles every group
    int rc = build_layout(*ch.plan, om.data(), (int)om.size(), c);
    if (rc) return rc;
    owner_bytes = align_up(owner_bytes + ch.plan->total, 4096);
  }
  D.total = D.off_owner + owner_bytes + 4096;
  return DION2_OK;
}

// Device tables + owner plan for a concrete workspace.
int build_tables(DistPlan& D, const dion2_config* c, void* ws) {
  const int n = D.n, P = D.world;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 1), 256);
    return o;
  };
  D.t_desc = take(sizeof(MatDesc) * n);
  D.t_rowmats = take(4 * (size_t)n);
  D.t_rowprefix = take(8 * (size_t)n);
  D.t_colmats = take(4 * (size_t)n);
  D.t_colprefix = take(8 * (size_t)n);
  D.t_mtmats = take(4 * (size_t)n);
  D.t_mtprefix = take(8 * (size_t)n);
  D.t_allcols = take(4 * (size_t)n);
  for (int l = 0; l < 2; ++l) {
    D.t_flgm[l] = take(4 * (size_t)n);
    D.t_flsm[l] = take(4 * (size_t)n);
    D.t_flg[l] = take(4 * (size_t)n);
    D.t_fls[l] = take(4 * (size_t)n);
  }
  D.t_gprefix = take(4 * (size_t)n);
  D.t_tiny = take(4 * std::max<size_t>(1, D.tiny_list.size()));
  for (auto& ch : D.oc) {
    ch.t_gidx = take(4 * std::max<size_t>(1, ch.owned.size()));
    ch.t_roff = take(8 * std::max<size_t>(1, ch.owned.size()) * P);
    ch.t_inpl = take(4 * std::max<size_t>(1, ch.owned.size()));
    const size_t ng = ch.plan ? ch.plan->groups.size() : 0;
    ch.t_pmaps = take(sizeof(CUtensorMap) * std::max<size_t>(1, ng * 3 * (size_t)P));
  }
  D.htab.assign(off, 0);
  if (!D.dtab && cudaMalloc(&D.dtab, off) != cudaSuccess) return DION2_ECUDA;
  auto H = [&](size_t o) { return D.htab.data() + o; };
  MatDesc* md = reinterpret_cast<MatDesc*>(H(D.t_desc));
  std::vector<int32_t> rowmats, colmats, mtmats, allcols, flgm[2], flsm[2], flg[2], fls[2];
  std::vector<int64_t> rowprefix, colprefix, mtprefix;
  std::vector<int32_t> gprefix(n, 0);
  D.total_gather_tiles = 0;
  D.total_rows = D.total_col_tiles = D.total_mt_tiles = 0;
  D.fl_gunits[0] = D.fl_gunits[1] = D.fl_sunits[0] = D.fl_sunits[1] = 0;
  D.fl_maxk = D.max_d = 0;
  D.max_cols_col = 0;
  int64_t score_off = 0;
  for (int j = 0; j < n; ++j) {
    const DistMat& q = D.dm[j];
    MatDesc& d = md[j];
    memset(&d, 0, sizeof(d));
    d.rows = q.srows;
    d.cols = q.scols;
    d.axis = q.axis;
    d.d = q.d;
    d.o = q.qo;
    d.k = q.k;
    d.sr = q.axis == DION2_AXIS_ROWS ? q.k : (int)q.srows;
    d.sc = q.axis == DION2_AXIS_ROWS ? (int)q.scols : q.k;
    d.transposed = q.axis == DION2_AXIS_COLS;  // the GLOBAL wide orientation (k <= o)
    d.p = q.k;
    d.q = q.qo;
    d.p_pad = q.k;
    d.q_pad = q.qo;
    d.sa_pad = d.sr;
    d.sb_pad = d.sc;
    d.grad_bf16 = c->grad_dtype == DION2_DT_BF16;
    d.update_scale = c->scale_mode == 0 ? (float)std::sqrt((double)q.m / (double)q.n)        // Alg. 1 l.6
                                        : (float)std::sqrt(q.axis == DION2_AXIS_ROWS ? (double)q.k / q.n
                                                                                     : (double)q.m / q.k);
    d.scores = (float*)at(ws, D.off_scores) + score_off;
    d.col_partials = q.axis == DION2_AXIS_COLS ? (float*)at(ws, q.off_partials) : nullptr;
    d.sel = (int32_t*)at(ws, q.off_sel);
    d.sumsq_partials = (float*)at(ws, q.off_sumsq);
    d.ns_scale = (float*)at(ws, D.off_nsscale) + 4 * j;
    d.x16 = 1;
    d.X0 = q.tiny ? at(ws, q.off_tx) : at(ws, D.off_send + D.sdispl[q.owner] + q.soff);
    d.X1 = q.tiny ? at(ws, q.off_to) : at(ws, D.off_orecv + D.sdispl[q.owner] + q.soff);
    d.final_in_x1 = 1;
    d.rowblocks = (int)ceil_div(q.srows, kColRowBlock);
    d.mid = j;
    d.path = q.path;
    d.n_sumsq = q.n_sumsq;
    d.mt = q.mt;
    d.scores_final = 1;
    d.gather_tile_base = D.total_gather_tiles;
    d.gather_tiles_a = q.ga;
    d.gather_tiles_b = q.gb;
    gprefix[j] = D.total_gather_tiles;
    D.total_gather_tiles += q.ga * q.gb;
    score_off += q.d;
    D.max_d = std::max(D.max_d, q.d);
    if (q.axis == DION2_AXIS_ROWS) {
      rowmats.push_back(j);
      rowprefix.push_back(D.total_rows);
      D.total_rows += q.srows;
    } else {
      allcols.push_back(j);
      D.max_cols_col = std::max<int64_t>(D.max_cols_col, q.scols);
      if (q.mt) {
        mtmats.push_back(j);
        mtprefix.push_back(D.total_mt_tiles);
        D.total_mt_tiles += (int64_t)d.rowblocks * ceil_div(q.scols, 64);
      } else {
        colmats.push_back(j);
        colprefix.push_back(D.total_col_tiles);
        D.total_col_tiles += (int64_t)d.rowblocks * ceil_div(q.scols, 256);
      }
    }
    // gather: rows streaming (rows mode, or transposed-M columns = rows of M^T), cols streaming,
    // or generic tiles; scatter: by path
    const int lg = (d.path == 1 || q.mt) ? 0 : d.path - 1;
    const int ls = d.path - 1;
    if (lg >= 0) {
      flgm[lg].push_back(j);
      flg[lg].push_back(D.fl_gunits[lg]);
      D.fl_gunits[lg] += lg == 0 ? q.k : q.qo / 32;
    }
    if (ls >= 0) {
      flsm[ls].push_back(j);
      fls[ls].push_back(D.fl_sunits[ls]);
      D.fl_sunits[ls] += ls == 0 ? q.k : q.qo / 32;
    }
    if (lg == 1 || ls == 1) D.fl_maxk = std::max(D.fl_maxk, q.k);
  }
  memcpy(H(D.t_gprefix), gprefix.data(), 4 * (size_t)n);
  if (!D.tiny_list.empty()) memcpy(H(D.t_tiny), D.tiny_list.data(), 4 * D.tiny_list.size());
  D.n_row_mats = (int)rowmats.size();
  D.n_col_mats = (int)colmats.size();
  D.n_mt_mats = (int)mtmats.size();
  D.n_allcols = (int)allcols.size();
  if (D.n_mt_mats) {
    memcpy(H(D.t_mtmats), mtmats.data(), 4 * mtmats.size());
    memcpy(H(D.t_mtprefix), mtprefix.data(), 8 * mtprefix.size());
  }
  if (D.n_allcols) memcpy(H(D.t_allcols), allcols.data(), 4 * allcols.size());
  if (D.n_row_mats) {
    memcpy(H(D.t_rowmats), rowmats.data(), 4 * rowmats.size());
    memcpy(H(D.t_rowprefix), rowprefix.data(), 8 * rowprefix.size());
  }
  if (D.n_col_mats) {
    memcpy(H(D.t_colmats), colmats.data(), 4 * colmats.size());
    memcpy(H(D.t_colprefix), colprefix.data(), 8 * colprefix.size());
  }
  for (int l = 0; l < 2; ++l) {
    D.fl_gn[l] = (int)flgm[l].size();
    D.fl_sn[l] = (int)flsm[l].size();
    if (D.fl_gn[l]) {
      memcpy(H(D.t_flgm[l]), flgm[l].data(), 4 * flgm[l].size());
      memcpy(H(D.t_flg[l]), flg[l].data(), 4 * flg[l].size());
    }
    if (D.fl_sn[l]) {
      memcpy(H(D.t_flsm[l]), flsm[l].data(), 4 * flsm[l].size());
      memcpy(H(D.t_fls[l]), fls[l].data(), 4 * fls[l].size());
    }
  }
  // owner chunk plans + piece tables
  for (auto& ch : D.oc) {
    ch.max_p_pad = ch.max_k = 0;
    if (ch.owned.empty()) continue;
    Plan& OP = *ch.plan;
    std::vector<dion2_matrix> om(ch.owned.size());
    for (size_t i = 0; i < ch.owned.size(); ++i) {
      memset(&om[i], 0, sizeof(om[i]));
      om[i].rows = D.dm[ch.owned[i]].m;
      om[i].cols = D.dm[ch.owned[i]].n;
      om[i].ld = D.dm[ch.owned[i]].n;
    }
    int rc = build_device_plan(OP, om.data(), c, at(ws, ch.off));
    if (rc) return rc;
    std::vector<int32_t> gidx(ch.owned.size());
    std::vector<int64_t> roff(ch.owned.size() * P);
    for (size_t i = 0; i < ch.owned.size(); ++i) {
      const DistMat& q = D.dm[ch.owned[i]];
      gidx[i] = ch.owned[i];
      for (int r = 0; r < P; ++r) roff[i * P + r] = q.soff;
      ch.max_p_pad = std::max(ch.max_p_pad, OP.mp[i].p_pad);
      ch.max_k = std::max(ch.max_k, q.k);
      // the owner's NS runs on the global orientation: X = k x o (k <= o)
      if (OP.mp[i].p != q.k || OP.mp[i].q != q.o) return DION2_EUNSUPPORTED;
    }
    memcpy(H(ch.t_gidx), gidx.data(), 4 * gidx.size());
    memcpy(H(ch.t_roff), roff.data(), 8 * roff.size());
    // In-place pieces: a Gram-space owner group whose q is a whole number of 256-column tiles
    // and of 64-column k-blocks per rank piece (q_pad == q, qo % 64 == 0, P <= 8) has its gram
    // and apply read X0 straight from the received pieces and its apply write X_T straight into
    // the outgoing pieces (no assemble / disassemble copies); other groups are copied.
    std::vector<int32_t> inpl(ch.owned.size(), 0);
    const bool inplace_on = P <= kMaxPieceRanks;
    CUtensorMap* hmaps = reinterpret_cast<CUtensorMap*>(H(ch.t_pmaps));
    std::vector<int> g_ok(OP.groups.size(), 0);
    for (size_t gi = 0; gi < OP.groups.size() && inplace_on; ++gi) {
      const Group& g = OP.groups[gi];
      if (!g.gs) continue;
      const DistMat& q0 = D.dm[ch.owned[g.mats[0]]];
      bool ok = true;
      for (size_t zi = 0; zi < g.mats.size() && ok; ++zi) {
        const DistMat& q = D.dm[ch.owned[g.mats[zi]]];
        ok = q.o == g.q_pad && q.qo % 64 == 0 && q.k == q0.k && q.qo == q0.qo && q.piece == q0.piece &&
             q.soff == q0.soff + (int64_t)zi * q0.piece;
      }
      if (!ok) continue;
      for (int r = 0; r < P; ++r) {
        uint8_t* rb = D.recv_base + (int64_t)r * D.R + q0.soff;
        uint8_t* sb = D.osend_base + (int64_t)r * D.R + q0.soff;
        CUtensorMap* m = hmaps + gi * 3 * P;
        if (!make_map_strided(&m[r], rb, q0.qo, q0.k, g.count, q0.piece, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
            !make_map_strided(&m[P + r], rb, q0.qo, q0.k, g.count, q0.piece, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B) ||
            !make_map_strided(&m[2 * P + r], sb, q0.qo, q0.k, g.count, q0.piece, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
          return DION2_ECUDA;
      }
      g_ok[gi] = 1;
      for (int i : g.mats) inpl[i] = 1;
    }
    // point the owner plan's launches that read X0 (the first gram: A = B = X0; the first apply:
    // B = X0) at the received pieces, and the last apply (D = X_T) at the outgoing pieces
    // (the last segment's apply reads X0 after an odd number of restart segments, else X1)
    const bool last_reads_x0 = ns_segments(c, c->ns_steps).size() & 1;
    for (int li = 0; li < (int)OP.ns_launches.size(); ++li) {
      Launch& ln = OP.ns_launches[li];
      if (ln.phase != PH_GRAM && ln.phase != PH_APPLY) continue;
      for (int j = 0; j < ln.tc.p.ngroups; ++j) {
        NsGroup& G = ln.tc.p.g[j];
        for (size_t gi = 0; gi < OP.groups.size(); ++gi) {
          if (!g_ok[gi]) continue;
          const Group& og = OP.groups[gi];
          const void* x0 = at(at(ws, ch.off), og.off_X0);
          const void* x1 = at(at(ws, ch.off), og.off_X1);
          // this entry belongs to group gi iff it reads or writes one of gi's X buffers
          const bool mine = ln.phase == PH_GRAM ? (G.a == x0 || G.a == x1) : (G.b == x0 || G.b == x1);
          if (!mine) continue;
          const bool load = ln.phase == PH_GRAM ? G.a == x0 : G.b == x0;
          const bool store = ln.phase == PH_APPLY && G.b == (last_reads_x0 ? x0 : x1);
          if (!load && !store) continue;
          const DistMat& q0 = D.dm[ch.owned[og.mats[0]]];
          G.pieces_qo = q0.qo;
          G.pieces_P = P;
          G.pieces_map = (int)(gi * 3 * P);
          G.pieces_load = load ? 1 : 0;
          G.pieces_store = store ? 1 : 0;
          for (int k = 0; k < 3 * P; ++k) ln.tc.mapP[j][k] = hmaps[gi * 3 * P + k];
        }
      }
    }
    memcpy(H(ch.t_inpl), inpl.data(), 4 * inpl.size());
    ch.all_inplace = std::all_of(inpl.begin(), inpl.end(), [](int32_t v) { return v == 1; });
    ch.all_inplace_in = std::all_of(inpl.begin(), inpl.end(), [](int32_t v) { return v != 0; });
    ch.ptab.inplace = (const int32_t*)dt(D, ch.t_inpl);
    ch.ptab.gidx = (const int32_t*)dt(D, ch.t_gidx);
    ch.ptab.roff = (const int64_t*)dt(D, ch.t_roff);
    ch.ptab.rstride = D.R;
    ch.ptab.world = P;
  }
  return DION2_OK;
}

std::map<std::string, std::unique_ptr<DistPlan>> g_dist_plans;
std::map<const void*, int> g_last_mode;  // aligned workspace -> exchange mode of its last step

// Direct mode: point K3's piece destination (X0) at the owner's receive buffer and K7's piece
// source (X1) at the owner's outgoing buffer, section `rank` (the owner's layout:
// rank * scount[owner] + soff, the offsets the NCCL exchange would copy between).
void apply_direct(DistPlan& D) {
  MatDesc* md = reinterpret_cast<MatDesc*>(D.htab.data() + D.t_desc);
  for (int j = 0; j < D.n; ++j) {
    const DistMat& q = D.dm[j];
    if (q.tiny) continue;  // local, no pieces
    const int64_t off = (int64_t)D.rank * D.scount[q.owner] + q.soff;
    void* x0 = D.peer_recv[q.owner] + off;
    void* x1 = D.peer_osend[q.owner] + off;
    if (md[j].X0 != x0 || md[j].X1 != x1) {
      md[j].X0 = x0;
      md[j].X1 = x1;
      D.uploaded = false;
    }
  }
}

std::string dist_key(const dion2_shard* sh, int n, const dion2_config* c, int world, int rank, void* ws,
                     void* comm = nullptr) {
  std::string k;
  auto put = [&](const void* p, size_t s) { k.append(reinterpret_cast<const char*>(p), s); };
  put(&n, 4);
  put(&world, 4);
  put(&rank, 4);
  put(&ws, sizeof ws);
  for (int i = 0; i < n; ++i) {
    put(&sh[i].rows, 8);
    put(&sh[i].cols, 8);
    put(&sh[i].ld, 8);
    put(&sh[i].m_transposed, 4);
  }
  put(&c->alpha, 4);
  put(&c->ns_steps, 4);
  put(c->ns_coeffs, sizeof(float) * 3 * c->ns_steps);
  put(&c->axis, 4);
  put(&c->precision, 4);
  put(&c->grad_dtype, 4);
  put(&c->w_dtype, 4);
  put(&c->decay_mode, 4);
  put(&c->scale_mode, 4);
  put(&c->ns_form, 4);  // shapes the owner's NS plan
  const int direct = (c->reserved0 & DION2_FLAG_DIST_DIRECT) ? 1 : 0;
  put(&direct, 4);
  if (direct) put(&comm, sizeof comm);  // the symmetric windows belong to one communicator
  k += env_key();
  return k;
}

int get_plan(DistPlan** out, const dion2_shard* sh, int n, const dion2_config* c, int world, int rank, void* workspace,
             size_t ws_bytes, void* comm = nullptr, cudaStream_t s = nullptr) {
  void* ws = reinterpret_cast<void*>(align_up(reinterpret_cast<uintptr_t>(workspace), 4096));
  const size_t slack = (uintptr_t)ws - (uintptr_t)workspace;
  std::string key = dist_key(sh, n, c, world, rank, ws, comm);
  auto it = g_dist_plans.find(key);
  if (it == g_dist_plans.end()) {
    auto D = std::make_unique<DistPlan>();
    int rc = resolve(*D, sh, n, c, world, rank);
    if (rc) return rc;
    if (D->total - 4096 + slack > ws_bytes) return DION2_EWORKSPACE;
    D->recv_base = static_cast<uint8_t*>(at(ws, D->off_recv));
    D->osend_base = static_cast<uint8_t*>(at(ws, D->off_osend));
    if (D->direct && comm) {  // NCCL: the owner-side buffers are the symmetric windows
      rc = symm_create(comm, world, (size_t)D->win_bytes, s, &D->symm, &D->recv_base, &D->osend_base, D->peer_recv,
                       D->peer_osend);
      // EUNSUPPORTED is decided before any collective call, identically on every rank (no
      // device API in this NCCL, or ranks outside one NVLink domain): fall back to send / recv
      if (rc == DION2_EUNSUPPORTED) {
        D->direct = 0;
        D->recv_base = static_cast<uint8_t*>(at(ws, D->off_recv));
        D->osend_base = static_cast<uint8_t*>(at(ws, D->off_osend));
      } else if (rc) {
        return rc;
      }
    }
    rc = build_tables(*D, c, ws);
    if (rc) return rc;
    if (D->direct && comm) apply_direct(*D);
    D->ws = ws;
    it = g_dist_plans.emplace(key, std::move(D)).first;
  }
  DistPlan& D = *it->second;
  if (D.total - 4096 + slack > ws_bytes) return DION2_EWORKSPACE;
  *out = &D;
  return DION2_OK;
}

// refresh the caller's shard pointers in the device table (upload only when they change)
int refresh(DistPlan& D, const dion2_shard* sh, const dion2_config* c, cudaStream_t s) {
  bool up = !D.uploaded;
  if ((int)D.last_ptrs.size() != 5 * D.n) {
    D.last_ptrs.assign(5 * D.n, nullptr);
    up = true;
  }
  MatDesc* md = reinterpret_cast<MatDesc*>(D.htab.data() + D.t_desc);
  for (int j = 0; j < D.n; ++j) {
    const void* p[5] = {sh[j].W, sh[j].M, sh[j].G, sh[j].sel_out,
                        reinterpret_cast<const void*>((uintptr_t)(sh[j].m_transposed ? sh[j].ldm : 0))};
    for (int t = 0; t < 5; ++t)
      if (D.last_ptrs[5 * j + t] != p[t]) { up = true; D.last_ptrs[5 * j + t] = p[t]; }
    md[j].W = sh[j].W;
    md[j].M = sh[j].M;
    md[j].G = sh[j].G;
    md[j].sel_out = sh[j].sel_out;
    md[j].O_out = nullptr;
    md[j].ld = sh[j].ld;
    md[j].ldm = sh[j].m_transposed ? sh[j].ldm : 0;
    const size_t gel = c->grad_dtype == DION2_DT_BF16 ? 2 : 4;
    md[j].vec4 = ((uintptr_t)sh[j].W % (c->w_dtype == DION2_DT_BF16 ? 8 : 16) == 0) && ((uintptr_t)sh[j].M % 16 == 0) &&
                 ((uintptr_t)sh[j].G % (gel == 4 ? 16 : 8) == 0) && (sh[j].ld % 4 == 0) &&
                 (!sh[j].m_transposed || sh[j].ldm % 4 == 0);
  }
  if (up) {
    if (cudaMemcpyAsync(D.dtab, D.htab.data(), D.htab.size(), cudaMemcpyHostToDevice, s) != cudaSuccess)
      return DION2_ECUDA;
    for (auto& ch : D.oc)
      if (ch.plan && cudaMemcpyAsync(ch.plan->dtab, ch.plan->host_tables.data(), ch.plan->host_tables.size(),
                                     cudaMemcpyHostToDevice, s) != cudaSuccess)
        return DION2_ECUDA;
    D.uploaded = true;
  }
  return DION2_OK;
}

// ------------------------------------------------------------------ phases (one rank)
void phase_local_k1(DistPlan& D, void* ws, Launcher& L, cudaStream_t s) {
  const int sms = g_sm_count > 0 ? g_sm_count : 148;
  const MatDesc* dm = (const MatDesc*)dt(D, D.t_desc);
  cudaMemsetAsync(at(ws, D.off_status), 0, 4, s);
  cudaMemsetAsync(at(ws, D.off_status + 4), 0x7f, 4, s);
  if (D.n_row_mats) {
    L.begin(PH_K1);
    const int64_t blocks = std::min<int64_t>(ceil_div(D.total_rows, 8), (int64_t)sms * 8);
    k_momentum_score_rows<<<(unsigned)blocks, 256, 0, s>>>(dm, (const int32_t*)dt(D, D.t_rowmats),
                                                           (const int64_t*)dt(D, D.t_rowprefix), D.n_row_mats,
                                                           D.total_rows);
    L.end();
  }
  if (D.n_col_mats) {
    L.begin(PH_K1);
    const int64_t blocks = std::min<int64_t>(D.total_col_tiles, (int64_t)sms * 8);
    k_momentum_score_cols<<<(unsigned)blocks, 256, 0, s>>>(dm, (const int32_t*)dt(D, D.t_colmats),
                                                           (const int64_t*)dt(D, D.t_colprefix), D.n_col_mats,
                                                           D.total_col_tiles);
    L.end();
  }
  if (D.n_mt_mats) {
    L.begin(PH_K1_MT);
    const int64_t blocks = std::min<int64_t>(D.total_mt_tiles, (int64_t)sms * 8);
    launch_k1_mt(reinterpret_cast<const MatDesc*>(D.htab.data() + D.t_desc), D.n,
                 reinterpret_cast<const MatDesc*>(D.htab.data() + D.t_desc)->grad_bf16 ? DION2_DT_BF16 : DION2_DT_F32,
                 D.total_mt_tiles,
                 (int)blocks, s, dm, (const int32_t*)dt(D, D.t_mtmats), (const int64_t*)dt(D, D.t_mtprefix),
                 D.n_mt_mats);
    L.end();
  }
  if (D.n_allcols) {
    L.begin(PH_K1);
    launch_cols_local_scores(s, dm, (const int32_t*)dt(D, D.t_allcols), D.n_allcols, D.max_cols_col);
    L.end();
  }
}

void phase_select(DistPlan& D, void* ws, const dion2_config* c, Launcher& L, cudaStream_t s) {
  const MatDesc* dm = (const MatDesc*)dt(D, D.t_desc);
  L.begin(PH_SELECT);
  launch_sum_rank_scores(s, (const float*)at(ws, D.off_scores_all), (float*)at(ws, D.off_scores), D.total_d, D.world);
  L.end();
  L.begin(PH_SELECT);
  k_topk_select<<<D.n, kSelectThreads, 4 * D.max_d, s>>>(dm, nullptr, (int32_t*)at(ws, D.off_bad),
                                                         (int32_t*)at(ws, D.off_status),
                                                         c->select == DION2_SELECT_RANDOM, c->seed, c->step);
  L.end();
}

void phase_gather(DistPlan& D, void* ws, const dion2_config* c, Launcher& L, cudaStream_t s) {
  const int sms = g_sm_count > 0 ? g_sm_count : 148;
  const MatDesc* dm = (const MatDesc*)dt(D, D.t_desc);
  const int32_t* bad = (const int32_t*)at(ws, D.off_bad);
  if (D.total_gather_tiles) {
    L.begin(PH_GATHER);
    launch_gather_decay(true, std::min(D.total_gather_tiles, sms * 8), s, dm, (const int32_t*)dt(D, D.t_gprefix), D.n,
                        D.total_gather_tiles, bad, 1, c->mu);
    L.end();
  }
  if (D.fl_gn[0]) {
    L.begin(PH_GATHER_ROWS);
    const int blocks = (int)std::min<int64_t>(ceil_div(D.fl_gunits[0], 8), (int64_t)sms * 8);
    launch_gather_rows(blocks, s, dm, (const int32_t*)dt(D, D.t_flgm[0]), (const int32_t*)dt(D, D.t_flg[0]),
                       D.fl_gn[0], D.fl_gunits[0], bad, c->mu);
    L.end();
  }
  if (D.fl_gn[1]) {
    L.begin(PH_GATHER_COLS);
    const int blocks = std::min(D.fl_gunits[1], sms * 6);  // as the single-GPU path
    launch_gather_cols_t(blocks, D.fl_maxk, D.max_cols_col, s, dm, (const int32_t*)dt(D, D.t_flgm[1]),
                         (const int32_t*)dt(D, D.t_flg[1]), D.fl_gn[1], D.fl_gunits[1], bad, c->mu);
    L.end();
  }
  L.begin(PH_NORM);
  launch_piece_sumsq(s, dm, D.n, (float*)at(ws, D.off_sumsq_local));
  L.end();
}

void phase_owner_ns(DistPlan& D, int chunk, void* ws, const dion2_config* c, Launcher& L, cudaStream_t s) {
  auto& ch = D.oc[chunk];
  if (ch.owned.empty()) return;
  Plan& P = *ch.plan;
  const MatDesc* om = (const MatDesc*)tab(P, P.off_desc);
  L.begin(PH_NORM);
  // all owned matrices in place: one block per matrix computes the norm scale only
  launch_assemble(s, om, (int)ch.owned.size(), ch.all_inplace_in ? 1 : ch.max_p_pad, ch.ptab,
                  D.recv_base, (const float*)at(ws, D.off_sumsq_all),
                  (const float*)at(ws, D.off_nsscale), D.n, c->ns_eps);
  L.end();
  run_ns(P, c, L, s, false);
  if (!ch.all_inplace) {
    L.begin(PH_SCATTER);
    launch_disassemble(s, om, (int)ch.owned.size(), ch.max_k, ch.ptab, D.osend_base);
    L.end();
  }
}

void phase_scatter(DistPlan& D, void* ws, const dion2_config* c, Launcher& L, cudaStream_t s) {
  const int sms = g_sm_count > 0 ? g_sm_count : 148;
  const float* lr_dev = (c->reserved0 & DION2_FLAG_LR_DEVICE) ? (const float*)at(ws, D.off_status + 8) : nullptr;
  const MatDesc* dm = (const MatDesc*)dt(D, D.t_desc);
  const int32_t* bad = (const int32_t*)at(ws, D.off_bad);
  if (D.total_gather_tiles) {
    L.begin(PH_SCATTER);
    launch_scatter_update(true, c->w_dtype == DION2_DT_BF16, std::min(D.total_gather_tiles, sms * 8), s, dm, (const int32_t*)dt(D, D.t_gprefix),
                          D.n, D.total_gather_tiles, bad, c->lr, lr_dev);
    L.end();
  }
  if (D.fl_sn[0]) {
    L.begin(PH_SCATTER_ROWS);
    const int blocks = (int)std::min<int64_t>(ceil_div(D.fl_sunits[0], 8), (int64_t)sms * 8);
    launch_scatter_rows(c->w_dtype == DION2_DT_BF16, blocks, s, dm, (const int32_t*)dt(D, D.t_flsm[0]), (const int32_t*)dt(D, D.t_fls[0]),
                        D.fl_sn[0], D.fl_sunits[0], bad, c->lr, lr_dev);
    L.end();
  }
  if (D.fl_sn[1]) {
    L.begin(PH_SCATTER_COLS);
    const int blocks = std::min(D.fl_sunits[1], sms * 6);  // as the single-GPU path
    launch_scatter_cols_t(c->w_dtype == DION2_DT_BF16, blocks, D.fl_maxk, D.max_cols_col, s, dm, (const int32_t*)dt(D, D.t_flsm[1]),
                          (const int32_t*)dt(D, D.t_fls[1]), D.fl_sn[1], D.fl_sunits[1], bad, c->lr, lr_dev);
    L.end();
  }
}

// ------------------------------------------------------------------ exchanges
struct Transport {
  virtual ~Transport() = default;
  virtual int allgather_scores(cudaStream_t s) = 0;
  virtual int allgather_sumsq(cudaStream_t s) = 0;
  // owner chunk `chunk` of every owner: pieces to the owners (C2) / results back (C3)
  virtual int to_owners(int chunk, cudaStream_t s) = 0;
  virtual int from_owners(int chunk, cudaStream_t s) = 0;
  virtual int allreduce_tiny(cudaStream_t s) = 0;  // sum of the short-X partial Gram matrices
  uint64_t bytes = 0;
};

struct NcclTransport : Transport {
  DistPlan& D;
  void* ws;
  ncclComm_t comm;
  NcclTransport(DistPlan& d, void* w, void* cm) : D(d), ws(w), comm(cm) {}
  int allgather_scores(cudaStream_t s) override {
    bytes += (uint64_t)D.total_d * 4 * (D.world - 1);
    return nccl_api().allgather(at(ws, D.off_scores), at(ws, D.off_scores_all), (size_t)D.total_d, kNcclFloat32, comm,
                                s)
               ? DION2_ENCCL
               : DION2_OK;
  }
  int allgather_sumsq(cudaStream_t s) override {
    bytes += (uint64_t)D.n * 4 * (D.world - 1);
    return nccl_api().allgather(at(ws, D.off_sumsq_local), at(ws, D.off_sumsq_all), (size_t)D.n, kNcclFloat32, comm, s)
               ? DION2_ENCCL
               : DION2_OK;
  }
  int exchange(bool forward, int ch, cudaStream_t s) {
    auto& api = nccl_api();
    int rc = 0;
    rc |= api.group_start();
    for (int peer = 0; peer < D.world; ++peer) {
      // forward: my pieces for owner `peer`'s chunk ch -> peer's recv section `rank`, and peer's
      //          pieces for my chunk ch -> my recv section `peer`; backward mirrors it
      const int64_t mo = D.cdispl[peer][ch], mn = D.cdispl[peer][ch + 1] - mo;            // in my section for peer
      const int64_t oo = D.cdispl[D.rank][ch], on = D.cdispl[D.rank][ch + 1] - oo;          // in my owner sections
      uint8_t* mine = (uint8_t*)at(ws, (forward ? D.off_send : D.off_orecv) + D.sdispl[peer] + mo);
      uint8_t* owner_side = (uint8_t*)at(ws, (forward ? D.off_recv : D.off_osend) + (size_t)peer * D.R + oo);
      if (forward) {
        if (mn) rc |= api.send(mine, (size_t)mn, kNcclChar, peer, comm, s);
        if (on) rc |= api.recv(owner_side, (size_t)on, kNcclChar, peer, comm, s);
      } else {
        if (on) rc |= api.send(owner_side, (size_t)on, kNcclChar, peer, comm, s);
        if (mn) rc |= api.recv(mine, (size_t)mn, kNcclChar, peer, comm, s);
      }
      if (peer != D.rank) bytes += forward ? mn : on;
    }
    rc |= api.group_end();
    return rc ? DION2_ENCCL : DION2_OK;
  }
  // direct mode: K3 already pushed the pieces (K7 will pull O): one LSA barrier each way
  int direct_sync(bool forward, cudaStream_t s) {
    for (int peer = 0; peer < D.world; ++peer)
      if (peer != D.rank) bytes += forward ? D.scount[peer] : D.R;
    return symm_barrier(D.symm, s);
  }
  int allreduce_tiny(cudaStream_t s) override {
    const size_t cnt = (size_t)kTinyP * kTinyP * D.tiny_list.size();
    bytes += (uint64_t)(2.0 * (D.world - 1) / D.world * 8.0 * (double)cnt);
    double* a = (double*)at(ws, D.off_tiny_a);
    return nccl_api().allreduce(a, a, cnt, /*ncclFloat64*/ 8, /*ncclSum*/ 0, comm, s) ? DION2_ENCCL : DION2_OK;
  }
  int to_owners(int ch, cudaStream_t s) override { return D.direct ? direct_sync(true, s) : exchange(true, ch, s); }
  int from_owners(int ch, cudaStream_t s) override { return D.direct ? direct_sync(false, s) : exchange(false, ch, s); }
};

// all ranks in one process: every exchange is a set of device-to-device copies
struct LoopbackTransport : Transport {
  std::vector<DistPlan*> D;
  std::vector<void*> ws;
  LoopbackTransport(std::vector<DistPlan*> d, std::vector<void*> w) : D(d), ws(w) {}
  int cp(void* dst, const void* src, size_t n, cudaStream_t s) {
    if (!n) return DION2_OK;
    return cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, s) == cudaSuccess ? DION2_OK : DION2_ECUDA;
  }
  int allgather_scores(cudaStream_t s) override {
    const int P = (int)D.size();
    int rc = 0;
    for (int r = 0; r < P; ++r)
      for (int r2 = 0; r2 < P; ++r2)
        rc |= cp(at(ws[r], D[r]->off_scores_all + (size_t)r2 * D[r]->total_d * 4), at(ws[r2], D[r2]->off_scores),
                 (size_t)D[r]->total_d * 4, s);
    bytes += (uint64_t)D[0]->total_d * 4 * (P - 1);
    return rc ? DION2_ECUDA : DION2_OK;
  }
  int allgather_sumsq(cudaStream_t s) override {
    const int P = (int)D.size();
    int rc = 0;
    for (int r = 0; r < P; ++r)
      for (int r2 = 0; r2 < P; ++r2)
        rc |= cp(at(ws[r], D[r]->off_sumsq_all + (size_t)r2 * D[r]->n * 4), at(ws[r2], D[r2]->off_sumsq_local),
                 (size_t)D[r]->n * 4, s);
    bytes += (uint64_t)D[0]->n * 4 * (P - 1);
    return rc ? DION2_ECUDA : DION2_OK;
  }
  int to_owners(int ch, cudaStream_t s) override {
    const int P = (int)D.size();
    int rc = 0;
    for (int r = 0; r < P; ++r)
      for (int o = 0; o < P; ++o) {
        const int64_t off = D[o]->cdispl[o][ch], len = D[o]->cdispl[o][ch + 1] - off;
        if (D[0]->direct) {  // pushed by K3 (stream order stands in for the barrier)
          if (o != 0 && r == 0) bytes += (uint64_t)len;
          continue;
        }
        rc |= cp(at(ws[o], D[o]->off_recv + (size_t)r * D[o]->R + off), at(ws[r], D[r]->off_send + D[r]->sdispl[o] + off),
                 (size_t)len, s);
        if (o != 0 && r == 0) bytes += (uint64_t)len;
      }
    return rc ? DION2_ECUDA : DION2_OK;
  }
  int allreduce_tiny(cudaStream_t s) override {
    const int P = (int)D.size();
    const int64_t cnt = (int64_t)kTinyP * kTinyP * (int64_t)D[0]->tiny_list.size();
    double* a0 = (double*)at(ws[0], D[0]->off_tiny_a);
    for (int r = 1; r < P; ++r) launch_add_f64(s, a0, (const double*)at(ws[r], D[r]->off_tiny_a), cnt);
    int rc = 0;
    for (int r = 1; r < P; ++r) rc |= cp(at(ws[r], D[r]->off_tiny_a), a0, (size_t)cnt * 8, s);
    bytes += (uint64_t)(2.0 * (P - 1) / P * 8.0 * (double)cnt);
    return rc ? DION2_ECUDA : DION2_OK;
  }
  int from_owners(int ch, cudaStream_t s) override {
    const int P = (int)D.size();
    int rc = 0;
    for (int o = 0; o < P; ++o)
      for (int r = 0; r < P; ++r) {
        const int64_t off = D[o]->cdispl[o][ch], len = D[o]->cdispl[o][ch + 1] - off;
        if (D[0]->direct) {  // pulled by K7
          if (o == 0 && r != 0) bytes += (uint64_t)len;
          continue;
        }
        rc |= cp(at(ws[r], D[r]->off_orecv + D[r]->sdispl[o] + off), at(ws[o], D[o]->off_osend + (size_t)r * D[o]->R + off),
                 (size_t)len, s);
        if (o == 0 && r != 0) bytes += (uint64_t)len;
      }
    return rc ? DION2_ECUDA : DION2_OK;
  }
};

// library-owned side stream for the chunked exchanges (non-blocking, default priority)
cudaStream_t comm_stream() {
  static cudaStream_t st = nullptr;
  if (!st) cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  return st;
}

// One distributed step.  With one owner chunk everything runs on `s` in order
// K1 -> C1 -> K2 -> K3 -> C2 -> NS -> C3 -> K7.  With C chunks the exchanges run on a side
// stream: C2(0..C-1) back to back, the owner NS of chunk c on `s` once C2(c) has landed, and
// C3(c) once NS(c) is done, so C2(c + 1) and C3(c - 1) overlap NS(c); `s` waits for the last
// C3 before the sparse update.  All sizes are host-known (no host synchronisation).
int run_dist(std::vector<DistPlan*>& plans, std::vector<void*>& wss, const std::vector<const dion2_shard*>& shards,
             const dion2_config* c, Transport& T, cudaStream_t s, uint64_t* bytes_out) {
  Launcher L{s};
  int rc = 0;
  const size_t R = plans.size();
  const int C = plans[0]->nchunks;
  for (size_t i = 0; i < R; ++i)
    if ((rc = refresh(*plans[i], shards[i], c, s))) return rc;
  for (size_t i = 0; i < R; ++i) phase_local_k1(*plans[i], wss[i], L, s);
  if ((rc = T.allgather_scores(s))) return rc;                      // C1
  for (size_t i = 0; i < R; ++i) phase_select(*plans[i], wss[i], c, L, s);
  if (!plans[0]->tiny_list.empty()) {
    // short X (R25): partial Gram matrices of the local blocks, their sum, the exact NS applied
    // locally -- before K3 decays M[K]
    NsSmallCoeffs cs{};
    for (int t = 0; t < c->ns_steps && t < 16; ++t)
      for (int e = 0; e < 3; ++e) cs.c[t][e] = c->ns_coeffs[t][e];
    cs.T = c->ns_steps;
    cs.eps = c->ns_eps;
    for (size_t i = 0; i < R; ++i) {
      DistPlan& D = *plans[i];
      const MatDesc* dm = (const MatDesc*)dt(D, D.t_desc);
      const int32_t* tl = (const int32_t*)dt(D, D.t_tiny);
      double* a = (double*)at(wss[i], D.off_tiny_a);
      const int n64 = D.n_tiny64, n128 = (int)D.tiny_list.size() - D.n_tiny64;
      L.begin(PH_NSMUL);
      launch_ns_small_partial(s, dm, tl, n64, a, false);
      launch_ns_small_partial(s, dm, tl + n64, n128, a + (int64_t)n64 * kTinyP * kTinyP, true);
      L.end();
    }
    if ((rc = T.allreduce_tiny(s))) return rc;
    for (size_t i = 0; i < R; ++i) {
      DistPlan& D = *plans[i];
      const MatDesc* dm = (const MatDesc*)dt(D, D.t_desc);
      const int32_t* tl = (const int32_t*)dt(D, D.t_tiny);
      const int32_t* bad = (const int32_t*)at(wss[i], D.off_bad);
      const double* a = (const double*)at(wss[i], D.off_tiny_a);
      const int n64 = D.n_tiny64, n128 = (int)D.tiny_list.size() - D.n_tiny64;
      L.begin(PH_NSMUL);
      launch_ns_small_finish(s, dm, tl, n64, bad, a, cs, false);
      launch_ns_small_finish(s, dm, tl + n64, n128, bad, a + (int64_t)n64 * kTinyP * kTinyP, cs, true);
      L.end();
    }
  }
  for (size_t i = 0; i < R; ++i) phase_gather(*plans[i], wss[i], c, L, s);
  if ((rc = T.allgather_sumsq(s))) return rc;
  if (C == 1) {
    if ((rc = T.to_owners(0, s))) return rc;                        // C2
    for (size_t i = 0; i < R; ++i) phase_owner_ns(*plans[i], 0, wss[i], c, L, s);
    if ((rc = T.from_owners(0, s))) return rc;                      // C3
  } else {
    static std::vector<cudaEvent_t> ev;  // [0] fork, [1 + c] C2(c) landed, [1 + C + c] NS(c) done, last: join
    while ((int)ev.size() < 2 * C + 2) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      ev.push_back(e);
    }
    cudaStream_t sc = comm_stream();
    cudaEventRecord(ev[0], s);
    cudaStreamWaitEvent(sc, ev[0], 0);
    for (int ch = 0; ch < C; ++ch) {
      if ((rc = T.to_owners(ch, sc))) return rc;                    // C2(ch)
      cudaEventRecord(ev[1 + ch], sc);
    }
    for (int ch = 0; ch < C; ++ch) {
      cudaStreamWaitEvent(s, ev[1 + ch], 0);
      for (size_t i = 0; i < R; ++i) phase_owner_ns(*plans[i], ch, wss[i], c, L, s);
      cudaEventRecord(ev[1 + C + ch], s);
      cudaStreamWaitEvent(sc, ev[1 + C + ch], 0);
      if ((rc = T.from_owners(ch, sc))) return rc;                  // C3(ch)
    }
    cudaEventRecord(ev[2 * C + 1], sc);
    cudaStreamWaitEvent(s, ev[2 * C + 1], 0);
  }
  for (size_t i = 0; i < R; ++i) phase_scatter(*plans[i], wss[i], c, L, s);
  g_last_launches = L.count;
  if (bytes_out) *bytes_out = T.bytes;
  return L.err;
}

// ------------------------------------------------------------------ compressed DP-sync
// Replicas (one per rank) hold full W, M and their own local G.  With the random rule the
// selection needs no global state, so only the selected fp32 rows M[K] are all-reduced
// (averaged); every replica then runs the rest of the step on identical rows.
struct DpPlan {
  DpPlan() = default;
  DpPlan(const DpPlan&) = delete;
  DpPlan& operator=(const DpPlan&) = delete;
  ~DpPlan() {
    if (dtab) cudaFree(dtab);
  }
  Plan P;
  int world = 1;
  size_t off_buf = 0, off_gather = 0, total = 0;
  int64_t buf_floats = 0;   // selected rows of every matrix, then the 2 n tail floats (k_dp_tail)
  int64_t data_floats = 0;
  int total_rows = 0;
  // direct exchange (DION2_FLAG_DIST_DIRECT): phase 1 packs into pack_buf, the reduce-scatter /
  // all-gather kernel writes the sum into every replica's red_buf (NCCL symmetric windows, or
  // the loopback replicas' own buffers); otherwise both are the workspace buffer (in-place
  // ncclAllReduce)
  int direct = 0;
  float* pack_buf = nullptr;
  float* red_buf = nullptr;
  std::vector<uint8_t*> peer_in, peer_out;
  SymmState* symm = nullptr;  // kept for the process lifetime (collective teardown)
  void* dtab = nullptr;  // [n] int32 row prefix, then [n] int64 buffer offsets
  size_t t_prefix = 0, t_off = 0;
  bool uploaded = false;
  std::vector<uint8_t> htab;
};
std::map<std::string, std::unique_ptr<DpPlan>> g_dp_plans;

int dp_layout(DpPlan& D, const dion2_matrix* mats, int n, const dion2_config* c, int world) {
  if (c->select != DION2_SELECT_RANDOM) return DION2_EUNSUPPORTED;  // l1 scores need the full momentum
  if (world < 1) return DION2_EINVAL_SHAPE;
  D.world = world;
  int rc = build_layout(D.P, mats, n, c);
  if (rc) return rc;
  D.buf_floats = 0;
  D.total_rows = 0;
  for (auto& q : D.P.mp) {
    D.buf_floats += (int64_t)q.sr * q.sc;
    D.total_rows += q.mt ? q.sc : q.sr;  // pack units: rows of S, or rows of S^T (transposed M)
  }
  D.data_floats = D.buf_floats;
  D.buf_floats += 2 * (int64_t)n;
  D.off_buf = align_up(D.P.total, 4096);
  D.off_gather = align_up(D.off_buf + 4 * (size_t)D.buf_floats, 4096);
  D.total = D.off_gather + 4 * (size_t)D.buf_floats * world + 4096;
  return DION2_OK;
}

int dp_get_plan(DpPlan** out, const dion2_matrix* mats, int n, const dion2_config* c, int world, void* workspace,
                size_t ws_bytes, void** ws_out, void* comm = nullptr, cudaStream_t s = nullptr) {
  void* ws = reinterpret_cast<void*>(align_up(reinterpret_cast<uintptr_t>(workspace), 4096));
  const size_t slack = (uintptr_t)ws - (uintptr_t)workspace;
  std::string key;
  auto put = [&](const void* p, size_t s) { key.append(reinterpret_cast<const char*>(p), s); };
  put(&n, 4);
  put(&world, 4);
  put(&ws, sizeof ws);
  for (int i = 0; i < n; ++i) {
    put(&mats[i].rows, 8);
    put(&mats[i].cols, 8);
    put(&mats[i].ld, 8);
    put(&mats[i].m_transposed, 4);
    put(&mats[i].storage_transposed, 4);
  }
  put(&c->alpha, 4);
  put(&c->ns_steps, 4);
  put(c->ns_coeffs, sizeof(float) * 3 * c->ns_steps);
  put(&c->axis, 4);
  put(&c->precision, 4);
  put(&c->grad_dtype, 4);
  put(&c->w_dtype, 4);
  put(&c->decay_mode, 4);
  put(&c->scale_mode, 4);
  put(&c->ns_form, 4);
  const int direct = (c->reserved0 & DION2_FLAG_DIST_DIRECT) && world <= kMaxPieceRanks ? 1 : 0;
  put(&direct, 4);
  if (direct) put(&comm, sizeof comm);
  key += env_key();
  auto it = g_dp_plans.find(key);
  if (it == g_dp_plans.end()) {
    auto D = std::make_unique<DpPlan>();
    int rc = dp_layout(*D, mats, n, c, world);
    if (rc) return rc;
    if (D->total - 4096 + slack > ws_bytes) return DION2_EWORKSPACE;
    if ((rc = build_device_plan(D->P, mats, c, ws))) return rc;
    D->t_prefix = 0;
    D->t_off = align_up(4 * (size_t)n, 256);
    D->htab.assign(D->t_off + 8 * (size_t)n, 0);
    int32_t* pre = reinterpret_cast<int32_t*>(D->htab.data());
    int64_t* off = reinterpret_cast<int64_t*>(D->htab.data() + D->t_off);
    int rows = 0;
    int64_t fo = 0;
    for (int i = 0; i < n; ++i) {
      pre[i] = rows;
      off[i] = fo;
      rows += D->P.mp[i].mt ? D->P.mp[i].sc : D->P.mp[i].sr;
      fo += (int64_t)D->P.mp[i].sr * D->P.mp[i].sc;
    }
    if (cudaMalloc(&D->dtab, D->htab.size()) != cudaSuccess) return DION2_ECUDA;
    D->pack_buf = D->red_buf = (float*)at(ws, D->off_buf);
    D->direct = direct;
    if (direct && comm) {  // NCCL: pack into / reduce into symmetric windows
      uint8_t *in = nullptr, *outb = nullptr;
      rc = symm_create(comm, world, 4 * (size_t)D->buf_floats, s, &D->symm, &in, &outb, D->peer_in, D->peer_out);
      if (rc == DION2_EUNSUPPORTED) {  // decided identically on every rank before any collective call
        D->direct = 0;
      } else if (rc) {
        return rc;
      } else {
        D->pack_buf = reinterpret_cast<float*>(in);
        D->red_buf = reinterpret_cast<float*>(outb);
      }
    }
    it = g_dp_plans.emplace(key, std::move(D)).first;
  }
  DpPlan& D = *it->second;
  if (D.total - 4096 + slack > ws_bytes) return DION2_EWORKSPACE;
  *out = &D;
  *ws_out = ws;
  return DION2_OK;
}

void dp_pack(DpPlan& D, void* ws, bool unpack, float scale, cudaStream_t s, Launcher& L) {
  L.begin(unpack ? PH_GATHER : PH_SELECT);
  launch_dp_pack(unpack, s, (const MatDesc*)tab(D.P, D.P.off_desc),
                 (const int32_t*)((uint8_t*)D.dtab + D.t_prefix), (const int64_t*)((uint8_t*)D.dtab + D.t_off),
                 D.P.n, D.total_rows, unpack ? D.red_buf : D.pack_buf, scale, (const int32_t*)at(ws, D.P.off_bad));
  L.end();
}

// phases 1: refresh + K1 + select + pack; 2: unpack + gather + NS + scatter
int dp_phase1(DpPlan& D, const dion2_matrix* mats, const dion2_config* c, void* ws, cudaStream_t s, Launcher& L) {
  int rc = refresh_tables(D.P, mats, c, s);
  if (rc) return rc;
  if (!D.uploaded) {
    if (cudaMemcpyAsync(D.dtab, D.htab.data(), D.htab.size(), cudaMemcpyHostToDevice, s) != cudaSuccess)
      return DION2_ECUDA;
    D.uploaded = true;
  }
  int32_t* status = (int32_t*)at(ws, D.P.off_status);
  if ((rc = reset_status(status, s))) return rc;
  stage_k1_select(D.P, c, ws, status, L, s, true);
  dp_pack(D, ws, false, 1.f, s, L);
  L.begin(PH_SELECT);
  launch_dp_tail(s, (const MatDesc*)tab(D.P, D.P.off_desc), D.P.n, D.pack_buf + D.data_floats,
                 (int32_t*)at(ws, D.P.off_bad), status, false);
  L.end();
  return DION2_OK;
}

void dp_phase2(DpPlan& D, const dion2_matrix* mats, const dion2_config* c, void* ws, cudaStream_t s, Launcher& L) {
  L.begin(PH_SELECT);  // global non-finite flags and the common fp16 prescale
  launch_dp_tail(s, (const MatDesc*)tab(D.P, D.P.off_desc), D.P.n, D.red_buf + D.data_floats,
                 (int32_t*)at(ws, D.P.off_bad), (int32_t*)at(ws, D.P.off_status), true);
  L.end();
  dp_pack(D, ws, true, 1.f / (float)D.world, s, L);  // M[K] <- mean over replicas (skips bad matrices)
  stage_gather(D.P, c, ws, L, s, true);
  run_ns(D.P, c, L, s, true);
  stage_post(D.P, mats, c, ws, L, s, true);
}

}  // namespace

int release_dist_plans(uintptr_t lo, uintptr_t hi) {
  int dropped = 0;
  for (auto it = g_dist_plans.begin(); it != g_dist_plans.end();) {
    const uintptr_t w = reinterpret_cast<uintptr_t>(it->second->ws);
    if (w >= lo && w < hi) { it = g_dist_plans.erase(it); ++dropped; } else { ++it; }
  }
  for (auto it = g_last_mode.begin(); it != g_last_mode.end();) {
    const uintptr_t w = reinterpret_cast<uintptr_t>(it->first);
    if (w >= lo && w < hi) it = g_last_mode.erase(it); else ++it;
  }
  for (auto it = g_dp_plans.begin(); it != g_dp_plans.end();) {
    const uintptr_t w = reinterpret_cast<uintptr_t>(it->second->P.ws);
    if (w >= lo && w < hi) { it = g_dp_plans.erase(it); ++dropped; } else { ++it; }
  }
  return dropped;
}

}  // namespace dion2rt

using namespace dion2rt;

extern "C" {

int dion2_dist_info(const dion2_shard* shards, int32_t n, const dion2_config* cfg, int32_t world, int32_t rank,
                    int32_t* axis_out, int32_t* owner_out, int64_t* shard_rows_out, int64_t* shard_cols_out,
                    int64_t* send_bytes_out, int64_t* recv_bytes_out, size_t* ws_bytes_out) {
  int rc = validate_config(cfg);
  if (rc) return rc;
  DistPlan D;
  rc = resolve(D, shards, n, cfg, world, rank);
  if (rc) return rc;
  for (int j = 0; j < n; ++j) {
    if (axis_out) axis_out[j] = D.dm[j].axis;
    if (owner_out) owner_out[j] = D.dm[j].owner;
    if (shard_rows_out) shard_rows_out[j] = D.dm[j].srows;
    if (shard_cols_out) shard_cols_out[j] = D.dm[j].scols;
  }
  for (int r = 0; r < world; ++r) {
    if (send_bytes_out) send_bytes_out[r] = D.scount[r];
    if (recv_bytes_out) recv_bytes_out[r] = D.R;
  }
  if (ws_bytes_out) *ws_bytes_out = D.total;
  return DION2_OK;
}

int dion2_step_batched_dist(const dion2_shard* shards, int32_t n, const dion2_config* cfg, void* workspace,
                            size_t ws_bytes, void* nccl_comm, int32_t world, int32_t rank, void* stream,
                            uint64_t* comm_bytes_out) {
  int rc = validate_config(cfg);
  if (rc) return rc;
  if (!workspace) return DION2_EWORKSPACE;
  for (int j = 0; j < n; ++j)
    if (!shards[j].W || !shards[j].M || !shards[j].G) return DION2_EINVAL_SHAPE;
  if (!nccl_comm) return DION2_ENCCL;
  if (!nccl_api().ok) return DION2_ENCCL;
  std::lock_guard<std::mutex> lock(g_mu);
  ensure_device_attrs();
  DistPlan* D = nullptr;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((rc = get_plan(&D, shards, n, cfg, world, rank, workspace, ws_bytes, nccl_comm, s))) return rc;
  void* ws = reinterpret_cast<void*>(align_up(reinterpret_cast<uintptr_t>(workspace), 4096));
  g_last_mode[ws] = D->direct;
  NcclTransport T(*D, ws, nccl_comm);
  std::vector<DistPlan*> plans{D};
  std::vector<void*> wss{ws};
  std::vector<const dion2_shard*> sh{shards};
  return run_dist(plans, wss, sh, cfg, T, s, comm_bytes_out);
}

int dion2_dist_exchange_mode(const void* workspace) {
  std::lock_guard<std::mutex> lock(g_mu);
  const void* ws = reinterpret_cast<const void*>(align_up(reinterpret_cast<uintptr_t>(workspace), 4096));
  auto it = g_last_mode.find(ws);
  return it == g_last_mode.end() ? -1 : it->second;
}

int dion2_step_batched_loopback(const dion2_shard* shards, int32_t n, const dion2_config* cfg,
                                void* const* workspaces, size_t ws_bytes, int32_t world, void* stream,
                                uint64_t* comm_bytes_out) {
  int rc = validate_config(cfg);
  if (rc) return rc;
  if (!workspaces || world < 1) return DION2_EWORKSPACE;
  for (int j = 0; j < n * world; ++j)
    if (!shards[j].W || !shards[j].M || !shards[j].G) return DION2_EINVAL_SHAPE;
  std::lock_guard<std::mutex> lock(g_mu);
  ensure_device_attrs();
  std::vector<DistPlan*> plans(world);
  std::vector<void*> wss(world);
  std::vector<const dion2_shard*> sh(world);
  for (int r = 0; r < world; ++r) {
    if (!workspaces[r]) return DION2_EWORKSPACE;
    if ((rc = get_plan(&plans[r], shards + (size_t)r * n, n, cfg, world, r, workspaces[r], ws_bytes))) return rc;
    wss[r] = reinterpret_cast<void*>(align_up(reinterpret_cast<uintptr_t>(workspaces[r]), 4096));
    sh[r] = shards + (size_t)r * n;
  }
  if (plans[0]->direct) {  // every loopback rank's buffers are addressable: push / pull directly
    for (int r = 0; r < world; ++r) {
      plans[r]->peer_recv.resize(world);
      plans[r]->peer_osend.resize(world);
      for (int o = 0; o < world; ++o) {
        plans[r]->peer_recv[o] = plans[o]->recv_base;
        plans[r]->peer_osend[o] = plans[o]->osend_base;
      }
      apply_direct(*plans[r]);
    }
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  LoopbackTransport T(plans, wss);
  return run_dist(plans, wss, sh, cfg, T, s, comm_bytes_out);
}

}  // extern "C"

// ------------------------------------------------------------------ compressed DP-sync ABI
extern "C" {

int dion2_dpsync_workspace_size(const dion2_matrix* user_mats, int32_t n, const dion2_config* cfg, int32_t world,
                                size_t* bytes_out) {
  int rc = validate_config(cfg);
  if (rc) return rc;
  if (!bytes_out) return DION2_EINVAL_CONFIG;
  if (n < 1 || !user_mats) return DION2_EINVAL_SHAPE;
  const std::vector<dion2_matrix> sv = storage_view(user_mats, n);
  const dion2_matrix* mats = sv.data();
  for (int i = 0; i < n; ++i)
    if ((rc = validate_shape(mats[i], false))) return rc;
  DpPlan D;
  if ((rc = dp_layout(D, mats, n, cfg, world))) return rc;
  *bytes_out = D.total;
  return DION2_OK;
}

int dion2_step_batched_dpsync(const dion2_matrix* user_mats, int32_t n, const dion2_config* cfg, void* workspace,
                              size_t ws_bytes, void* nccl_comm, int32_t world, int32_t rank, void* stream,
                              uint64_t* comm_bytes_out) {
  int rc = validate_config(cfg);
  if (rc) return rc;
  if (n < 1 || !user_mats) return DION2_EINVAL_SHAPE;
  const std::vector<dion2_matrix> sv = storage_view(user_mats, n);
  const dion2_matrix* mats = sv.data();
  for (int i = 0; i < n; ++i)
    if ((rc = validate_shape(mats[i], true))) return rc;
  if (!workspace) return DION2_EWORKSPACE;
  if (!nccl_comm || !nccl_api().ok) return DION2_ENCCL;
  if (rank < 0 || rank >= world) return DION2_EINVAL_SHAPE;
  std::lock_guard<std::mutex> lock(g_mu);
  ensure_device_attrs();
  DpPlan* D = nullptr;
  void* ws = nullptr;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((rc = dp_get_plan(&D, mats, n, cfg, world, workspace, ws_bytes, &ws, nccl_comm, s))) return rc;
  g_last_mode[ws] = D->direct;
  Launcher L{s};
  if ((rc = dp_phase1(*D, mats, cfg, ws, s, L))) return rc;
  if (D->direct) {
    // every replica's pack is in its window -> reduce this rank's slice into every window -> all
    // slices landed (the second barrier also keeps the next step's pack off the windows until
    // every replica is done reading)
    if ((rc = symm_barrier(D->symm, s))) return rc;
    DpPeerBufs B{};
    for (int r = 0; r < world; ++r) {
      B.in[r] = reinterpret_cast<const float*>(D->peer_in[r]);
      B.out[r] = reinterpret_cast<float*>(D->peer_out[r]);
    }
    L.begin(PH_SELECT);
    launch_dp_reduce_direct(s, B, world, rank, D->buf_floats, g_sm_count > 0 ? g_sm_count : 148);
    L.end();
    if ((rc = symm_barrier(D->symm, s))) return rc;
  } else {
    float* buf = (float*)at(ws, D->off_buf);
    if (nccl_api().allreduce(buf, buf, (size_t)D->buf_floats, kNcclFloat32, /*ncclSum*/ 0, nccl_comm, s))
      return DION2_ENCCL;
  }
  dp_phase2(*D, mats, cfg, ws, s, L);
  g_last_launches = L.count;
  if (comm_bytes_out) *comm_bytes_out = (uint64_t)(2.0 * (world - 1) / world * 4.0 * (double)D->buf_floats);
  return L.err;
}

int dion2_step_batched_dpsync_loopback(const dion2_matrix* user_mats, int32_t n, const dion2_config* cfg,
                                       void* const* workspaces, size_t ws_bytes, int32_t world, void* stream,
                                       uint64_t* comm_bytes_out) {
  int rc = validate_config(cfg);
  if (rc) return rc;
  if (n < 1 || !user_mats || world < 1 || !workspaces) return DION2_EINVAL_SHAPE;
  const std::vector<dion2_matrix> sv = storage_view(user_mats, n * world);
  const dion2_matrix* mats = sv.data();
  for (int i = 0; i < n * world; ++i)
    if ((rc = validate_shape(mats[i], true))) return rc;
  std::lock_guard<std::mutex> lock(g_mu);
  ensure_device_attrs();
  std::vector<DpPlan*> D(world);
  std::vector<void*> ws(world);
  for (int r = 0; r < world; ++r)
    if ((rc = dp_get_plan(&D[r], mats + (size_t)r * n, n, cfg, world, workspaces[r], ws_bytes, &ws[r]))) return rc;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Launcher L{s};
  for (int r = 0; r < world; ++r)
    if ((rc = dp_phase1(*D[r], mats + (size_t)r * n, cfg, ws[r], s, L))) return rc;
  const size_t bytes = 4 * (size_t)D[0]->buf_floats;
  if (D[0]->direct) {
    // direct exchange: each replica's slice summed over every replica's buffer (rank order) and
    // written back into every buffer (in place; the slices are disjoint)
    DpPeerBufs B{};
    for (int r = 0; r < world; ++r) B.in[r] = B.out[r] = D[r]->pack_buf;
    for (int r = 0; r < world; ++r) {
      L.begin(PH_SELECT);
      launch_dp_reduce_direct(s, B, world, r, D[0]->buf_floats, g_sm_count > 0 ? g_sm_count : 148);
      L.end();
    }
  } else {
    // all-reduce (sum) emulated: gather every replica's buffer at replica 0, sum in rank order, broadcast
    for (int r = 0; r < world; ++r)
      cudaMemcpyAsync(at(ws[0], D[0]->off_gather + r * bytes), at(ws[r], D[r]->off_buf), bytes,
                      cudaMemcpyDeviceToDevice, s);
    launch_sum_rank_scores(s, (const float*)at(ws[0], D[0]->off_gather), (float*)at(ws[0], D[0]->off_buf),
                           D[0]->buf_floats, world);
    for (int r = 1; r < world; ++r)
      cudaMemcpyAsync(at(ws[r], D[r]->off_buf), at(ws[0], D[0]->off_buf), bytes, cudaMemcpyDeviceToDevice, s);
  }
  for (int r = 0; r < world; ++r) dp_phase2(*D[r], mats + (size_t)r * n, cfg, ws[r], s, L);
  g_last_launches = L.count;
  if (comm_bytes_out) *comm_bytes_out = (uint64_t)(2.0 * (world - 1) / world * (double)bytes);
  return L.err;
}

}  // extern "C"
