// runtime.h -- host-runtime internals shared by the single-GPU C ABI (dion2_api.cu)
// and the distributed step (dion2_dist.cu).  Not part of the public ABI.
#pragma once
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: phase ranges for nsys / ncu --nvtx

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dion2.h"
#include "kernels.cuh"

namespace dion2rt {
using namespace dion2;

constexpr int kNumPhases = 15;
extern const char* kPhaseNames[kNumPhases];
enum Phase {
  PH_K1 = 0, PH_SELECT, PH_GATHER, PH_NORM, PH_GRAM, PH_POLY, PH_APPLY, PH_SCATTER, PH_FULLDECAY,
  PH_GATHER_ROWS, PH_GATHER_COLS, PH_SCATTER_ROWS, PH_SCATTER_COLS, PH_NSMUL, PH_K1_MT
};

extern std::mutex g_mu;
extern std::map<std::string, std::unique_ptr<struct Plan>> g_plans;
// number of SMs of the current device (queried once; 148 if no device is visible)
int sm_count();
// drop the cached distributed / DP-sync plans whose workspace lies in [lo, hi) (dion2_dist.cu)
int release_dist_plans(uintptr_t lo, uintptr_t hi);
extern int g_sm_count;
extern bool g_attr_done;
extern int32_t g_last_launches;
extern bool g_timing;
struct TimedLaunch {
  int phase;
  cudaEvent_t a, b;
};
extern std::vector<TimedLaunch> g_timed;
extern std::vector<cudaEvent_t> g_event_pool;
cudaEvent_t take_event();

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

bool make_map(CUtensorMap* m, const void* base, int64_t cols, int64_t rows, int64_t count, int box_cols, int box_rows,
              CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B);
bool make_map_strided(CUtensorMap* m, const void* base, int64_t cols, int64_t rows, int64_t count,
                      int64_t zstride_bytes, int box_cols, int box_rows, CUtensorMapSwizzle swz);
int validate_config(const dion2_config* c);
// The kernels' view of the caller's matrices: storage_transposed ones get their storage shape
// (rows and cols swapped); build_layout recovers the logical shape for the axis, k and scale.
std::vector<dion2_matrix> storage_view(const dion2_matrix* mats, int n);
std::string env_key();
int validate_shape(const dion2_matrix& m, bool need_ptrs);

// AUTO evaluates NS in Gram space only for X with at least this many rows (reading R25)
constexpr int kGramMinP = 64;

struct MatPlan {
  int mt;  // M stored transposed (cols mode): gather = rows path on M^T, scatter = path (cols / generic)
  int axis, d, o, k, sr, sc, transposed, p, q, p_pad, q_pad, group, zi, rowblocks, ga, gb, sa_pad, sb_pad, path,
      n_sumsq, spath;  // spath: scatter path (the cols streaming scatter takes k up to kMaxColKScatter)
  int tiny = 0;        // short X under AUTO: NS by k_ns_small (fp64 Gram space), not the tensor cores
  float fan_sqrt;
  size_t off_scores, off_partials, off_sel, off_sumsq;
};

struct Group {
  int p_pad, q_pad, count;
  std::vector<int> mats;  // global matrix indices
  size_t off_X0, off_X1, off_A, off_B, off_gmats;
  int gs;                           // Newton-Schulz in Gram space (reading R23)
  int tiny = 0;                     // members take k_ns_small (no tensor-core NS launches)
  size_t off_C, off_Q0, off_Q1;     // Gram-space p x p buffers (gs only)
};

struct Launch {
  int phase;
  int bn;
  int kind;  // 0 = tc BN128, 1 = tc BN256, 2 = simt, 3 = 2-SM pair, 5 = 2-SM apply with resident A
  NsTcParams tc;
  int simt_group;
};

struct Plan {
  Plan() = default;
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;
  ~Plan() {
    if (dtab) cudaFree(dtab);
  }
  int n;
  bool bf16_ns;
  int ns_steps;
  std::vector<MatPlan> mp;
  std::vector<Group> groups;
  size_t off_status, off_bad, off_desc, off_rowmats, off_rowprefix, off_colmats, off_colprefix, off_gprefix,
      off_nsscale, off_ns_begin, off_ns_end, total;
  size_t off_cf_mats = 0, off_cf_prefix = 0;  // cols-mode matrices whose scores k_col_scores_finalize sums
  int cf_n = 0;
  int64_t cf_total = 0;
  int64_t total_rows = 0, total_col_tiles = 0;
  int generic_gather_mats = 0;   // matrices the generic K3 tile kernel gathers (not transposed-M ones)
  int generic_scatter_mats = 0;  // matrices the generic K7 tile kernel updates (spath == 0)
  int n_row_mats = 0, n_col_mats = 0, total_gather_tiles = 0, max_d = 0;
  // streaming fast paths: list 0 = rows (units: X rows p_pad / selected rows k),
  // list 1 = cols with X = S^T (units: 32-row slabs of X's columns, q_pad / 32)
  // gather and scatter memberships differ for transposed-M column matrices (rows gather
  // on M^T, column scatter on W)
  size_t off_flg_mats[2], off_fls_mats[2], off_fl_gprefix[2], off_fl_sprefix[2];
  int fl_gn[2] = {0, 0}, fl_sn[2] = {0, 0}, fl_gunits[2] = {0, 0}, fl_sunits[2] = {0, 0}, fl_maxk = 0,
      fl_smaxk = 0;  // largest k of the cols streaming gather / scatter lists
  // K1 for column matrices with transposed M
  size_t off_mtmats = 0, off_mtprefix = 0;
  int n_mt_mats = 0;
  int64_t total_mt_tiles = 0;
  int64_t fl_maxn = 0;
  // split-K of the long-K gram launches when their tiles cannot fill the GPU (bf16 pair path)
  int gram_splitk = 1;
  size_t off_splitk = 0;
  bool no_tiny = false;  // set before build_layout: short X stays on the tensor cores (owner plans of
                         // the distributed step, whose X arrives as fp16 pieces)
  size_t off_tiny_list = 0;
  int n_tiny = 0, n_tiny64 = 0;  // the list holds the p <= 64 matrices first, then 64 < p <= 128
  std::vector<uint8_t> host_tables;  // [off_desc, off_ns_begin) image (descriptors + aux)
  std::vector<Launch> ns_launches;
  void* ws = nullptr;
  uint64_t id = 0;
  std::vector<const void*> last_ptrs;  // W, M, G, sel_out, O_out, ldm per matrix as last uploaded
  void* dtab = nullptr;                // plan-owned device copy of host_tables
};

// device address of a table offset (tables are carved with workspace-style offsets
// starting at off_desc but live in the plan-owned buffer)
inline void* tab(Plan& P, size_t off) { return static_cast<uint8_t*>(P.dtab) + (off - P.off_desc); }

inline void* at(void* ws, size_t off) { return static_cast<uint8_t*>(ws) + off; }

struct Launcher {
  cudaStream_t s;
  int count = 0;
  int err = DION2_OK;
  int cur_phase = -1;
  cudaEvent_t ev_a = nullptr;
  void begin(int phase) {
    cur_phase = phase;
    nvtxRangePushA(kPhaseNames[phase]);  // one host range per launch, named by phase
    if (g_timing) {
      ev_a = take_event();
      cudaEventRecord(ev_a, s);
    }
  }
  void end() {
    ++count;
    nvtxRangePop();
    if (cudaPeekAtLastError() != cudaSuccess) {
      cudaGetLastError();
      err = DION2_ECUDA;
    }
    static const bool debug_sync = getenv("DION2_DEBUG_SYNC") != nullptr;
    if (debug_sync) {
      cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) {
        fprintf(stderr, "[dion2] launch %d (phase %s) failed: %s\n", count, kPhaseNames[cur_phase],
                cudaGetErrorString(e));
        err = DION2_ECUDA;
      }
    }
    if (g_timing) {
      cudaEvent_t b = take_event();
      cudaEventRecord(b, s);
      g_timed.push_back({cur_phase, ev_a, b});
    }
  }
};

int build_layout(Plan& P, const dion2_matrix* mats, int n, const dion2_config* c);
// restart segments [t0, t1) of the Gram-space NS form (reading R24)
std::vector<std::pair<int, int>> ns_segments(const dion2_config* c, int T);
int build_device_plan(Plan& P, const dion2_matrix* mats, const dion2_config* c, void* ws);
void ensure_device_attrs();
int run_ns(Plan& P, const dion2_config* c, Launcher& L, cudaStream_t s, bool do_norm);
int refresh_tables(Plan& P, const dion2_matrix* mats, const dion2_config* c, cudaStream_t s);
int reset_status(int32_t* status, cudaStream_t s);
void launch_k1_mt(const MatDesc* host_desc, int n_desc, int grad_dtype, int64_t total_tiles, int legacy_grid,
                  cudaStream_t s, const MatDesc* dmats, const int32_t* list, const int64_t* prefix, int n_list);
void stage_pre(Plan& P, const dion2_config* c, void* ws, int32_t* status, Launcher& L, cudaStream_t s,
               bool persistent);
void stage_k1_select(Plan& P, const dion2_config* c, void* ws, int32_t* status, Launcher& L, cudaStream_t s,
                     bool persistent);
void stage_gather(Plan& P, const dion2_config* c, void* ws, Launcher& L, cudaStream_t s, bool persistent);
void stage_post(Plan& P, const dion2_matrix* mats, const dion2_config* c, void* ws, Launcher& L, cudaStream_t s,
                bool persistent);

}  // namespace dion2rt
