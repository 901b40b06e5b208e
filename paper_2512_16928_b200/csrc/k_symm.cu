// Direct peer exchange of the owner-compute step over NCCL symmetric memory (NCCL 2.28
// device API): the fused "gather + send" / "receive + scatter" of SURVEY §8(e) step 3.
//
// The owner's receive buffer (pieces of X, C2) and outgoing buffer (pieces of X_T, C3) are
// ncclMemAlloc'd and registered as symmetric windows (ncclCommWindowRegister,
// NCCL_WIN_COLL_SYMMETRIC); every rank maps every peer's windows into its own address space
// (LSA: load/store accessible over NVLink / NVSwitch).  The step then needs no NCCL send/recv:
//   K3 (gather + decay) stores each piece straight into the OWNER's receive window (push),
//   one LSA barrier, the owner runs its NS on its local window, one LSA barrier,
//   K7 (sparse update) loads its piece of O straight from the owner's outgoing window (pull).
// Both barriers are one-CTA kernels (ncclLsaBarrierSession, acquire-release at system scope);
// kernel boundaries order the pushes / pulls of K3 and K7 against them.  The next step's K3
// cannot overwrite an owner's receive window while that owner's NS still reads it, nor an
// owner's apply overwrite its outgoing window while a rank still pulls: each of those accesses
// sits behind a barrier that the other side only reaches after it is done.
//
// The peer base addresses are read once at setup (ncclGetPeerPointer in a tiny kernel) and
// used as ordinary pointers by the existing gather / scatter kernels, so the fused path is the
// same K3 / K7 code with different destinations.  Host NCCL entry points are resolved with
// dlsym from the process's libnccl (torch's 2.28.9); the device functions are the header-only
// NCCL device API.  Built without the NCCL device headers, setup reports DION2_EUNSUPPORTED.
#include <dlfcn.h>

#include <vector>

#include "dion2.h"
#include "symm.h"

#if __has_include(<nccl_device.h>)
#define DION2_HAVE_NCCL_DEVICE 1
#include <nccl.h>
#include <nccl_device.h>
#endif

namespace dion2 {

#ifdef DION2_HAVE_NCCL_DEVICE

struct SymmState {
  ncclComm_t comm = nullptr;
  void* buf[2] = {nullptr, nullptr};        // receive window, outgoing window
  ncclWindow_t win[2] = {nullptr, nullptr};
  ncclDevComm dev{};
};

namespace {

struct SymmApi {
  ncclResult_t (*mem_alloc)(void**, size_t) = nullptr;
  ncclResult_t (*win_register)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
  ncclResult_t (*devcomm_create)(ncclComm_t, const ncclDevCommRequirements_t*, ncclDevComm_t*) = nullptr;
  ncclTeam_t (*team_lsa)(ncclComm_t) = nullptr;
  ncclResult_t (*mem_free)(void*) = nullptr;
  ncclResult_t (*allreduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
      nullptr;
  bool ok = false;
};

SymmApi& symm_api() {
  static SymmApi api = [] {
    SymmApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.mem_alloc = reinterpret_cast<decltype(a.mem_alloc)>(dlsym(h, "ncclMemAlloc"));
    a.win_register = reinterpret_cast<decltype(a.win_register)>(dlsym(h, "ncclCommWindowRegister"));
    a.devcomm_create = reinterpret_cast<decltype(a.devcomm_create)>(dlsym(h, "ncclDevCommCreate"));
    a.team_lsa = reinterpret_cast<decltype(a.team_lsa)>(dlsym(h, "ncclTeamLsa"));
    a.mem_free = reinterpret_cast<decltype(a.mem_free)>(dlsym(h, "ncclMemFree"));
    a.allreduce = reinterpret_cast<decltype(a.allreduce)>(dlsym(h, "ncclAllReduce"));
    a.ok = a.mem_alloc && a.win_register && a.devcomm_create && a.team_lsa && a.mem_free && a.allreduce;
    return a;
  }();
  return api;
}

// out[p] = rank p's receive window, out[P + p] = rank p's outgoing window, as mapped here
__global__ void k_symm_peers(ncclWindow_t wrecv, ncclWindow_t wosend, int P, void** out) {
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    out[p] = ncclGetPeerPointer(wrecv, 0, p);
    out[P + p] = ncclGetPeerPointer(wosend, 0, p);
  }
}

// every rank arrives (release: this rank's earlier kernels' peer stores / loads are done) and
// waits for every other rank (acquire)
__global__ void k_symm_barrier(ncclDevComm dev) {
  __threadfence_system();
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dev, ncclTeamTagLsa(), 0);
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

}  // namespace

int symm_create(void* comm, int world, size_t bytes, cudaStream_t s, SymmState** out, uint8_t** local_recv,
                uint8_t** local_osend, std::vector<uint8_t*>& peer_recv, std::vector<uint8_t*>& peer_osend) {
  SymmApi& api = symm_api();
  if (!api.ok || !comm) return DION2_EUNSUPPORTED;
  ncclComm_t cm = reinterpret_cast<ncclComm_t>(comm);
  const ncclTeam_t lsa = api.team_lsa(cm);
  if (lsa.nRanks != world) return DION2_EUNSUPPORTED;  // every rank must be load/store reachable
  auto* st = new SymmState();
  st->comm = cm;
  const size_t sz = (bytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
  // the (local) allocations first, then agree on them over the communicator: every rank falls
  // back to send / recv together if any rank could not allocate, before the collective
  // registrations
  int ok = 1;
  for (int b = 0; b < 2; ++b)
    if (api.mem_alloc(&st->buf[b], sz) != ncclSuccess) {
      st->buf[b] = nullptr;
      ok = 0;
    }
  int* dok = nullptr;
  int all_ok = 0;
  if (cudaMalloc(&dok, sizeof(int)) != cudaSuccess) return DION2_ECUDA;
  if (cudaMemcpyAsync(dok, &ok, sizeof(int), cudaMemcpyHostToDevice, s) != cudaSuccess ||
      api.allreduce(dok, dok, 1, ncclInt32, ncclMin, cm, s) != ncclSuccess ||
      cudaMemcpyAsync(&all_ok, dok, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess) {
    cudaFree(dok);
    return DION2_ENCCL;
  }
  cudaFree(dok);
  if (!all_ok) {
    for (int b = 0; b < 2; ++b)
      if (st->buf[b]) api.mem_free(st->buf[b]);
    delete st;
    return DION2_EUNSUPPORTED;
  }
  for (int b = 0; b < 2; ++b)
    if (api.win_register(cm, st->buf[b], sz, &st->win[b], NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess) return DION2_ENCCL;
  ncclDevCommRequirements_t req{};
  req.lsaBarrierCount = 1;
  if (api.devcomm_create(cm, &req, &st->dev) != ncclSuccess) return DION2_ENCCL;
  void** dptr = nullptr;
  if (cudaMalloc(&dptr, 2 * sizeof(void*) * world) != cudaSuccess) return DION2_ECUDA;
  k_symm_peers<<<1, 32, 0, s>>>(st->win[0], st->win[1], world, dptr);
  std::vector<void*> h(2 * world);
  const bool got = cudaMemcpyAsync(h.data(), dptr, 2 * sizeof(void*) * world, cudaMemcpyDeviceToHost, s) == cudaSuccess &&
                   cudaStreamSynchronize(s) == cudaSuccess;
  cudaFree(dptr);
  if (!got) return DION2_ECUDA;
  peer_recv.resize(world);
  peer_osend.resize(world);
  for (int p = 0; p < world; ++p) {
    peer_recv[p] = static_cast<uint8_t*>(h[p]);
    peer_osend[p] = static_cast<uint8_t*>(h[world + p]);
  }
  *local_recv = static_cast<uint8_t*>(st->buf[0]);
  *local_osend = static_cast<uint8_t*>(st->buf[1]);
  *out = st;
  return DION2_OK;
}

int symm_barrier(SymmState* st, cudaStream_t s) {
  if (!st) return DION2_EINVAL_CONFIG;
  k_symm_barrier<<<1, 128, 0, s>>>(st->dev);
  return cudaGetLastError() == cudaSuccess ? DION2_OK : DION2_ECUDA;
}

#else  // built without the NCCL device headers

struct SymmState {};
int symm_create(void*, int, size_t, cudaStream_t, SymmState**, uint8_t**, uint8_t**, std::vector<uint8_t*>&,
                std::vector<uint8_t*>&) {
  return DION2_EUNSUPPORTED;
}
int symm_barrier(SymmState*, cudaStream_t) { return DION2_EUNSUPPORTED; }

#endif

}  // namespace dion2
