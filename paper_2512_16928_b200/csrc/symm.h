// Direct peer exchange over NCCL symmetric memory (k_symm.cu): the setup and the barrier the
// distributed step uses when DION2_FLAG_DIST_DIRECT is set.  Plain C++ interface (no NCCL
// types) so dion2_dist.cu does not depend on the NCCL headers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace dion2 {

struct SymmState;

// Collective over the communicator (every rank calls it with the same `bytes`): allocates the
// receive and outgoing windows (`bytes` each, ncclMemAlloc + symmetric registration), a device
// communicator with one LSA barrier, and returns this rank's window bases and every rank's
// window bases as mapped into this process.  DION2_EUNSUPPORTED when NCCL lacks the device API
// or not every rank is load/store reachable (one NVLink domain), or any rank could not allocate
// its windows (agreed with one all-reduce before the collective registration, so every rank
// returns the same code).  Synchronises `s`.
int symm_create(void* comm, int world, size_t bytes, cudaStream_t s, SymmState** out, uint8_t** local_recv,
                uint8_t** local_osend, std::vector<uint8_t*>& peer_recv, std::vector<uint8_t*>& peer_osend);

// One LSA barrier over all ranks on stream s (a one-CTA kernel).
int symm_barrier(SymmState* st, cudaStream_t s);

}  // namespace dion2
