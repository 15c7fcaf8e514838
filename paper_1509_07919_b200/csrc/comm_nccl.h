// Native NCCL data plane of the distributed handle (comm_nccl.cu).
#pragma once

#include <string>

#include "common.cuh"

namespace sapgpu {

constexpr int kNcclIdBytes = 128;
struct NcclComm;

void nccl_unique_id(unsigned char* out);                                // rank 0, shared out of band
NcclComm* nccl_create(const unsigned char* id, int rank, int world);  // collective over the ranks
void nccl_destroy(NcclComm* c);
// neighbour exchange of device buffers on stream s (left = rank - 1, right = rank + 1; counts may be 0)
void nccl_exchange(NcclComm* c, const double* sl, int n_sl, const double* sr, int n_sr, double* rl, int n_rl,
                   double* rr, int n_rr, cudaStream_t s);
// in-place sum over ranks of count device doubles on stream s
void nccl_allreduce(NcclComm* c, double* d, int count, cudaStream_t s);
bool nccl_available(std::string* why);

}  // namespace sapgpu
