// Host-staged sum-allreduce between rank processes on one machine (hostcoll.cpp).
#pragma once
#include <cuda_runtime.h>

#include <string>

namespace rs {

struct HostColl;
// attach to the shared-memory group `name` as rank / world (blocks until every rank attached)
HostColl* hostcoll_create(const char* name, int rank, int world, std::string* err);
void hostcoll_destroy(HostColl* h);
// enqueue buf[0:count) <- sum over ranks (rank order) on stream st (capturable in a CUDA graph)
cudaError_t hostcoll_allreduce(HostColl* h, double* buf, size_t count, cudaStream_t st);
bool hostcoll_failed(const HostColl* h);   // a barrier timed out
void hostcoll_new_name(char* out128);

}  // namespace rs
