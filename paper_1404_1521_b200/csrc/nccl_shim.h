// nccl_shim.h -- NCCL entry points resolved at run time with dlopen, so libpg
// loads without NCCL and a process never maps two different libnccl builds
// (torch's 2.28 is found first when torch is already loaded).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include <string>

int nccl_shim_unique_id(void* out128, std::string* err);
int nccl_shim_init(void** comm, int rank, int world, const void* uid128, std::string* err);
int nccl_shim_allgather_f32(const float* send, float* recv, size_t count, void* comm, cudaStream_t s,
                            std::string* err);
int nccl_shim_destroy(void* comm);
int nccl_shim_group(bool start, std::string* err);
