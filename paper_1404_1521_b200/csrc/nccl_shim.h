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
int nccl_shim_allgather_bytes(const void* send, void* recv, size_t bytes, void* comm, cudaStream_t s,
                              std::string* err);
int nccl_shim_allreduce_sum_f32(const float* send, float* recv, size_t count, void* comm, cudaStream_t s,
                                std::string* err);
// symmetric-memory windows (PEER exchange)
bool nccl_shim_has_symmetric();
int nccl_shim_lsa_size(void* comm);   // ranks reachable by load/store (0: unavailable)
int nccl_shim_mem_alloc(void** ptr, size_t bytes, std::string* err);
int nccl_shim_mem_free(void* ptr);
int nccl_shim_window_register(void* comm, void* buf, size_t bytes, void** win, std::string* err);
int nccl_shim_window_deregister(void* comm, void* win);
// nccl_lsa.cu: the load/store address of every rank's copy of the window
// (device-side ncclGetLsaPointer), written to host out[world]
int nccl_lsa_pointers(void* win, int world, unsigned long long* out, std::string* err);
