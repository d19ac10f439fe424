// comm.hpp — the collective of the split step path: an all-gather of each
// window's spike bitmasks (plus a sum for NaN counters), over NCCL.
// libnccl is loaded with dlopen on first use, so a process that never
// splits a network needs no NCCL (and one that imported torch reuses the
// libnccl.so.2 torch already loaded).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstddef>

namespace ssb {

class Comm {
public:
    Comm(int world, int rank, const unsigned char* id128);
    ~Comm();
    Comm(const Comm&) = delete;
    Comm& operator=(const Comm&) = delete;
    // recv[world][count] <- every rank's send[count] (32-bit words), in rank order
    void allgather_u32(const void* send, void* recv, std::size_t count, cudaStream_t s);
    void allreduce_sum_u64(void* buf, std::size_t count, cudaStream_t s);
    int world() const { return world_; }
    int rank() const { return rank_; }

private:
    void* comm_ = nullptr;
    int world_ = 1, rank_ = 0;
};

std::array<unsigned char, 128> nccl_unique_id();

}  // namespace ssb
