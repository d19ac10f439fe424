// comm.hpp — the collective of the split step path: an all-gather of each
// window's spike bitmasks (plus a sum for NaN counters), over NCCL.
// libnccl is loaded with dlopen on first use, so a process that never
// splits a network needs no NCCL (and one that imported torch reuses the
// libnccl.so.2 torch already loaded).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstddef>
#include <memory>

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
    // point to point (the rank pipeline's partial sums, fp32)
    void send_f32(const void* buf, std::size_t count, int peer, cudaStream_t s);
    void recv_f32(void* buf, std::size_t count, int peer, cudaStream_t s);
    // a second communicator over the same ranks (ncclCommSplit): point-to-point
    // traffic on its own stream never orders against this one's
    std::unique_ptr<Comm> split() const;
    int world() const { return world_; }
    int rank() const { return rank_; }

private:
    Comm() = default;
    void* comm_ = nullptr;
    int world_ = 1, rank_ = 0;
};

std::array<unsigned char, 128> nccl_unique_id();

}  // namespace ssb
