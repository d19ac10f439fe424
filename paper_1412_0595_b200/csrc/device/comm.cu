// comm.cu — NCCL through dlopen (see comm.hpp).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../engine.hpp"
#include "comm.hpp"

namespace ssb {

namespace {

struct Nccl {
    void* lib = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            n.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (n.lib) break;
        }
        if (!n.lib) return;
        n.getUniqueId = reinterpret_cast<decltype(n.getUniqueId)>(dlsym(n.lib, "ncclGetUniqueId"));
        n.commInitRank = reinterpret_cast<decltype(n.commInitRank)>(dlsym(n.lib, "ncclCommInitRank"));
        n.commDestroy = reinterpret_cast<decltype(n.commDestroy)>(dlsym(n.lib, "ncclCommDestroy"));
        n.allGather = reinterpret_cast<decltype(n.allGather)>(dlsym(n.lib, "ncclAllGather"));
        n.allReduce = reinterpret_cast<decltype(n.allReduce)>(dlsym(n.lib, "ncclAllReduce"));
        n.errorString = reinterpret_cast<decltype(n.errorString)>(dlsym(n.lib, "ncclGetErrorString"));
        n.send = reinterpret_cast<decltype(n.send)>(dlsym(n.lib, "ncclSend"));
        n.recv = reinterpret_cast<decltype(n.recv)>(dlsym(n.lib, "ncclRecv"));
        n.commSplit = reinterpret_cast<decltype(n.commSplit)>(dlsym(n.lib, "ncclCommSplit"));
        n.groupStart = reinterpret_cast<decltype(n.groupStart)>(dlsym(n.lib, "ncclGroupStart"));
        n.groupEnd = reinterpret_cast<decltype(n.groupEnd)>(dlsym(n.lib, "ncclGroupEnd"));
    });
    if (!n.lib || !n.getUniqueId || !n.commInitRank || !n.allGather || !n.allReduce)
        throw DeviceError("NCCL (libnccl.so.2) is not available for a multi-GPU run");
    return n;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw DeviceError(std::string("NCCL error in ") + what + ": " +
                          (nccl().errorString ? nccl().errorString(r) : std::to_string(r)));
}

}  // namespace

std::array<unsigned char, 128> nccl_unique_id() {
    ncclUniqueId id;
    nck(nccl().getUniqueId(&id), "ncclGetUniqueId");
    std::array<unsigned char, 128> out{};
    std::memcpy(out.data(), id.internal, 128);
    return out;
}

std::array<unsigned char, 128> comm_unique_id() { return nccl_unique_id(); }

Comm::Comm(int world, int rank, const unsigned char* id128) : world_(world), rank_(rank) {
    ncclUniqueId id;
    std::memcpy(id.internal, id128, 128);
    ncclComm_t c = nullptr;
    nck(nccl().commInitRank(&c, world, id, rank), "ncclCommInitRank");
    comm_ = c;
}

Comm::~Comm() {
    if (comm_ && nccl().commDestroy) nccl().commDestroy(static_cast<ncclComm_t>(comm_));
}

void Comm::allgather_u32(const void* send, void* recv, std::size_t count, cudaStream_t s) {
    nck(nccl().allGather(send, recv, count, ncclUint32, static_cast<ncclComm_t>(comm_), s),
        "ncclAllGather");
}

void Comm::allreduce_sum_u64(void* buf, std::size_t count, cudaStream_t s) {
    nck(nccl().allReduce(buf, buf, count, ncclUint64, ncclSum, static_cast<ncclComm_t>(comm_), s),
        "ncclAllReduce");
}

void Comm::send_f32(const void* buf, std::size_t count, int peer, cudaStream_t s) {
    if (!nccl().send) throw DeviceError("ncclSend is not available");
    nck(nccl().send(buf, count, ncclFloat32, peer, static_cast<ncclComm_t>(comm_), s), "ncclSend");
}

void Comm::recv_f32(void* buf, std::size_t count, int peer, cudaStream_t s) {
    if (!nccl().recv) throw DeviceError("ncclRecv is not available");
    nck(nccl().recv(buf, count, ncclFloat32, peer, static_cast<ncclComm_t>(comm_), s), "ncclRecv");
}

std::unique_ptr<Comm> Comm::split() const {
    if (!nccl().commSplit) throw DeviceError("ncclCommSplit is not available");
    ncclComm_t c = nullptr;
    nck(nccl().commSplit(static_cast<ncclComm_t>(comm_), 0, rank_, &c, nullptr), "ncclCommSplit");
    std::unique_ptr<Comm> out(new Comm());
    out->comm_ = c;
    out->world_ = world_;
    out->rank_ = rank_;
    return out;
}

}  // namespace ssb

namespace ssb {

void comm_selftest(int device) {
    auto ck = [](cudaError_t e, const char* what) {
        if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
    };
    ck(cudaSetDevice(device), "cudaSetDevice");
    const auto id = nccl_unique_id();
    Comm comm(1, 0, id.data());
    cudaStream_t s;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    constexpr int n = 1000;
    std::uint32_t* send = nullptr;
    std::uint32_t* recv = nullptr;
    unsigned long long* sum = nullptr;
    ck(cudaMalloc(&send, n * 4), "cudaMalloc");
    ck(cudaMalloc(&recv, n * 4), "cudaMalloc");
    ck(cudaMalloc(&sum, 8), "cudaMalloc");
    std::vector<std::uint32_t> h(n), back(n);
    for (int i = 0; i < n; ++i) h[i] = 0x9e3779b9u * static_cast<std::uint32_t>(i + 1);
    ck(cudaMemcpy(send, h.data(), n * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
    const unsigned long long seven = 7;
    ck(cudaMemcpy(sum, &seven, 8, cudaMemcpyHostToDevice), "cudaMemcpy");
    comm.allgather_u32(send, recv, n, s);
    comm.allreduce_sum_u64(sum, 1, s);
    // the same all-gather captured in a graph, as the window graphs issue it
    cudaGraph_t g;
    cudaGraphExec_t ge;
    ck(cudaMemsetAsync(recv, 0, n * 4, s), "cudaMemsetAsync");
    ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    comm.allgather_u32(send, recv, n, s);
    ck(cudaStreamEndCapture(s, &g), "cudaStreamEndCapture");
    ck(cudaGraphInstantiate(&ge, g, 0), "cudaGraphInstantiate");
    ck(cudaGraphLaunch(ge, s), "cudaGraphLaunch");
    ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    unsigned long long got = 0;
    ck(cudaMemcpy(back.data(), recv, n * 4, cudaMemcpyDeviceToHost), "cudaMemcpy");
    ck(cudaMemcpy(&got, sum, 8, cudaMemcpyDeviceToHost), "cudaMemcpy");
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaFree(send);
    cudaFree(recv);
    cudaFree(sum);
    if (back != h) throw DeviceError("NCCL self-test: all-gather returned wrong words");
    if (got != 7) throw DeviceError("NCCL self-test: all-reduce returned a wrong sum");
    // the rank pipeline's pieces: a split communicator and fp32 send / recv
    // (to this rank itself, in one group), captured in a graph
    auto split = comm.split();
    float* a = nullptr;
    float* b = nullptr;
    ck(cudaMalloc(&a, n * 4), "cudaMalloc");
    ck(cudaMalloc(&b, n * 4), "cudaMalloc");
    std::vector<float> hf(n), bf(n);
    for (int i = 0; i < n; ++i) hf[i] = 0.25f * static_cast<float>(i) - 3.0f;
    ck(cudaMemcpy(a, hf.data(), n * 4, cudaMemcpyHostToDevice), "cudaMemcpy");
    ck(cudaMemset(b, 0, n * 4), "cudaMemset");
    if (!nccl().groupStart || !nccl().groupEnd) throw DeviceError("ncclGroupStart/End unavailable");
    ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    nck(nccl().groupStart(), "ncclGroupStart");
    split->send_f32(a, n, 0, s);
    split->recv_f32(b, n, 0, s);
    nck(nccl().groupEnd(), "ncclGroupEnd");
    ck(cudaStreamEndCapture(s, &g), "cudaStreamEndCapture");
    ck(cudaGraphInstantiate(&ge, g, 0), "cudaGraphInstantiate");
    ck(cudaGraphLaunch(ge, s), "cudaGraphLaunch");
    ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    ck(cudaMemcpy(bf.data(), b, n * 4, cudaMemcpyDeviceToHost), "cudaMemcpy");
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaFree(a);
    cudaFree(b);
    cudaStreamDestroy(s);
    if (bf != hf) throw DeviceError("NCCL self-test: send / recv returned wrong values");
}

}  // namespace ssb
