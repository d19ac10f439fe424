// standalone.cu — the reference's free functions propagate() and
// detect_nans() (engine.cpp:27-80) as device kernels over caller arrays.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../engine.hpp"
#include "kernels.cuh"
#include "synscale/synscale.hpp"

namespace ssb {

namespace {

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw DeviceError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
#define CK(x) check((x), #x)

// RAII device buffer for the host-array entry points.
struct Buf {
    void* p = nullptr;
    explicit Buf(std::size_t bytes) { CK(cudaMalloc(&p, bytes ? bytes : 1)); }
    ~Buf() { cudaFree(p); }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

void require_device() {
    if (device_count() == 0) throw DeviceError("no CUDA device is visible (no CPU path exists)");
}

constexpr int kTile = 256;

}  // namespace

void device_propagate_dense_dev(const float* w, int nPre, int nPost, const std::int32_t* spikes,
                                int nSpikes, float* acc, void* stream) {
    (void)nPre;
    if (nPost <= 0 || nSpikes <= 0) return;
    const bool vec = nPost % 4 == 0 && reinterpret_cast<std::uintptr_t>(w) % 16 == 0 &&
                     reinterpret_cast<std::uintptr_t>(acc) % 16 == 0;
    if (vec)
        ssbk::propagate_dense4_kernel<<<(nPost / 4 + 255) / 256, 256, 0,
                                        static_cast<cudaStream_t>(stream)>>>(w, nPost, spikes,
                                                                             nSpikes, acc);
    else
        ssbk::propagate_dense_kernel<<<(nPost + 127) / 128, 128, 0,
                                       static_cast<cudaStream_t>(stream)>>>(w, nPost, spikes,
                                                                            nSpikes, acc);
    CK(cudaGetLastError());
}

void device_crs_segments_dev(const std::int32_t* ind, const std::int64_t* rowStart, int nPre,
                             int nPost, int tile, std::int32_t* seg, void* stream) {
    const int nTiles = (nPost + tile - 1) / tile;
    const long long total = static_cast<long long>(nPre) * (nTiles + 1);
    if (total <= 0) return;
    ssbk::crs_segments_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0,
                                static_cast<cudaStream_t>(stream)>>>(
        ind, reinterpret_cast<const long long*>(rowStart), nPre, nTiles, tile, seg);
    CK(cudaGetLastError());
}

void device_propagate_crs_dev(const float* g, const std::int32_t* ind, const std::int32_t* seg,
                              int tile, int nPre, int nPost, const std::int32_t* spikes,
                              int nSpikes, float* acc, void* stream) {
    (void)nPre;
    if (nPost <= 0 || nSpikes <= 0) return;
    const int nTiles = (nPost + tile - 1) / tile;
    ssbk::propagate_crs_kernel<<<nTiles, tile, 0, static_cast<cudaStream_t>(stream)>>>(
        g, ind, seg, nTiles, nPost, spikes, nSpikes, acc);
    CK(cudaGetLastError());
}

std::int64_t crs_slices(const float* g, const std::int32_t* ind, const std::int64_t* rowStart,
                        int nPre, int nPost, std::int64_t* sliceOff, std::int32_t* rows,
                        float* vals, std::int64_t cap) {
    const int nSlices = (nPost + 31) / 32;
    std::vector<std::int64_t> colLen(static_cast<std::size_t>(nPost), 0);
    for (std::int64_t k = 0; k < rowStart[nPre]; ++k) {
        if (ind[k] < 0 || ind[k] >= nPost) throw synscale::SpecError("post index out of range");
        ++colLen[ind[k]];
    }
    sliceOff[0] = 0;
    for (int s = 0; s < nSlices; ++s) {
        std::int64_t m = 0;
        for (int l = 0; l < 32 && s * 32 + l < nPost; ++l) m = std::max(m, colLen[s * 32 + l]);
        sliceOff[s + 1] = sliceOff[s] + 32 * m;
    }
    const std::int64_t need = sliceOff[nSlices];
    if (!rows || !vals) return need;
    if (cap < need) throw synscale::SpecError("slice arrays too small");
    std::fill(rows, rows + need, -1);
    std::fill(vals, vals + need, 0.0f);
    std::vector<std::int64_t> fill(static_cast<std::size_t>(nPost), 0);
    for (int r = 0; r < nPre; ++r)  // rows ascending: every column stays sorted
        for (std::int64_t k = rowStart[r]; k < rowStart[r + 1]; ++k) {
            const int j = ind[k];
            const std::int64_t at = sliceOff[j / 32] + 32 * fill[j]++ + (j % 32);
            rows[at] = r;
            vals[at] = g[k];
        }
    return need;
}

void device_propagate_crs_sliced_dev(const std::int32_t* rows, const float* vals,
                                     const std::int64_t* sliceOff, int nPre, int nPost,
                                     const std::int32_t* spikes, int nSpikes, float* acc,
                                     void* stream) {
    if (nPost <= 0 || nSpikes <= 0) return;
    const int smem = ((nPre + 31) / 32) * 4;
    if (smem > 48 * 1024)
        CK(cudaFuncSetAttribute(ssbk::propagate_crs_sliced_kernel,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int slices = (nPost + 31) / 32;
    const int blocks = std::min((slices + 7) / 8, 148 * 8);
    ssbk::propagate_crs_sliced_kernel<<<blocks, 256, smem, static_cast<cudaStream_t>(stream)>>>(
        rows, vals, reinterpret_cast<const long long*>(sliceOff), nPre, nPost, spikes, nSpikes, acc);
    CK(cudaGetLastError());
}

void device_propagate_dense(const float* w, int nPre, int nPost, const std::int32_t* spikes,
                            std::int64_t nSpikes, float* acc) {
    require_device();
    const std::size_t nw = static_cast<std::size_t>(nPre) * static_cast<std::size_t>(nPost);
    Buf dW(nw * 4), dS(static_cast<std::size_t>(nSpikes) * 4), dA(static_cast<std::size_t>(nPost) * 4);
    CK(cudaMemcpy(dW.p, w, nw * 4, cudaMemcpyHostToDevice));
    if (nSpikes) CK(cudaMemcpy(dS.p, spikes, static_cast<std::size_t>(nSpikes) * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dA.p, acc, static_cast<std::size_t>(nPost) * 4, cudaMemcpyHostToDevice));
    device_propagate_dense_dev(dW.as<float>(), nPre, nPost, dS.as<std::int32_t>(),
                               static_cast<int>(nSpikes), dA.as<float>(), nullptr);
    CK(cudaMemcpy(acc, dA.p, static_cast<std::size_t>(nPost) * 4, cudaMemcpyDeviceToHost));
}

void device_propagate_crs(const float* g, const std::int32_t* ind, const std::int64_t* rowStart,
                          int nPre, int nPost, const std::int32_t* spikes, std::int64_t nSpikes,
                          float* acc) {
    require_device();
    const std::size_t nnz = static_cast<std::size_t>(rowStart[nPre]);
    bool ascending = true;
    for (std::int64_t k = 1; k < nSpikes && ascending; ++k) ascending = spikes[k] > spikes[k - 1];
    if (ascending && nSpikes > 0 && nPost > 0) {
        // column slices: coalesced at every density (gather_tma.cuh)
        std::vector<std::int64_t> off(static_cast<std::size_t>((nPost + 31) / 32) + 1);
        const std::int64_t need = crs_slices(g, ind, rowStart, nPre, nPost, off.data(), nullptr,
                                             nullptr, 0);
        std::vector<std::int32_t> rows(static_cast<std::size_t>(need));
        std::vector<float> vals(static_cast<std::size_t>(need));
        crs_slices(g, ind, rowStart, nPre, nPost, off.data(), rows.data(), vals.data(), need);
        Buf dR(rows.size() * 4), dV(vals.size() * 4), dO(off.size() * 8),
            dS(static_cast<std::size_t>(nSpikes) * 4), dA(static_cast<std::size_t>(nPost) * 4);
        if (need) {
            CK(cudaMemcpy(dR.p, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dV.p, vals.data(), vals.size() * 4, cudaMemcpyHostToDevice));
        }
        CK(cudaMemcpy(dO.p, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dS.p, spikes, static_cast<std::size_t>(nSpikes) * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dA.p, acc, static_cast<std::size_t>(nPost) * 4, cudaMemcpyHostToDevice));
        device_propagate_crs_sliced_dev(dR.as<std::int32_t>(), dV.as<float>(), dO.as<std::int64_t>(),
                                        nPre, nPost, dS.as<std::int32_t>(),
                                        static_cast<int>(nSpikes), dA.as<float>(), nullptr);
        CK(cudaMemcpy(acc, dA.p, static_cast<std::size_t>(nPost) * 4, cudaMemcpyDeviceToHost));
        return;
    }
    const int nTiles = (nPost + kTile - 1) / kTile;
    Buf dG(nnz * 4), dI(nnz * 4), dR((static_cast<std::size_t>(nPre) + 1) * 8),
        dSeg(static_cast<std::size_t>(nPre) * (nTiles + 1) * 4),
        dS(static_cast<std::size_t>(nSpikes) * 4), dA(static_cast<std::size_t>(nPost) * 4);
    if (nnz) {
        CK(cudaMemcpy(dG.p, g, nnz * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dI.p, ind, nnz * 4, cudaMemcpyHostToDevice));
    }
    CK(cudaMemcpy(dR.p, rowStart, (static_cast<std::size_t>(nPre) + 1) * 8, cudaMemcpyHostToDevice));
    if (nSpikes) CK(cudaMemcpy(dS.p, spikes, static_cast<std::size_t>(nSpikes) * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dA.p, acc, static_cast<std::size_t>(nPost) * 4, cudaMemcpyHostToDevice));
    device_crs_segments_dev(dI.as<std::int32_t>(), dR.as<std::int64_t>(), nPre, nPost, kTile,
                            dSeg.as<std::int32_t>(), nullptr);
    device_propagate_crs_dev(dG.as<float>(), dI.as<std::int32_t>(), dSeg.as<std::int32_t>(), kTile,
                             nPre, nPost, dS.as<std::int32_t>(), static_cast<int>(nSpikes),
                             dA.as<float>(), nullptr);
    CK(cudaMemcpy(acc, dA.p, static_cast<std::size_t>(nPost) * 4, cudaMemcpyDeviceToHost));
}

std::int64_t device_detect_nans(int kind, const float* v, const float* u, const float* gExc,
                                const float* gInh, std::uint8_t* flag, std::int64_t n) {
    require_device();
    if (n <= 0) return 0;
    const std::size_t fb = static_cast<std::size_t>(n) * 4;
    auto up = [&](const float* src) {
        auto b = std::make_unique<Buf>(fb);
        if (src) CK(cudaMemcpy(b->p, src, fb, cudaMemcpyHostToDevice));
        else CK(cudaMemset(b->p, 0, fb));
        return b;
    };
    auto dv = up(v), du = up(u), dge = up(gExc), dgi = up(gInh);
    Buf dF(static_cast<std::size_t>(n)), dN(8);
    CK(cudaMemcpy(dF.p, flag, static_cast<std::size_t>(n), cudaMemcpyHostToDevice));
    CK(cudaMemset(dN.p, 0, 8));
    const int blocks = static_cast<int>(std::min<std::int64_t>((n + 255) / 256, 148 * 8));
    ssbk::detect_nans_kernel<<<blocks, 256>>>(kind, dv->as<float>(), du->as<float>(),
                                              dge->as<float>(), dgi->as<float>(),
                                              dF.as<std::uint8_t>(), n,
                                              dN.as<unsigned long long>());
    CK(cudaGetLastError());
    unsigned long long newly = 0;
    CK(cudaMemcpy(&newly, dN.p, 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(flag, dF.p, static_cast<std::size_t>(n), cudaMemcpyDeviceToHost));
    return static_cast<std::int64_t>(newly);
}

}  // namespace ssb
