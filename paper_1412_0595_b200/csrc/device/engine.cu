// engine.cu — DeviceEngine: device memory layout, launch schedule, CUDA
// graphs and raster management of the windowed step engine.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <numeric>
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

int round_up(int v, int u) { return (v + u - 1) / u * u; }

}  // namespace

int device_count() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

DeviceProps device_props(int device) {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, device));
    DeviceProps d;
    d.name = p.name;
    d.smCount = p.multiProcessorCount;
    d.warpSize = p.warpSize;
    d.maxThreadsPerSM = p.maxThreadsPerMultiProcessor;
    d.maxBlocksPerSM = p.maxBlocksPerMultiProcessor;
    d.maxThreadsPerBlock = p.maxThreadsPerBlock;
    d.regsPerSM = p.regsPerMultiprocessor;
    d.sharedPerSM = static_cast<std::int64_t>(p.sharedMemPerMultiprocessor);
    d.sharedPerBlockOptin = static_cast<std::int64_t>(p.sharedMemPerBlockOptin);
    return d;
}

bool kernel_attributes(const std::string& name, int& regs, int& sharedBytes, int& maxThreads) {
    cudaFuncAttributes a;
    cudaError_t e;
    if (name == "condlif_window") e = cudaFuncGetAttributes(&a, ssbk::condlif_window_kernel);
    else if (name == "poisson_window") e = cudaFuncGetAttributes(&a, ssbk::poisson_window_kernel);
    else if (name == "dense_window") e = cudaFuncGetAttributes(&a, ssbk::dense_window_kernel);
    else if (name == "sparse_window") e = cudaFuncGetAttributes(&a, ssbk::sparse_window_kernel);
    else if (name == "compact_window") e = cudaFuncGetAttributes(&a, ssbk::compact_window_kernel);
    else if (name == "raster_window") e = cudaFuncGetAttributes(&a, ssbk::raster_window_kernel);
    else if (name == "propagate_dense") e = cudaFuncGetAttributes(&a, ssbk::propagate_dense_kernel);
    else if (name == "propagate_crs") e = cudaFuncGetAttributes(&a, ssbk::propagate_crs_kernel);
    else return false;
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    regs = a.numRegs;
    sharedBytes = static_cast<int>(a.sharedSizeBytes);
    maxThreads = a.maxThreadsPerBlock;
    return true;
}

// ---------------------------------------------------------------------------

struct DeviceEngine::Impl {
    struct PopRt {
        int kind = 0, n = 0, nwords = 0;
        int block = 0, grid = 0;
        bool sparseInline = false;  // needs a dynamic shared tile
        ssbk::PopDev dev{};
        ssbk::AccDev acc[2]{};
        std::vector<int> accGroups[2];  // group indices in spec order
        std::string name;
    };
    struct LaunchStat {
        std::string name;
        std::int64_t launches = 0;
        double ms = 0.0;
    };

    EngineConfig cfg;
    int Wmax = 1;
    bool stepMode = false;
    int smCount = 148;
    cudaStream_t stream = nullptr;
    std::vector<PopRt> pops;
    std::vector<HostGroup> groupMeta;  // sizes only (arrays cleared)
    std::vector<ssbk::GroupDev> groupDev;
    std::vector<int> order;
    std::vector<void*> allocations;
    std::int64_t bytes = 0;
    std::int64_t totalNeurons = 0;
    std::int64_t stepsTotal = 0;
    std::int64_t stepsDone = 0;
    std::int64_t windowsLaunched = 0;

    // raster
    ssbk::RasterDev raster{};
    std::int64_t rasterCap = 0;
    std::int64_t eventBound = 0;  // upper bound of events in the arena
    std::vector<std::int32_t> hostNeurons;
    bool rasterDiscarded = false;

    std::map<int, cudaGraphExec_t> graphs;

    // profiling
    std::map<std::string, LaunchStat> stats;
    std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::vector<cudaEvent_t> eventPool;

    template <typename T>
    T* alloc(std::size_t count) {
        void* p = nullptr;
        const std::size_t b = std::max<std::size_t>(count, 1) * sizeof(T);
        CK(cudaMalloc(&p, b));
        CK(cudaMemsetAsync(p, 0, b, stream));
        allocations.push_back(p);
        bytes += static_cast<std::int64_t>(b);
        return static_cast<T*>(p);
    }
    template <typename T>
    T* upload(const T* src, std::size_t count) {
        T* d = alloc<T>(count);
        if (count) CK(cudaMemcpyAsync(d, src, count * sizeof(T), cudaMemcpyHostToDevice, stream));
        return d;
    }

    cudaEvent_t take_event() {
        if (!eventPool.empty()) {
            cudaEvent_t e = eventPool.back();
            eventPool.pop_back();
            return e;
        }
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        return e;
    }

    template <typename F>
    void launch(const std::string& name, F&& f) {
        if (!cfg.profile) {
            f();
            CK(cudaGetLastError());
            return;
        }
        cudaEvent_t a = take_event(), b = take_event();
        CK(cudaEventRecord(a, stream));
        f();
        CK(cudaGetLastError());
        CK(cudaEventRecord(b, stream));
        pending.push_back({name, {a, b}});
    }

    void harvest() {
        if (pending.empty()) return;
        CK(cudaStreamSynchronize(stream));
        for (auto& [name, ev] : pending) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ev.first, ev.second));
            auto& s = stats[name];
            s.name = name;
            s.launches += 1;
            s.ms += ms;
            eventPool.push_back(ev.first);
            eventPool.push_back(ev.second);
        }
        pending.clear();
    }

    int choose_block(int n, bool sparseInline) const;
    void build(const HostNet& net);
    void enqueue_window(int W);
    void run_window(int W);
    void flush_raster();
};

int DeviceEngine::Impl::choose_block(int n, bool sparseInline) const {
    const int single = std::min(1024, round_up(std::max(n, 1), 32));
    if (cfg.blockSize > 0) return std::min(round_up(cfg.blockSize, 32), 1024);
    int regs = 32, shared = 0, maxThreads = 1024;
    kernel_attributes("condlif_window", regs, shared, maxThreads);
    synscale::DeviceSpec dev = synscale::device_preset("sm100");
    auto smemFor = [&](int bs) {
        return static_cast<std::int64_t>(shared) + (sparseInline ? bs * 4 : 0);
    };
    if (cfg.blockPolicy == 1) {
        // the paper's model as is: highest occupancy, ties to the larger block
        // (reference occupancy.cpp:79-101), capped by what one block needs
        const auto [bs, r] = synscale::recommend_block_size(dev, regs, smemFor(1024));
        (void)r;
        return std::min<int>(static_cast<int>(bs), single);
    }
    // Default: the same model, restricted to block sizes whose grid still
    // covers every SM (the model is per-SM and blind to wave quantisation).
    int best = 0;
    std::int64_t bestWarps = -1;
    for (int bs = 32; bs <= std::min(maxThreads, 1024); bs += 32) {
        const int grid = (n + bs - 1) / bs;
        if (grid < smCount && bs != 32) continue;
        const auto r = synscale::occupancy(dev, {bs, regs, smemFor(bs)});
        if (r.activeWarps >= bestWarps) {
            bestWarps = r.activeWarps;
            best = bs;
        }
    }
    if (best == 0 || (n + best - 1) / best < smCount) return single;  // small population
    return best;
}

void DeviceEngine::Impl::build(const HostNet& net) {
    const int nPops = static_cast<int>(net.pops.size());
    if (nPops > ssbk::kMaxPops)
        throw synscale::SpecError("the device engine supports at most " +
                                  std::to_string(ssbk::kMaxPops) + " populations");
    stepsTotal = net.steps;

    // population graph: edges pre -> post for posts that consume input
    std::vector<std::vector<int>> succ(nPops);
    std::vector<int> indeg(nPops, 0);
    bool cyclic = false;
    for (const auto& g : net.groups) {
        if (net.pops[g.post].kind == kPoisson) continue;
        if (g.pre == g.post) cyclic = true;
        succ[g.pre].push_back(g.post);
        ++indeg[g.post];
    }
    {
        std::vector<int> q, deg = indeg;
        for (int i = 0; i < nPops; ++i)
            if (deg[i] == 0) q.push_back(i);
        for (std::size_t h = 0; h < q.size(); ++h)
            for (int s : succ[q[h]])
                if (--deg[s] == 0) q.push_back(s);
        if (static_cast<int>(q.size()) != nPops) cyclic = true;
        order = cyclic ? std::vector<int>() : q;
    }
    for (const auto& p : net.pops)
        if (p.kind == kIzhikevich)
            throw synscale::SpecError(
                "population '" + p.name +
                "': the Izhikevich model is not implemented by the B200 engine yet");
    stepMode = cyclic || cfg.forceStepMode;
    if (stepMode) {
        order.resize(nPops);
        std::iota(order.begin(), order.end(), 0);
    }
    Wmax = stepMode ? 1 : std::max(1, cfg.window);
    if (!stepMode && net.steps > 0) Wmax = static_cast<int>(std::min<std::int64_t>(Wmax, net.steps));

    // accumulator plans
    pops.resize(nPops);
    for (int gi = 0; gi < static_cast<int>(net.groups.size()); ++gi) {
        const auto& g = net.groups[gi];
        pops[g.post].accGroups[g.inhibitory ? 1 : 0].push_back(gi);
    }
    for (int pi = 0; pi < nPops; ++pi) {
        auto& P = pops[pi];
        const auto& hp = net.pops[pi];
        P.kind = hp.kind;
        P.n = hp.n;
        P.name = hp.name;
        P.nwords = (hp.n + 31) / 32;
        totalNeurons += hp.n;
        for (int a = 0; a < 2; ++a) {
            auto& A = P.acc[a];
            const auto& gl = P.accGroups[a];
            if (static_cast<int>(gl.size()) > ssbk::kMaxAccGroups)
                throw synscale::SpecError("population '" + hp.name + "' has more than " +
                                          std::to_string(ssbk::kMaxAccGroups) +
                                          " synapse groups feeding one accumulator");
            A.ng = static_cast<int>(gl.size());
            if (gl.empty()) A.mode = ssbk::kAccNone;
            else if (stepMode || hp.kind == kPoisson) A.mode = ssbk::kAccDeliver;
            else {
                bool heavy = false;
                for (int gi : gl)
                    if (net.groups[gi].preCount >= cfg.heavyPreThreshold) heavy = true;
                A.mode = heavy ? ssbk::kAccBuffered : ssbk::kAccInline;
            }
            if (A.mode == ssbk::kAccInline)
                for (int gi : gl)
                    if (!net.groups[gi].dense) P.sparseInline = true;
        }
        if (hp.kind == kCondLif) {
            P.block = choose_block(hp.n, P.sparseInline);
            P.grid = (hp.n + P.block - 1) / P.block;
        } else {
            P.block = 320;
            P.grid = 1;
        }
    }

    // population buffers
    for (int pi = 0; pi < nPops; ++pi) {
        auto& P = pops[pi];
        const auto& hp = net.pops[pi];
        auto& d = P.dev;
        const std::size_t n = static_cast<std::size_t>(hp.n);
        d.kind = hp.kind;
        d.n = hp.n;
        d.nwords = P.nwords;
        d.Wmax = Wmax;
        d.v = alloc<float>(n);
        d.u = alloc<float>(n);
        d.gExc = alloc<float>(n);
        d.gInh = alloc<float>(n);
        d.excIn = alloc<float>(n);
        d.inhIn = alloc<float>(n);
        d.nanFlag = alloc<uint8_t>(n);
        d.flagged = alloc<unsigned long long>(1);
        d.bits = alloc<uint32_t>(static_cast<std::size_t>(Wmax) * P.nwords);
        d.list = alloc<int>(static_cast<std::size_t>(Wmax) * n);
        d.count = alloc<int>(static_cast<std::size_t>(Wmax));
        d.tauM = hp.tauM;
        d.eLeak = hp.eLeak;
        d.eExc = hp.eExc;
        d.eInh = hp.eInh;
        d.vThresh = hp.vThresh;
        d.vReset = hp.vReset;
        d.synDecay = hp.synDecay;
        d.dt = net.dtS;
        d.p = hp.p;
        d.mt = upload<unsigned long long>(reinterpret_cast<const unsigned long long*>(hp.mt.data()),
                                          312);
        d.mtPos = upload<int>(&hp.mtPos, 1);
        if (hp.kind == kCondLif) {
            std::vector<float> v0(n, hp.eLeak);  // engine.cpp:199
            CK(cudaMemcpyAsync(d.v, v0.data(), n * sizeof(float), cudaMemcpyHostToDevice, stream));
            CK(cudaStreamSynchronize(stream));
        }
        for (int a = 0; a < 2; ++a)
            if (P.acc[a].mode == ssbk::kAccBuffered)
                P.acc[a].buf = alloc<float>(static_cast<std::size_t>(Wmax + 1) * n);
    }

    // groups
    groupDev.resize(net.groups.size());
    for (std::size_t gi = 0; gi < net.groups.size(); ++gi) {
        const auto& g = net.groups[gi];
        auto& G = groupDev[gi];
        const auto& pre = pops[g.pre];
        const auto& post = pops[g.post];
        G.dense = g.dense ? 1 : 0;
        G.nPost = g.nPost;
        G.preOffset = g.preOffset;
        G.preCount = g.preCount;
        G.preN = pre.n;
        G.preList = pre.dev.list;
        G.preCnt = pre.dev.count;
        if (g.dense) {
            G.W = upload<float>(g.W, static_cast<std::size_t>(g.nPre) * g.nPost);
        } else {
            G.segTile = post.kind == kCondLif ? post.block : 256;
            G.nTiles = (g.nPost + G.segTile - 1) / G.segTile;
            G.g = upload<float>(g.g, static_cast<std::size_t>(g.nnz));
            G.ind = upload<int>(g.ind, static_cast<std::size_t>(g.nnz));
            long long* rs = upload<long long>(
                reinterpret_cast<const long long*>(g.rowStart), static_cast<std::size_t>(g.nPre) + 1);
            int* seg = alloc<int>(static_cast<std::size_t>(g.preCount) * (G.nTiles + 1));
            const long long total = static_cast<long long>(g.preCount) * (G.nTiles + 1);
            if (total > 0) {
                ssbk::crs_segments_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0,
                                            stream>>>(G.ind, rs, g.preCount, G.nTiles, G.segTile,
                                                      seg);
                CK(cudaGetLastError());
            }
            G.seg = seg;
        }
        HostGroup meta;
        meta.name = g.name;
        meta.pre = g.pre;
        meta.post = g.post;
        meta.dense = g.dense;
        meta.preCount = g.preCount;
        meta.nPost = g.nPost;
        groupMeta.push_back(meta);
    }
    for (auto& P : pops)
        for (int a = 0; a < 2; ++a)
            for (int k = 0; k < P.acc[a].ng; ++k) P.acc[a].g[k] = groupDev[P.accGroups[a][k]];

    // raster arena
    raster.nPops = nPops;
    for (int pi = 0; pi < nPops; ++pi) {
        raster.n[pi] = pops[pi].n;
        raster.count[pi] = pops[pi].dev.count;
        raster.list[pi] = pops[pi].dev.list;
    }
    const std::int64_t perWindow = static_cast<std::int64_t>(Wmax) * totalNeurons;
    rasterCap = cfg.rasterCapacity > 0 ? cfg.rasterCapacity
                                       : std::max<std::int64_t>(std::int64_t(1) << 24, 2 * perWindow);
    rasterCap = std::max(rasterCap, perWindow);
    raster.arena = alloc<int>(static_cast<std::size_t>(rasterCap));
    raster.cursor = alloc<long long>(2);
    raster.countsAll = alloc<int>(static_cast<std::size_t>(std::max<std::int64_t>(stepsTotal, 1)) *
                                  nPops);
    raster.stepCounter = alloc<long long>(1);
    raster.windowCounter = alloc<long long>(1);
    raster.doneCounter = alloc<unsigned>(1);

    // kernels with large dynamic shared tiles
    CK(cudaFuncSetAttribute(ssbk::condlif_window_kernel,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 4));
    CK(cudaFuncSetAttribute(ssbk::sparse_window_kernel,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 4));
    CK(cudaStreamSynchronize(stream));
}

void DeviceEngine::Impl::enqueue_window(int W) {
    for (int pi : order) {
        auto& P = pops[pi];
        if (P.kind == kPoisson) {
            launch("poisson_window:" + P.name, [&] {
                ssbk::poisson_window_kernel<<<1, 320, 0, stream>>>(P.dev, W, P.acc[0].mode,
                                                                   P.acc[1].mode);
            });
            continue;
        }
        for (int a = 0; a < 2; ++a) {
            if (P.acc[a].mode != ssbk::kAccBuffered) continue;
            for (int k = 0; k < P.acc[a].ng; ++k) {
                const auto& G = P.acc[a].g[k];
                const int gi = P.accGroups[a][k];
                float* out = P.acc[a].buf + P.n;  // row w = 1
                if (G.dense) {
                    dim3 grid((G.nPost + 127) / 128, W);
                    launch("dense_window:" + groupMeta[gi].name, [&] {
                        ssbk::dense_window_kernel<<<grid, 128, 0, stream>>>(G, out, P.n, 1,
                                                                            k == 0);
                    });
                } else {
                    dim3 grid(G.nTiles, W);
                    launch("sparse_window:" + groupMeta[gi].name, [&] {
                        ssbk::sparse_window_kernel<<<grid, G.segTile, G.segTile * 4, stream>>>(
                            G, out, P.n, 1, k == 0);
                    });
                }
            }
        }
        const int smem = P.sparseInline ? P.block * 4 : 0;
        launch("condlif_window:" + P.name, [&] {
            ssbk::condlif_window_kernel<<<P.grid, P.block, smem, stream>>>(P.dev, P.acc[0],
                                                                         P.acc[1], W);
        });
        if (P.grid > 1) {
            const int bs = std::min(1024, round_up(P.nwords, 32));
            launch("compact_window:" + P.name, [&] {
                ssbk::compact_window_kernel<<<W, bs, 0, stream>>>(P.dev.bits, P.nwords, P.n,
                                                                  P.dev.list, P.dev.count);
            });
        }
    }
    // accumulators written after every population advanced (cyclic graphs,
    // Poisson targets): inputs of the next step from the last step's spikes
    for (auto& P : pops) {
        for (int a = 0; a < 2; ++a) {
            if (P.acc[a].mode != ssbk::kAccDeliver) continue;
            float* out = a == 0 ? P.dev.excIn : P.dev.inhIn;
            for (int k = 0; k < P.acc[a].ng; ++k) {
                const auto& G = P.acc[a].g[k];
                const int gi = P.accGroups[a][k];
                if (G.dense) {
                    dim3 grid((G.nPost + 127) / 128, 1);
                    launch("dense_deliver:" + groupMeta[gi].name, [&] {
                        ssbk::dense_window_kernel<<<grid, 128, 0, stream>>>(G, out, 0, W, k == 0);
                    });
                } else {
                    dim3 grid(G.nTiles, 1);
                    launch("sparse_deliver:" + groupMeta[gi].name, [&] {
                        ssbk::sparse_window_kernel<<<grid, G.segTile, G.segTile * 4, stream>>>(
                            G, out, 0, W, k == 0);
                    });
                }
            }
        }
    }
    const int rb = 128;
    launch("raster_window", [&] {
        ssbk::raster_window_kernel<<<W * raster.nPops, rb, 0, stream>>>(raster, W);
    });
}

void DeviceEngine::Impl::flush_raster() {
    CK(cudaStreamSynchronize(stream));
    long long cur = 0;
    const int parity = static_cast<int>(windowsLaunched & 1);
    CK(cudaMemcpy(&cur, raster.cursor + parity, sizeof(long long), cudaMemcpyDeviceToHost));
    if (cur > 0 && !rasterDiscarded) {
        const std::size_t at = hostNeurons.size();
        hostNeurons.resize(at + static_cast<std::size_t>(cur));
        CK(cudaMemcpy(hostNeurons.data() + at, raster.arena, static_cast<std::size_t>(cur) * 4,
                      cudaMemcpyDeviceToHost));
    }
    const long long zero = 0;
    CK(cudaMemcpy(raster.cursor + parity, &zero, sizeof(long long), cudaMemcpyHostToDevice));
    eventBound = 0;
}

void DeviceEngine::Impl::run_window(int W) {
    const std::int64_t add = static_cast<std::int64_t>(W) * totalNeurons;
    if (eventBound + add > rasterCap) flush_raster();
    eventBound += add;
    if (cfg.useGraphs && !cfg.profile) {
        auto it = graphs.find(W);
        if (it == graphs.end()) {
            cudaGraph_t g;
            CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
            enqueue_window(W);
            CK(cudaStreamEndCapture(stream, &g));
            cudaGraphExec_t exec;
            CK(cudaGraphInstantiate(&exec, g, 0));
            CK(cudaGraphDestroy(g));
            it = graphs.emplace(W, exec).first;
        }
        CK(cudaGraphLaunch(it->second, stream));
    } else {
        enqueue_window(W);
        harvest();
    }
    ++windowsLaunched;
    stepsDone += W;
}

// ---------------------------------------------------------------------------

DeviceEngine::DeviceEngine(const HostNet& net, const EngineConfig& cfg)
    : impl_(std::make_unique<Impl>()) {
    auto& m = *impl_;
    m.cfg = cfg;
    if (m.cfg.heavyPreThreshold <= 0) m.cfg.heavyPreThreshold = 1024;
    if (m.cfg.window <= 0) m.cfg.window = 64;
    if (device_count() == 0) throw DeviceError("no CUDA device is visible (the engine has no CPU path)");
    CK(cudaSetDevice(cfg.device));
    m.smCount = device_props(cfg.device).smCount;
    CK(cudaStreamCreateWithFlags(&m.stream, cudaStreamNonBlocking));
    try {
        m.build(net);
    } catch (...) {
        for (void* p : m.allocations) cudaFree(p);
        cudaStreamDestroy(m.stream);
        throw;
    }
}

DeviceEngine::~DeviceEngine() {
    auto& m = *impl_;
    cudaSetDevice(m.cfg.device);
    if (m.stream) cudaStreamSynchronize(m.stream);
    for (auto& [w, g] : m.graphs) cudaGraphExecDestroy(g);
    for (auto& [n, ev] : m.pending) {
        cudaEventDestroy(ev.first);
        cudaEventDestroy(ev.second);
    }
    for (cudaEvent_t e : m.eventPool) cudaEventDestroy(e);
    for (void* p : m.allocations) cudaFree(p);
    if (m.stream) cudaStreamDestroy(m.stream);
}

void DeviceEngine::step(std::int64_t n) {
    auto& m = *impl_;
    CK(cudaSetDevice(m.cfg.device));
    while (n > 0) {
        const int W = static_cast<int>(std::min<std::int64_t>(m.Wmax, n));
        m.run_window(W);
        n -= W;
    }
}

void DeviceEngine::sync() {
    CK(cudaSetDevice(impl_->cfg.device));
    CK(cudaStreamSynchronize(impl_->stream));
}

std::int64_t DeviceEngine::steps_done() const { return impl_->stepsDone; }

namespace {
void* field_ptr(const ssbk::PopDev& d, int field, std::size_t& esz) {
    esz = 4;
    switch (field) {
    case kFieldV: return d.v;
    case kFieldU: return d.u;
    case kFieldGExc: return d.gExc;
    case kFieldGInh: return d.gInh;
    case kFieldExcIn: return d.excIn;
    case kFieldInhIn: return d.inhIn;
    case kFieldNanFlag: esz = 1; return d.nanFlag;
    case kFieldFlagged: esz = 8; return d.flagged;
    }
    return nullptr;
}
}  // namespace

void DeviceEngine::pull(int pop, int field, void* dst, std::int64_t count) {
    auto& m = *impl_;
    CK(cudaSetDevice(m.cfg.device));
    std::size_t esz;
    void* src = field_ptr(m.pops.at(pop).dev, field, esz);
    if (!src) throw synscale::SpecError("unknown state field " + std::to_string(field));
    CK(cudaStreamSynchronize(m.stream));
    CK(cudaMemcpy(dst, src, esz * static_cast<std::size_t>(count), cudaMemcpyDeviceToHost));
}

void DeviceEngine::push(int pop, int field, const void* src, std::int64_t count) {
    auto& m = *impl_;
    CK(cudaSetDevice(m.cfg.device));
    std::size_t esz;
    void* dst = field_ptr(m.pops.at(pop).dev, field, esz);
    if (!dst) throw synscale::SpecError("unknown state field " + std::to_string(field));
    CK(cudaStreamSynchronize(m.stream));
    CK(cudaMemcpy(dst, src, esz * static_cast<std::size_t>(count), cudaMemcpyHostToDevice));
}

void DeviceEngine::collect_raster(std::vector<std::int32_t>& counts,
                                  std::vector<std::int32_t>& neurons) {
    auto& m = *impl_;
    CK(cudaSetDevice(m.cfg.device));
    if (m.rasterDiscarded)
        throw synscale::SpecError("the raster was discarded (ssb_raster_discard)");
    m.flush_raster();
    const std::size_t nc = static_cast<std::size_t>(m.stepsDone) * m.pops.size();
    counts.resize(nc);
    if (nc)
        CK(cudaMemcpy(counts.data(), m.raster.countsAll, nc * 4, cudaMemcpyDeviceToHost));
    neurons = m.hostNeurons;
}

void DeviceEngine::discard_raster() {
    auto& m = *impl_;
    m.flush_raster();
    m.hostNeurons.clear();
    m.hostNeurons.shrink_to_fit();
    m.rasterDiscarded = true;
}

void DeviceEngine::spike_totals(std::vector<std::int64_t>& perPop) {
    auto& m = *impl_;
    CK(cudaSetDevice(m.cfg.device));
    CK(cudaStreamSynchronize(m.stream));
    const std::size_t np = m.pops.size();
    const std::size_t nc = static_cast<std::size_t>(m.stepsDone) * np;
    std::vector<std::int32_t> counts(nc);
    if (nc) CK(cudaMemcpy(counts.data(), m.raster.countsAll, nc * 4, cudaMemcpyDeviceToHost));
    perPop.assign(np, 0);
    for (std::size_t i = 0; i < nc; ++i) perPop[i % np] += counts[i];
}

void* DeviceEngine::stream() const { return impl_->stream; }
int DeviceEngine::window() const { return impl_->Wmax; }
int DeviceEngine::block_size(int pop) const { return impl_->pops.at(pop).block; }
bool DeviceEngine::step_mode() const { return impl_->stepMode; }
std::int64_t DeviceEngine::device_bytes() const { return impl_->bytes; }

std::vector<KernelStat> DeviceEngine::kernel_stats() {
    auto& m = *impl_;
    m.harvest();
    std::vector<KernelStat> out;
    for (auto& [k, s] : m.stats) out.push_back({s.name, s.launches, s.ms, 0.0});
    return out;
}

void DeviceEngine::reset_kernel_stats() {
    impl_->harvest();
    impl_->stats.clear();
}

}  // namespace ssb
