// engine.cu — DeviceEngine: device memory layout, launch schedule, CUDA
// graphs and raster management of the windowed step engine.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <array>
#include <map>
#include <mutex>
#include <utility>
#include <numeric>
#include <string>
#include <atomic>
#include <thread>
#include <vector>

#include "../engine.hpp"
#include "comm.hpp"
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

// Raises (never lowers) a kernel's dynamic shared-memory limit.  The limit is
// per function and process-wide, so engines built concurrently (sweep
// workers) and groups with different needs go through one lock.
std::mutex gSmemLimitMutex;
void allow_smem(const void* fn, int bytes) {
    std::lock_guard<std::mutex> lk(gSmemLimitMutex);
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, fn));
    if (fa.maxDynamicSharedSizeBytes < bytes)
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

// Tensor map of a dense group's weights [preCount][nPost] (fp32, row-major)
// for TMA row gathers: box = one whole row, out-of-range rows read as +0.
// cuTensorMapEncodeTiled is a driver entry point (the library links cudart
// statically and never links libcuda).  False when unavailable.
bool encode_row_tmap(CUtensorMap* tm, const float* w, int rows, int cols, int boxCols = 0,
                     int boxRows = 1) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
        }
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode || rows < 1 || cols < 4 || cols > 256 || cols % 4) return false;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 4};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(boxCols > 0 ? boxCols : cols),
                               static_cast<cuuint32_t>(boxRows)};
    const cuuint32_t elem[2] = {1, 1};
    return encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(w), dims, strides, box,
                  elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Host store of drained raster events: anonymous mappings with transparent
// huge pages (first touch of tens of MB in 4 KB pages costs more than the
// device-to-host copy itself).
std::shared_ptr<std::int32_t> host_events(std::size_t n) {
    const std::size_t huge = std::size_t(2) << 20;
    const std::size_t bytes = (std::max<std::size_t>(n, 1) * 4 + huge - 1) / huge * huge;
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) {
        return std::shared_ptr<std::int32_t>(new std::int32_t[std::max<std::size_t>(n, 1)],
                                             std::default_delete<std::int32_t[]>());
    }
    madvise(p, bytes, MADV_HUGEPAGE);
    return std::shared_ptr<std::int32_t>(static_cast<std::int32_t*>(p),
                                         [bytes](std::int32_t* q) { munmap(q, bytes); });
}

// memcpy split over a few host threads (pinned staging -> the host store).
void parallel_copy(void* dst, const void* src, std::size_t bytes) {
    constexpr std::size_t kMin = std::size_t(2) << 20;
    const unsigned nt = static_cast<unsigned>(std::min<std::size_t>(4, bytes / kMin));
    if (nt <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const std::size_t part = (bytes / nt + 63) / 64 * 64;
    std::vector<std::thread> ts;
    for (unsigned t = 1; t < nt; ++t) {
        const std::size_t off = t * part;
        if (off >= bytes) break;
        ts.emplace_back([=] {
            std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off,
                        std::min(part, bytes - off));
        });
    }
    std::memcpy(dst, src, std::min(part, bytes));
    for (auto& t : ts) t.join();
}

// CRS tile pack of an inline sparse group for post tiles of tileN neurons
// (layout in kernels.cuh, GroupDev::tpack).  With words == nullptr only the
// largest tile's size (in 32-bit words, a multiple of 4) is computed.
// perm > 0: columns in the order of the quad kernel with perm neurons per
// thread (ssbk::quad_perm).
std::int64_t tile_pack(const HostGroup& g, int tileN, std::vector<std::uint32_t>* words,
                       std::vector<long long>* off, int perm = 0) {
    const int nwT = tileN / 32;
    const int nTiles = (g.nPost + tileN - 1) / tileN;
    const int rows = g.preCount;
    std::vector<std::int64_t> cur(g.rowStart, g.rowStart + rows);
    std::int64_t maxWords = 0;
    if (off) off->assign(1, 0);
    for (int t = 0; t < nTiles; ++t) {
        const int hiPost = static_cast<int>(std::min<std::int64_t>(
            static_cast<std::int64_t>(t + 1) * tileN, g.nPost));
        std::int64_t nnzTile = 0;
        std::vector<std::int64_t> hi(rows);
        for (int r = 0; r < rows; ++r) {
            std::int64_t h = cur[r];
            const std::int64_t end = g.rowStart[r + 1];
            while (h < end && g.ind[h] < hiPost) ++h;
            hi[r] = h;
            nnzTile += h - cur[r];
        }
        const std::int64_t nw = (2LL * rows * nwT + nnzTile + 3) / 4 * 4;
        maxWords = std::max(maxWords, nw);
        if (words) {
            const std::size_t base = words->size();
            words->resize(base + nw, 0u);
            std::uint32_t* M = words->data() + base;
            std::uint32_t* Pf = M + static_cast<std::size_t>(rows) * nwT;
            float* V = reinterpret_cast<float*>(Pf + static_cast<std::size_t>(rows) * nwT);
            std::uint32_t vi = 0;
            const int tile0 = t * tileN;
            std::vector<std::pair<int, float>> ent;
            for (int r = 0; r < rows; ++r) {
                std::uint32_t* m = M + static_cast<std::size_t>(r) * nwT;
                ent.clear();
                for (std::int64_t q = cur[r]; q < hi[r]; ++q) {
                    int c = g.ind[q] - tile0;
                    if (perm) c = ssbk::quad_perm(c, perm);
                    ent.emplace_back(c, g.g[q]);
                }
                // values in ascending (packed) column order = the mask's bit rank
                if (perm) std::sort(ent.begin(), ent.end(),
                                    [](const auto& a, const auto& b) { return a.first < b.first; });
                for (const auto& [c, x] : ent) {
                    m[c >> 5] |= 1u << (c & 31);
                    std::memcpy(V + vi++, &x, 4);
                }
                std::uint32_t run = vi - static_cast<std::uint32_t>(ent.size());
                for (int k = 0; k < nwT; ++k) {
                    Pf[static_cast<std::size_t>(r) * nwT + k] = run;
                    run += static_cast<std::uint32_t>(__builtin_popcount(m[k]));
                }
            }
            off->push_back(static_cast<long long>(words->size()));
        }
        cur.swap(hi);
    }
    return maxWords;
}

// Largest tile pack (words) staged in shared memory.
constexpr std::int64_t kTilePackMaxWords = 64 * 1024 / 4;

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
    else if (name == "condlif_quad_window")
        e = cudaFuncGetAttributes(&a, ssbk::condlif_quad_window_kernel);
    else if (name == "condlif_pair_window")
        e = cudaFuncGetAttributes(&a, ssbk::condlif_pair_window_kernel);
    else if (name == "izh_window") e = cudaFuncGetAttributes(&a, ssbk::izh_window_kernel);
    else if (name == "hh_window") e = cudaFuncGetAttributes(&a, ssbk::hh_window_kernel);
    else if (name == "gaussian_window") e = cudaFuncGetAttributes(&a, ssbk::gaussian_draw_kernel);
    else if (name == "poisson_window") e = cudaFuncGetAttributes(&a, ssbk::poisson_window_kernel);
    else if (name == "dense_window") e = cudaFuncGetAttributes(&a, ssbk::dense_window_kernel);
    else if (name == "dense_window_warp")
        e = cudaFuncGetAttributes(&a, ssbk::dense_window_warp_kernel);
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

using ChainFn = void (*)(ssbk::GroupDev, float*, long long, int, int, int);
// steps a chain block folds side by side (its stage rows <= 32 floats wide)
constexpr int chain_steps(int nPost) { return nPost <= 8 ? 4 : nPost <= 16 ? 2 : 1; }
template <int... NP>
constexpr std::array<ChainFn, sizeof...(NP)> chain_table(std::integer_sequence<int, NP...>) {
    return {ssbk::dense_window_chain_kernel<4 * (NP + 1), chain_steps(4 * (NP + 1))>...};
}
ChainFn chain_kernel(int nPost) {  // nPost % 4 == 0, <= kChainMaxPost
    static constexpr auto k =
        chain_table(std::make_integer_sequence<int, ssbk::kChainMaxPost / 4>{});
    return k[nPost / 4 - 1];
}
int chain_threads(int nPost) {
    return ssbk::kChainCopiers + 32 * ((nPost * chain_steps(nPost) + 31) / 32);
}

struct DeviceEngine::Impl {
    // window-buffer sets: every window of a graph launch gets its own set of
    // spike lists / bitmasks / buffered inputs, so no window waits for an
    // earlier one's consumers to free a buffer (launches serialise anyway)
    static constexpr int kMaxSets = 48;
    int nSets = 2;
    struct PopRt {
        int kind = 0, n = 0, nwords = 0;
        int block = 0, grid = 0;
        bool sparseInline = false;  // needs a dynamic shared tile
        ssbk::PopDev dev{};             // state + window buffer set 0
        ssbk::AccDev acc[2]{};          // accumulator plans (buffer set 0 views)
        ssbk::PopDev devb[kMaxSets]{};     // per window-buffer set b
        ssbk::AccDev accb[kMaxSets][2]{};  // [b][sign]
        std::vector<int> prePops;       // populations whose spikes of the same window feed it
        std::vector<int> consumers;     // populations reading its spike lists
        ssbk::StageAcc stage[2]{};  // shared-memory staging plan (condlif)
        int smemBytes = 0;          // dynamic shared memory of the population kernel
        int offBits = -1;           // shared copy of the window's spike bits (1-block pops)
        int tileN = 0;              // neurons per block
        int quad = 0;               // CondLif: neurons per thread of the quad kernel (0: tile kernel)
        bool globalUse = false;     // some consumer group reads its global spikes (not row-split)
        int tailGroup = -1;         // plastic group whose post population this is (plastic.cuh)
        float* tailExc = nullptr;   // [2][n] the tail kernel's fold results
        bool pipeSource = false;    // a row-split group reads its local lists
        int chunk = 1;              // steps per phase-A/phase-B chunk
        int offIn = 0;              // shared offset of the phase-A inputs
        std::vector<int> accGroups[2];  // group indices in spec order
        std::string name;
        // split population (multi-GPU): the kernel advances the local range
        // [lo, lo + n) into kdev[b] (local bits, stride nwords = chunk words);
        // the exchange gathers every rank's bits and devb[b] holds the global
        // bits / lists (n = nGlobal) that consumers and the raster read.
        bool sharded = false;
        int nGlobal = 0, lo = 0, shardChunk = 0, nwGlobal = 0;
        ssbk::PopDev kdev[kMaxSets]{};
        uint32_t* gathered[kMaxSets] = {};  // [world][exchange words]
        bool rankCounts = false;            // exchange carries per-step counts (see build)
    };
    struct LaunchStat {
        std::string name;
        std::int64_t launches = 0;
        double ms = 0.0;
    };

    EngineConfig cfg;
    int world = 1;              // ranks (or virtual shards) the network is split over
    bool virtualShard = false;  // one of several shards in this process (exchange by copies)
    bool emulateExchange = false;  // SSB_EMULATE_EXCHANGE diagnostic (see the constructor)
    bool rasterLocal = false;      // split run recording this rank's neurons only
    bool serial = false;        // one stream, no graphs (profiling, virtual shards)
    bool ownsStream = true;
    std::unique_ptr<Comm> comm;  // NCCL, one process per GPU
    // rank pipeline (ShardPlan::pipeSink): per row-split group, this rank's
    // partial sums [Wmax + 1][nPost] per window-buffer set; chain and final
    // hop on communicators of their own (split off comm)
    struct PipeRt {
        int gi = 0, post = 0, a = 0, nPost = 0;
        std::string name;
        float* buf[kMaxSets] = {};
        ssbk::GroupDev dev[kMaxSets]{};
    };
    std::vector<PipeRt> pipes;
    std::unique_ptr<Comm> chainComm, finalComm;
    void enqueue_pipes(int pi, int W, int b, cudaStream_t sg, cudaStream_t sm);
    void pipe_gather(const PipeRt& L, int W, int b, int first, cudaStream_t s);
    char* commScratch = nullptr;  // state gathers of split populations
    std::size_t commScratchBytes = 0;
    char* comm_scratch(std::size_t bytes) {
        if (bytes > commScratchBytes) {
            commScratch = alloc<char>(bytes);
            commScratchBytes = bytes;
        }
        return commScratch;
    }
    int Wmax = 1;
    bool stepMode = false;
    // small recurrent networks: one block runs each window (cyclic.cuh)
    bool cycBlock = false;
    ssbk::CycDev* cycDev[kMaxSets] = {};
    int smCount = 148;
    // SMs the block-size choice leaves to the other populations' kernels,
    // which run concurrently in the window graphs (~10% with several
    // populations; measured: KC at 768 threads / 131 blocks beats 704 / 143)
    int reservedSMs = 0;
    cudaStream_t stream = nullptr;
    std::vector<PopRt> pops;
    std::vector<HostGroup> groupMeta;  // sizes only (arrays cleared)
    // extension F2: plastic groups (step mode), one device view per buffer set
    struct StdpRt {
        int gi = 0, grid = 1, smem = 0;
        bool tail = false;  // run by the post population's tail kernel, not per step
        ssbk::StdpDev dev[kMaxSets]{};
        ssbk::TailDev tdev[kMaxSets]{};
        float* WT = nullptr;  // the tail's transposed weights [nPost][nPre]
        int tailGrid = 1;     // sink_step_kernel blocks
        int tailSmem = 0;
    };
    std::vector<StdpRt> stdp;
    // SSB_SINK_WATCH (diagnostic): a host thread printing the plastic sink's progress
    std::thread watchThread;
    std::atomic<bool> watchStop{false};
    int* watchHost = nullptr;
    std::vector<ssbk::GroupDev> groupDev;
    std::vector<int> order;
    std::vector<void*> allocations;
    std::int64_t bytes = 0;
    std::int64_t totalNeurons = 0;
    std::int64_t stepsTotal = 0;
    std::int64_t stepsDone = 0;
    std::int64_t windowsLaunched = 0;

    // raster: the device arena records each window's spike bitmask rows (a
    // fixed rowWords words per step, kernels.cuh RasterDev), so the host knows
    // its fill exactly and flushes it only when the next launch would not
    // fit; a flush decodes the rows into events on the device (copy stream)
    // and moves them to host memory while the simulation fills the other arena.
    ssbk::RasterDev raster{};
    std::int64_t rasterCap = 0;      // words per arena
    std::int64_t cursorHost = 0;     // words recorded in the active arena
    std::int64_t arenaStep0 = 0;     // first step recorded in the active arena
    std::vector<int> arenaWins;      // window sizes recorded in the active arena
    static constexpr std::size_t kEvStage = std::size_t(1) << 24;  // decoded events per chunk
    std::size_t evStageCap = 0;
    int* evStage = nullptr;          // device: decoded events of one chunk
    long long* rowOffDev = nullptr;  // device: arena offset of each drained step
    long long* evOffDev = nullptr;   // device: event offset of each (step, pop)
    std::int64_t maxArenaSteps = 0;
    cudaEvent_t flushEv = nullptr;       // recorded on the stream when an arena is switched out
    long long* pinnedConst = nullptr;    // pinned {0, 1, 0}: arena selector values, zero cursor
    bool rasterDiscarded = false;
    // Host copy of the raster: drained arenas, in order.  A flush switches the
    // device to the other arena and drains the full one on a copy stream from
    // a helper thread, so the simulation keeps running during the copy.
    std::vector<std::pair<std::shared_ptr<std::int32_t>, std::size_t>> hostChunks;
    int* arenaSelDev = nullptr;
    int arenaSel = 0;
    cudaStream_t copyStream = nullptr;
    static constexpr std::size_t kPinnedInts = std::size_t(1) << 22;  // 16 MB per stage
    std::int32_t* pinned[2] = {nullptr, nullptr};
    // Optional pinned host pool (EngineConfig::rasterPinnedMB): a drain that
    // fits takes whole blocks and copies straight into them (52 GB/s against
    // ~11 GB/s through staging into fresh pageable pages); the blocks come
    // back to the pool when the host chunks holding them are released.
    struct PinnedPool {
        std::mutex mu;
        std::vector<std::int32_t*> free, all;
        ~PinnedPool() {
            for (auto* p : all) cudaFreeHost(p);
        }
    };
    static constexpr std::size_t kPoolBlockInts = std::size_t(1) << 23;  // 32 MB per block
    std::shared_ptr<PinnedPool> pinPool;
    std::thread copier;
    void join_copier() {
        if (copier.joinable()) copier.join();
    }

    std::map<int, cudaGraphExec_t> graphs;

    // profiling
    std::map<std::string, LaunchStat> stats;
    std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::vector<cudaEvent_t> eventPool;

    template <typename T>
    T* alloc(std::size_t count, bool zero = true) {
        void* p = nullptr;
        const std::size_t b = std::max<std::size_t>(count, 1) * sizeof(T);
        CK(cudaMalloc(&p, b));
        if (zero) CK(cudaMemsetAsync(p, 0, b, stream));
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

    std::int64_t kernelLaunches = 0;  // kernels of this engine launched so far
    int enqueued = 0;                 // kernels put on the stream by enqueue_window
    std::map<int, int> kernelsPerWindow;

    // Diagnostic timeline (env SSB_TIMELINE=<file>): no graphs, the normal
    // multi-stream schedule, events around every launch on its own stream;
    // harvest() appends "name start_us end_us" lines (relative to the first
    // launch) to the file.
    std::string timelinePath;
    int prioHigh = 0;          // the device's greatest launch priority
    bool usePdl = false;       // SSB_PDL=1: programmatic launch of consecutive updates
    int chainBlocks = 0;       // SSB_CHAIN_BLOCKS: persistent chain-gather grid (0: a block per step)
    bool usePriority = true;   // SSB_PRIORITY=0 disables the update priority
    std::string tracePath;  // SSB_TRACE: per-block records written at release
    unsigned long long* traceBuf = nullptr;
    cudaEvent_t timelineBase = nullptr;
    cudaStream_t launchStream = nullptr;  // stream of the launches being enqueued
    bool timed() const { return cfg.profile || !timelinePath.empty(); }

    template <typename F>
    void launch(const std::string& name, F&& f) {
        ++enqueued;
        const std::string what = "launch of " + name;
        if (!timed()) {
            f();
            check(cudaGetLastError(), what.c_str());
            return;
        }
        cudaStream_t ls = launchStream && !timelinePath.empty() ? launchStream : stream;
        cudaEvent_t a = take_event(), b = take_event();
        if (!timelinePath.empty() && !timelineBase) {
            CK(cudaEventCreate(&timelineBase));
            CK(cudaEventRecord(timelineBase, ls));
        }
        CK(cudaEventRecord(a, ls));
        f();
        check(cudaGetLastError(), what.c_str());
        CK(cudaEventRecord(b, ls));
        pending.push_back({name, {a, b}});
    }

    void harvest() {
        if (pending.empty()) return;
        CK(cudaDeviceSynchronize());
        FILE* tl = timelinePath.empty() ? nullptr : std::fopen(timelinePath.c_str(), "a");
        for (auto& [name, ev] : pending) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ev.first, ev.second));
            if (tl) {
                float t0 = 0.f;
                CK(cudaEventElapsedTime(&t0, timelineBase, ev.first));
                std::fprintf(tl, "%s %.3f %.3f\n", name.c_str(), t0 * 1e3, (t0 + ms) * 1e3);
            }
            auto& s = stats[name];
            s.name = name;
            s.launches += 1;
            s.ms += ms;
            eventPool.push_back(ev.first);
            eventPool.push_back(ev.second);
        }
        if (tl) std::fclose(tl);
        pending.clear();
    }

    int choose_block(int n, const std::function<std::int64_t(int)>& smemFor,
                     const void* kernelFn) const;
    int plan_stage_quad(const HostNet& net, int pi, int tileN, ssbk::StageAcc out[2]) const;
    int plan_stage(const HostNet& net, int pi, int tileN, ssbk::StageAcc out[2], int& offIn,
                   int& C, int& offBits) const;
    void build(const HostNet& net);
    void enqueue_pop(int pi, int W, int b, cudaStream_t s) { enqueue_pop(pi, W, b, s, s, s); }
    // sg: group kernels filling buffered inputs; sm: the population update;
    // sp: compaction / exchange (the window's lists for consumers)
    void enqueue_pop(int pi, int W, int b, cudaStream_t sg, cudaStream_t sm, cudaStream_t sp);
    void edge(cudaStream_t from, cudaStream_t to) {
        if (from == to) return;
        cudaEvent_t e = capture_event();
        CK(cudaEventRecord(e, from));
        CK(cudaStreamWaitEvent(to, e, 0));
    }
    void assemble_compact(int pi, int W, int b, cudaStream_t s);
    // words a split population's rank sends per window: its local bits, plus
    // its per-step counts when the global lists are assembled per rank slice
    std::size_t exchange_words(const PopRt& P, int W = 0) const {
        return P.rankCounts ? static_cast<std::size_t>(Wmax) * P.nwords + Wmax
                            : static_cast<std::size_t>(W > 0 ? W : Wmax) * P.nwords;
    }
    std::int64_t pre_launch(int W, int M);
    void post_launch(int W, int M, std::int64_t add);
    void enqueue_tail(int W, int b, cudaStream_t s);
    void enqueue_cyclic(int W, int M);
    // the Gaussian transform kernel's blocks for a window of W steps of n neurons
    int gauss_grid(int n, int W) const {
        const long long pairs = (static_cast<long long>(W) * n + 1) / 2;
        return static_cast<int>(std::max<long long>(1, std::min<long long>((pairs + 255) / 256, 4ll * smCount)));
    }
    void enqueue_windows(int W, int M);
    void run_windows(int W, int M);
    void flush_raster(bool wait = false);
    void release();

    // multi-window graphs
    ssbk::RasterDev rasterb[kMaxSets]{};
    std::vector<cudaStream_t> auxStreams;
    std::vector<cudaEvent_t> capEvents;
    std::size_t evUsed = 0;
    int graphWindows = 1;
    // Wide kernels (a grid that fills a large part of the GPU with shared-
    // memory-heavy blocks: KC's update, kc_dn's gather) are chained across
    // streams so they never compete for SMs; narrow ones overlap them freely.
    bool multiStream = false;
    cudaEvent_t lastWide = nullptr;
    cudaEvent_t lastCollective = nullptr;  // the previous NCCL call of this enqueue
    bool is_wide(long long blocks, int smem) const {
        return blocks >= smCount / 4 && smem >= 32 * 1024;
    }
    cudaStream_t lastWideStream = nullptr;
    void before_wide(cudaStream_t s) {
        // same stream: ordered anyway (an event edge would also turn the
        // programmatic launch of the next update into a full dependency)
        if (multiStream && lastWide && lastWideStream != s)
            CK(cudaStreamWaitEvent(s, lastWide, 0));
    }
    void after_wide(cudaStream_t s) {
        if (!multiStream) return;
        lastWide = capture_event();
        lastWideStream = s;
        CK(cudaEventRecord(lastWide, s));
    }
    std::int64_t launchesDone = 0;
    std::map<int, int> kernelsPerLaunch;
    cudaEvent_t capture_event() {
        if (evUsed == capEvents.size()) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            capEvents.push_back(e);
        }
        return capEvents[evUsed++];
    }

    static constexpr int kRowBlock = 128;
    static constexpr int kWarpRingBytes =
        ssbk::kWarpStages * 32 * ssbk::kWarpRowStride * 4 + ssbk::kWarpListCap * 4;
    static int ring_smem() {
        return ssbk::kRingStages * ssbk::kRingRows * kRowBlock * 4 + ssbk::kListSeg * 4;
    }
    // Dense group inputs for window steps [wLo, wLo + nW): spiking rows
    // streamed through shared memory when they are 16-byte multiples (one
    // warp per step with a per-lane cp.async ring; SSB_DENSE_KERNEL=pipe
    // selects the block-per-step ring), plain coalesced gathers otherwise.
    bool usePipe = false;
    // heavy dense groups: the cp.async chain kernel by default; SSB_DENSE_KERNEL=
    // tma (TMA gather4 rows), ldg (rows through registers) or rowstream (the
    // matrix streamed in row order) select the experimental gathers of
    // gather_tma.cuh (all bit-exact; slower at config 3)
    bool useTmaGather = false;
    bool useLdgGather = false;
    std::vector<CUtensorMap> rowTmaps;  // per group (heavy dense groups; see hasRowTmap)
    std::vector<char> hasRowTmap;
    std::vector<CUtensorMap> tileTmaps;  // per group: 256-row x 8-column boxes (row streaming)
    bool useRowStream = false;
    void launch_dense(const ssbk::GroupDev& G, const std::string& gname, const char* tag,
                      float* out, long long stride, int wLo, int nW, int first, cudaStream_t s,
                      const CUtensorMap* tm = nullptr, const CUtensorMap* tileTm = nullptr) {
        if (tileTm && useRowStream) {
            // the matrix streamed once in row order, every step taking its rows
            const dim3 grid((G.nPost + ssbk::kRsCols - 1) / ssbk::kRsCols,
                            (nW + ssbk::kRsThreads - 1) / ssbk::kRsThreads);
            launch(std::string(tag) + gname, [&] {
                ssbk::dense_window_rowstream_kernel<<<grid, ssbk::kRsThreads, ssbk::kRsSmem, s>>>(
                    *tileTm, G, out, stride, wLo, nW, first);
            });
        } else if (tm && useLdgGather) {
            // rows through registers, one warp per window step (gather_tma.cuh)
            const int blocks = (nW + 7) / 8;
            launch(std::string(tag) + gname, [&] {
                ssbk::dense_window_ldg_kernel<<<blocks, 256, 0, s>>>(G, out, stride, wLo, nW, first);
            });
        } else if (tm && useTmaGather) {
            // TMA row gathers, one warp per window step (gather_tma.cuh)
            const int blocks = (nW + ssbk::kTmaWarps - 1) / ssbk::kTmaWarps;
            const int smem = ssbk::tma_smem_bytes(G.nPost);
            launch(std::string(tag) + gname, [&] {
                ssbk::dense_window_tma_kernel<<<blocks, 32 * ssbk::kTmaWarps, smem, s>>>(
                    *tm, G, out, stride, wLo, nW, first);
            });
        } else if (G.nPost % 4 == 0 && G.nPost <= ssbk::kChainMaxPost && !usePipe) {
            const int cw = G.nPost * chain_steps(G.nPost);  // stage row width
            const int smem = ssbk::kChainStages * ssbk::kChainPer * (ssbk::kChainCopiers / (cw / 4)) *
                             cw * 4;
            launch(std::string(tag) + gname, [&] {
                const int groups = (nW + chain_steps(G.nPost) - 1) / chain_steps(G.nPost);
                const int gy = chainBlocks > 0 ? std::min(groups, chainBlocks) : groups;
                chain_kernel(G.nPost)<<<dim3(1, gy), chain_threads(G.nPost), smem, s>>>(
                    G, out, stride, wLo, nW, first);
            });
        } else if (G.nPost % 4 == 0 && !usePipe) {
            dim3 grid((G.nPost + ssbk::kWarpSlab - 1) / ssbk::kWarpSlab, nW);
            launch(std::string(tag) + gname, [&] {
                ssbk::dense_window_warp_kernel<<<grid, 32, kWarpRingBytes, s>>>(G, out, stride,
                                                                                 wLo, first);
            });
        } else if (G.nPost % 4 == 0) {
            dim3 grid((G.nPost + kRowBlock - 1) / kRowBlock, nW);
            const bool wide = is_wide(static_cast<long long>(grid.x) * grid.y, ring_smem());
            if (wide) before_wide(s);
            launch(std::string(tag) + gname, [&] {
                ssbk::dense_window_pipe_kernel<<<grid, kRowBlock, ring_smem(), s>>>(
                    G, out, stride, wLo, first);
            });
            if (wide) after_wide(s);
        } else {
            dim3 grid((G.nPost + 127) / 128, nW);
            launch(std::string(tag) + gname, [&] {
                ssbk::dense_window_kernel<<<grid, 128, 0, s>>>(G, out, stride, wLo, first);
            });
        }
    }
};

int DeviceEngine::Impl::choose_block(int n, const std::function<std::int64_t(int)>& smemFor,
                                     const void* kernelFn) const {
    const int single = std::min(1024, round_up(std::max(n, 1), 32));
    if (n <= 256) return single;  // one block; extra threads serve the parallel phases
    // a forced block size applies to the multi-block populations (the ones
    // whose update the occupancy model sizes)
    int regs = 32, shared = 0, maxThreads = 1024;
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kernelFn) == cudaSuccess) {
        regs = fa.numRegs;
        shared = static_cast<int>(fa.sharedSizeBytes);
        maxThreads = fa.maxThreadsPerBlock;
    } else {
        cudaGetLastError();
    }
    if (cfg.blockSize > 0)
        return std::min(round_up(cfg.blockSize, 32), std::min(1024, maxThreads / 32 * 32));
    const synscale::DeviceSpec dev = synscale::device_preset("sm100");
    auto smem = [&](int bs) { return static_cast<std::int64_t>(shared) + smemFor(bs); };
    auto fits = [&](int bs) { return smem(bs) <= 220 * 1024; };
    int best = 0;
    std::int64_t bestWarps = -1, bestLoad = INT64_MAX;
    for (int bs = 32; bs <= std::min(maxThreads, 1024); bs += 32) {
        if (!fits(bs)) continue;
        const auto r = synscale::occupancy(dev, {bs, regs, smem(bs)});
        if (cfg.blockPolicy == 1) {
            // the paper's model as is (reference occupancy.cpp:79-101):
            // highest occupancy, ties to the larger block
            if (r.activeWarps >= bestWarps) {
                bestWarps = r.activeWarps;
                best = bs;
            }
            continue;
        }
        // default: the model's resident blocks per SM, plus the wave
        // quantisation it is blind to — minimise the neurons the busiest SM
        // advances (waves x resident blocks x tile), ties to more warps
        if (r.activeBlocks < 1) continue;
        const std::int64_t grid = (n + bs - 1) / bs;
        // SMs left to this population: the others' kernels run concurrently
        const int sms = std::max(1, smCount - reservedSMs);
        const std::int64_t perWave = static_cast<std::int64_t>(sms) * r.activeBlocks;
        const std::int64_t waves = (grid + perWave - 1) / perWave;
        const std::int64_t resident = std::min<std::int64_t>(r.activeBlocks, (grid + sms - 1) / sms);
        const std::int64_t load = waves * resident * bs;
        if (load < bestLoad || (load == bestLoad && r.activeWarps >= bestWarps)) {
            bestLoad = load;
            bestWarps = r.activeWarps;
            best = bs;
        }
    }
    if (best == 0) best = 32;
    return std::min(best, single);
}

// Shared-memory layout of the quad CondLif kernel (quad.cuh) for tiles of
// tileN = 4 x threads: per inline group its pre lists and either the permuted
// dense tile + a zero row + the first-four-rows table, or the permuted CRS
// tile pack.  Returns the bytes, or -1 when the population does not qualify
// (an accumulator with several inline groups, or a tile that does not fit).
int DeviceEngine::Impl::plan_stage_quad(const HostNet& net, int pi, int tileN,
                                        ssbk::StageAcc out[2]) const {
    const auto& P = pops[pi];
    auto align = [](std::int64_t v, std::int64_t a) { return (v + a - 1) / a * a; };
    const int W = Wmax;
    std::int64_t off = 0;
    for (int a = 0; a < 2; ++a) {
        out[a] = ssbk::StageAcc{};
        const auto& A = P.acc[a];
        if (A.mode == ssbk::kAccNone || A.mode == ssbk::kAccBuffered) continue;
        if (A.mode != ssbk::kAccInline || A.ng != 1) return -1;
        const auto& g = net.groups[P.accGroups[a][0]];
        const int preN = net.pops[g.pre].n;
        auto& S = out[a].g[0];
        // (a window whose lists overflow reads them from global memory; 2048
        // keeps a KC block at ~131 KB so a kc_dn gather block fits beside it)
        S.listCap = static_cast<int>(std::min<std::int64_t>(static_cast<std::int64_t>(W) * preN, 2048));
        S.offCnt = static_cast<int>(off);
        off += (W + 1) * 4;
        S.offList = static_cast<int>(off);
        off += static_cast<std::int64_t>(S.listCap) * 4;
        if (g.dense) {
            S.stageW = 1;
            off = align(off, 16);
            S.offW = static_cast<int>(off);
            off += static_cast<std::int64_t>(g.preCount + 1) * tileN * 4;
            S.offRoff = static_cast<int>(off);
            off += static_cast<std::int64_t>(W + 1) * 4;
            off = align(off, 16);
            S.offRows4 = static_cast<int>(off);  // chunks: at most listCap / 4 + W
            off += (static_cast<std::int64_t>(S.listCap) / 4 + W + 1) * 16;
        } else {
            const std::int64_t tw = tile_pack(g, tileN, nullptr, nullptr);
            if (tw > kTilePackMaxWords) return -1;
            S.tpackWords = static_cast<int>(std::max<std::int64_t>(tw, 4));
            off = align(off, 16);
            S.offT = static_cast<int>(off);
            off += static_cast<std::int64_t>(S.tpackWords) * 4;
        }
    }
    const std::int64_t total = align(off, 16);
    return total <= 200 * 1024 ? static_cast<int>(total) : -1;
}

// Shared-memory layout of a CondLif population kernel for tiles of tileN
// neurons (StageGroup in kernels.cuh): staging regions, the phase-A input
// buffer s_in [2][C][tileN] and, for single-block populations, a copy of the
// window's spike bits.  Dense weight tiles are dropped from the plan (read
// from L2 instead) when the whole plan would not fit.  Returns the bytes.
int DeviceEngine::Impl::plan_stage(const HostNet& net, int pi, int tileN, ssbk::StageAcc out[2],
                                   int& offIn, int& C, int& offBits) const {
    const auto& P = pops[pi];
    auto align = [](std::int64_t v, std::int64_t a) { return (v + a - 1) / a * a; };
    const int W = Wmax;
    const bool single = P.n <= tileN;
    std::int64_t total = 0;
    for (int pass = 0; pass < 3; ++pass) {
        // pass 0: stage dense weight tiles and CRS tile packs; 1: tile packs
        // only; 2: neither (the fold reads them from L2)
        const bool allowW = pass == 0, allowT = pass <= 1;
        std::int64_t off = 0;
        for (int a = 0; a < 2; ++a) {
            out[a] = ssbk::StageAcc{};
            const auto& A = P.acc[a];
            if (A.mode != ssbk::kAccInline) continue;
            for (int k = 0; k < A.ng; ++k) {
                const auto& g = net.groups[P.accGroups[a][k]];
                const int preN = net.pops[g.pre].n;
                auto& S = out[a].g[k];
                S.listCap = static_cast<int>(
                    std::min<std::int64_t>(static_cast<std::int64_t>(W) * preN, 2048));
                S.offCnt = static_cast<int>(off);
                off += (W + 1) * 4;
                S.offList = static_cast<int>(off);
                off += static_cast<std::int64_t>(S.listCap) * 4;
                if (g.dense) {
                    const std::int64_t wbytes = static_cast<std::int64_t>(g.preCount) * tileN * 4;
                    if (allowW && wbytes <= 96 * 1024) {
                        S.stageW = 1;
                        off = align(off, 16);
                        S.offW = static_cast<int>(off);
                        off += wbytes;
                    }
                    continue;
                }
                const std::int64_t tw = allowT ? tile_pack(g, tileN, nullptr, nullptr) : 0;
                if (allowT && tw <= kTilePackMaxWords) {
                    S.tpackWords = static_cast<int>(std::max<std::int64_t>(tw, 4));
                    off = align(off, 16);
                    S.offT = static_cast<int>(off);
                    off += static_cast<std::int64_t>(S.tpackWords) * 4;
                    continue;
                }
                S.offLo = static_cast<int>(off);
                off += static_cast<std::int64_t>(S.listCap) * 4;
                S.offEoff = static_cast<int>(off);
                off += static_cast<std::int64_t>(S.listCap + 1) * 4;
                const double perRow = g.preCount > 0 ? static_cast<double>(g.nnz) /
                                                           g.preCount * tileN /
                                                           std::max(1, g.nPost)
                                                     : 0.0;
                S.entCap = static_cast<int>(std::min<double>(
                    4096.0, std::max(512.0, S.listCap * (1.5 * perRow + 4.0))));
                S.offEidx = static_cast<int>(off);
                off += static_cast<std::int64_t>(S.entCap) * 2;
                off = align(off, 4);
                S.offEg = static_cast<int>(off);
                off += static_cast<std::int64_t>(S.entCap) * 4;
            }
        }
        // phase-A input planes: more steps per chunk = fewer block barriers
        // (env SSB_IN_KB overrides the multi-block budget, for sweeps)
        static const std::int64_t multiKb = [] {
            const char* e = std::getenv("SSB_IN_KB");
            return e ? std::max(16, std::atoi(e)) : 96;
        }();
        const std::int64_t inBudget = std::max<std::int64_t>(
            16 * 1024, std::min<std::int64_t>(single ? 96 * 1024 : multiKb * 1024, 200 * 1024 - off));
        const int planes = P.kind == kIzhikevich ? 3 : 2;  // ex, ih (+ noise)
        C = static_cast<int>(std::clamp<std::int64_t>(inBudget / (planes * tileN * 4LL), 4, 64));
        C = std::min(C, W);
        off = align(off, 16);
        offIn = static_cast<int>(off);
        off += static_cast<std::int64_t>(planes) * C * tileN * 4;
        offBits = -1;
        if (single && P.nwords <= 32) {
            offBits = static_cast<int>(off);
            off += static_cast<std::int64_t>(W) * P.nwords * 4;
        }
        total = align(off, 16);
        if (total <= 200 * 1024) break;
    }
    return static_cast<int>(total);
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
    // a plastic group's weights change after every step: step mode (the
    // window pipeline's lagged post updates would read stale weights)
    bool plastic = false;
    for (const auto& g : net.groups) plastic = plastic || g.plastic;
    // ... unless every plastic group feeds a sink that has no other input: then
    // the rest of the network keeps its windows and two kernels per window
    // run the sink and the learning step by step (plastic.cuh)
    std::vector<int> tailOf(nPops, -1);
    bool tail = plastic && !cyclic && !cfg.forceStepMode &&
                !(std::getenv("SSB_PLASTIC_TAIL") && std::string(std::getenv("SSB_PLASTIC_TAIL")) == "0");
    for (int gi = 0; tail && gi < static_cast<int>(net.groups.size()); ++gi) {
        const auto& g = net.groups[gi];
        if (!g.plastic) continue;
        const int p = g.post;
        // the window's trace table ([W][nPre] floats) within a quarter of the free memory
        std::size_t freeB = 0, totalB = 0;
        CK(cudaMemGetInfo(&freeB, &totalB));
        const std::size_t xdBytes = static_cast<std::size_t>(cfg.window) * g.nPre * 4;
        bool ok = net.pops[p].kind == kCondLif && g.pre != p && g.nPost <= ssbk::kTailMaxPost &&
                  net.pops[p].nGlobal == 0 && net.pops[g.pre].nGlobal == 0 && !g.rowSplit &&
                  cfg.window <= ssbk::kSinkMaxW && xdBytes <= freeB / 4 &&
                  ssbk::kSinkRing * ((net.pops[g.pre].n + 31) / 32) * 4 + ssbk::kSinkLearnBytes +
                          ssbk::kSinkIdxBytes <= 180 * 1024 &&
                  tailOf[p] < 0;
        for (const auto& h : net.groups) {
            if (h.pre == p) ok = false;                // a sink
            if (h.post == p && &h != &g) ok = false;   // fed by the plastic group alone
        }
        if (ok) tailOf[p] = gi;
        else tail = false;
    }
    if (!tail) std::fill(tailOf.begin(), tailOf.end(), -1);
    stepMode = cyclic || cfg.forceStepMode || (plastic && !tail);
    if (stepMode) {
        order.resize(nPops);
        std::iota(order.begin(), order.end(), 0);
    }
    // a small recurrent network keeps windows: one block advances every
    // population step by step (the step-mode plans are built but not launched)
    if (cyclic && !plastic && !cfg.forceStepMode &&
        !(std::getenv("SSB_CYCLIC_BLOCK") && std::string(std::getenv("SSB_CYCLIC_BLOCK")) == "0")) {
        bool ok = nPops <= ssbk::kCycMaxPops &&
                  static_cast<int>(net.groups.size()) <= ssbk::kCycMaxGroups;
        int pad = 0, nAcc = 0, rows = 0;
        for (int pi = 0; pi < nPops; ++pi) {
            const auto& hp = net.pops[pi];
            ok = ok && hp.nGlobal == 0 &&
                 (hp.kind == kIzhikevich || hp.kind == kCondLif || hp.kind == kPoisson);
            pad += (hp.n + 31) / 32 * 32;
            for (int a = 0; a < 2; ++a) {
                bool any = false;
                for (const auto& g : net.groups)
                    any = any || (g.post == pi && (g.inhibitory ? 1 : 0) == a && hp.kind != kPoisson);
                if (any) nAcc += hp.n;
            }
        }
        for (const auto& g : net.groups) {
            rows = std::max(rows, g.preCount);
            ok = ok && !g.rowSplit;
            // the block expands CRS rows to dense ones: each post at most once per row
            for (int r = 0; ok && !g.dense && r < g.preCount; ++r)
                for (std::int64_t k = g.rowStart[r] + 1; k < g.rowStart[r + 1]; ++k)
                    ok = ok && g.ind[k] > g.ind[k - 1];
        }
        cycBlock = ok && pad <= ssbk::kCycMaxN && nAcc <= ssbk::kCycMaxAcc && rows <= ssbk::kCycMaxRows;
    }
    Wmax = stepMode && !cycBlock ? 1 : std::max(1, cfg.window);
    if ((!stepMode || cycBlock) && net.steps > 0)
        Wmax = static_cast<int>(std::min<std::int64_t>(Wmax, net.steps));

    // accumulator plans
    pops.resize(nPops);
    reservedSMs = nPops > 1 && !stepMode ? std::max(4, smCount / 10) : 0;
    if (const char* e = std::getenv("SSB_RESERVED_SMS")) reservedSMs = std::atoi(e);
    for (int gi = 0; gi < static_cast<int>(net.groups.size()); ++gi) {
        const auto& g = net.groups[gi];
        pops[g.post].accGroups[g.inhibitory ? 1 : 0].push_back(gi);
    }
    for (int pi = 0; pi < nPops; ++pi) {
        auto& P = pops[pi];
        const auto& hp = net.pops[pi];
        P.kind = hp.kind;
        P.n = hp.n;
        P.tailGroup = tailOf[pi];
        P.name = hp.name;
        P.sharded = hp.nGlobal > 0;
        P.nGlobal = P.sharded ? hp.nGlobal : hp.n;
        P.lo = hp.lo;
        P.shardChunk = hp.chunk;
        P.nwGlobal = (P.nGlobal + 31) / 32;
        // kernel-side bitmask stride: a split population sends equal slices
        P.nwords = P.sharded ? (hp.chunk + 31) / 32 : (hp.n + 31) / 32;
        // events a window can record: a local raster holds this rank's part
        totalNeurons += !rasterLocal ? P.nGlobal : P.sharded ? P.n : cfg.rank == 0 ? P.nGlobal : 0;
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
        // multi-block CondLif populations whose inputs qualify take the quad
        // kernel (four neurons per thread): threads per block so that the
        // blocks cover the SMs left to this population once (the paper's
        // occupancy model as is, blockPolicy 1, keeps the tile kernel)
        static const bool quadOff = std::getenv("SSB_QUAD") && std::string(std::getenv("SSB_QUAD")) == "0";
        static const int quadNpt = [] {
            const char* e = std::getenv("SSB_QUAD_NPT");
            return e && std::atoi(e) == 4 ? 4 : 2;
        }();
        if (hp.kind == kCondLif && !quadOff && cfg.blockPolicy != 1 && hp.n >= 2048) {
            // a quarter of the SMs stay free for the other populations and the
            // heavy gathers (kc_dn), which otherwise take SMs the next window's
            // update waits for (device trace: 14 reserved SMs -> KC blocks up
            // to 26 us late, window 97 us; 37 -> ~4 us, 91 us)
            static const int quadReserved = [&] {
                const char* e = std::getenv("SSB_RESERVED_SMS");
                return e ? std::atoi(e) : smCount / 4;
            }();
            const int sms = std::max(1, smCount - (nPops > 1 && !stepMode ? quadReserved : 0));
            const int npt = quadNpt;
            int T = cfg.blockSize > 0 ? round_up(cfg.blockSize, 32)
                                      : round_up((hp.n + npt * sms - 1) / (npt * sms), 32);
            T = std::clamp(T, 64, ssbk::kQuadMaxThreads);
            for (; T >= 64 && !P.quad; T -= 32) {
                const int bytes = plan_stage_quad(net, pi, npt * T, P.stage);
                if (bytes < 0) {
                    if (cfg.blockSize > 0) break;
                    continue;
                }
                P.quad = npt;
                P.tileN = npt * T;
                P.block = T;
                P.grid = (hp.n + P.tileN - 1) / P.tileN;
                P.smemBytes = bytes;
            }
        }
        if (P.quad) {
            // planned above
        } else if (hp.kind == kCondLif || hp.kind == kIzhikevich || hp.kind == kTraubMiles) {
            // tile size from the occupancy model (registers of the kernel +
            // this tile's shared-memory plan, 1 KB per-block reservation)
            ssbk::StageAcc tmp[2];
            int tmpIn, tmpC, tmpBits;
            P.tileN = choose_block(
                hp.n,
                [&](int tn) {
                    return plan_stage(net, pi, tn, tmp, tmpIn, tmpC, tmpBits) + 1024;
                },
                hp.kind == kIzhikevich   ? reinterpret_cast<const void*>(&ssbk::izh_window_kernel)
                : hp.kind == kTraubMiles ? reinterpret_cast<const void*>(&ssbk::hh_window_kernel)
                                         : reinterpret_cast<const void*>(&ssbk::condlif_window_kernel));
            P.grid = (hp.n + P.tileN - 1) / P.tileN;
            // a single-block population gets extra threads for the parallel phases
            P.block = P.grid == 1 ? P.tileN * std::max(1, 256 / P.tileN) : P.tileN;
            P.smemBytes = plan_stage(net, pi, P.tileN, P.stage, P.offIn, P.chunk, P.offBits);
            if (P.smemBytes > 220 * 1024)
                throw synscale::SpecError("population '" + hp.name +
                                          "': shared-memory staging plan exceeds the SM budget");
        } else {
            P.block = 320;
            P.grid = 1;
        }
    }

    // windows per graph launch.  Step mode (one-step windows) chains its
    // steps inside a graph too: each step's updates wait on the previous
    // step's deliveries (enqueue_windows), so a graph of many steps replaces a
    // launch per step (SSB_STEP_GRAPH_WINDOWS=1 restores that).
    graphWindows = kMaxSets;
    if (const char* e = std::getenv(stepMode ? "SSB_STEP_GRAPH_WINDOWS" : "SSB_GRAPH_WINDOWS"))
        graphWindows = std::clamp(std::atoi(e), 1, kMaxSets);
    {
        // Every window of a launch has its own window-buffer set (spike lists
        // [W][n] per population, the global ones too for split populations);
        // the sets of one launch may take 25% of the device memory free now
        // (the raster arena is fixed-size bitmask rows, see flush_raster).
        std::size_t freeB = 0, totalB = 0;
        if (cudaMemGetInfo(&freeB, &totalB) != cudaSuccess) {
            cudaGetLastError();
            freeB = 0;
        }
        std::int64_t perSet = 0;
        for (const auto& P : pops)
            perSet += static_cast<std::int64_t>(Wmax) * 4 *
                      (P.n + (P.sharded ? P.nGlobal : 0) + 2 * (P.nwords + P.nwGlobal));
        const std::int64_t budget = static_cast<std::int64_t>(0.25 * static_cast<double>(freeB));
        const std::int64_t fit = budget / std::max<std::int64_t>(perSet, 1);
        graphWindows = static_cast<int>(std::clamp<std::int64_t>(fit, 1, graphWindows));
    }
    nSets = std::clamp(graphWindows, 2, kMaxSets);

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
        d.halves = !(std::getenv("SSB_HALVES") && std::string(std::getenv("SSB_HALVES")) == "0");
        d.vReset = hp.vReset;
        d.synDecay = hp.synDecay;
        d.dt = net.dtS;
        d.p = hp.p;
        // k * 2^-53 < p  <=>  k < p * 2^53 (exact scaling)  <=>  k < ceil(p * 2^53)
        d.pThresh = static_cast<unsigned long long>(std::ceil(std::ldexp(hp.p, 53)));
        d.mt = upload<unsigned long long>(reinterpret_cast<const unsigned long long*>(hp.mt.data()),
                                          312);
        d.mtPos = upload<int>(&hp.mtPos, 1);
        if (hp.kind == kCondLif) {
            std::vector<float> v0(n, hp.eLeak);  // engine.cpp:199
            CK(cudaMemcpyAsync(d.v, v0.data(), n * sizeof(float), cudaMemcpyHostToDevice, stream));
            CK(cudaStreamSynchronize(stream));
        }
        if (hp.kind == kTraubMiles) {
            // extension (F1): GeNN TraubMiles initial state
            std::vector<float> v0(n, -60.0f), m0(n, 0.0529324f), h0(n, 0.3176767f),
                n0(n, 0.5961207f);
            d.hm = alloc<float>(n);
            d.hh = alloc<float>(n);
            d.hn = alloc<float>(n);
            CK(cudaMemcpyAsync(d.v, v0.data(), n * 4, cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(d.hm, m0.data(), n * 4, cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(d.hh, h0.data(), n * 4, cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(d.hn, n0.data(), n * 4, cudaMemcpyHostToDevice, stream));
            d.gNa = hp.gNa;
            d.ENa = hp.ENa;
            d.gK = hp.gK;
            d.EK = hp.EK;
            d.gl = hp.gl;
            d.El = hp.El;
            d.Cm = hp.Cm;
            d.mdt = hp.mdt;
            d.substeps = hp.substeps;
            CK(cudaStreamSynchronize(stream));
        }
        if (hp.kind == kIzhikevich) {
            // engine.cpp:164-183: v = -65, u = b v (fp32); noise stream state
            std::vector<float> v0(n, -65.0f), u0(n);
            for (std::size_t i = 0; i < n; ++i) u0[i] = hp.b[i] * v0[i];
            CK(cudaMemcpyAsync(d.v, v0.data(), n * sizeof(float), cudaMemcpyHostToDevice, stream));
            CK(cudaMemcpyAsync(d.u, u0.data(), n * sizeof(float), cudaMemcpyHostToDevice, stream));
            d.ia = upload<float>(hp.a.data(), n);
            d.ib = upload<float>(hp.b.data(), n);
            d.ic = upload<float>(hp.c.data(), n);
            d.id = upload<float>(hp.d.data(), n);
            d.bias = upload<double>(hp.bias.data(), n);
            d.amp = upload<double>(hp.noise.data(), n);
            d.spare = alloc<double>(1);
            d.hasSpare = alloc<int>(1);
            d.noiseIn = alloc<float>(static_cast<std::size_t>(Wmax) * n);
            // the window's uniforms, then the draw kernel's stash (3 words)
            d.draws = alloc<unsigned long long>(static_cast<std::size_t>(Wmax) * n + 5);
            CK(cudaStreamSynchronize(stream));
        }
        for (int a = 0; a < 2; ++a)
            if (P.acc[a].mode == ssbk::kAccBuffered)
                P.acc[a].buf = alloc<float>(static_cast<std::size_t>(Wmax + 1) * n);
        // further window-buffer sets (the windows of one graph are in flight
        // together): spike lists, bitmasks, counts, buffered inputs
        for (int b = 0; b < nSets; ++b) {
            P.devb[b] = d;
            if (b > 0) {
                P.devb[b].bits = alloc<uint32_t>(static_cast<std::size_t>(Wmax) * P.nwords);
                P.devb[b].list = alloc<int>(static_cast<std::size_t>(Wmax) * n);
                P.devb[b].count = alloc<int>(static_cast<std::size_t>(Wmax));
                // the one-block path draws a window's noise while the block
                // kernel runs the previous window
                if (cycBlock && hp.kind == kIzhikevich)
                    P.devb[b].noiseIn = alloc<float>(static_cast<std::size_t>(Wmax) * n);
            }
            for (int a = 0; a < 2; ++a) {
                P.accb[b][a] = P.acc[a];
                if (b > 0 && P.acc[a].mode == ssbk::kAccBuffered)
                    P.accb[b][a].buf = alloc<float>(static_cast<std::size_t>(Wmax + 1) * n);
            }
            P.kdev[b] = P.devb[b];
        }
        if (P.sharded) {
            const std::size_t ng = static_cast<std::size_t>(P.nGlobal);
            // ranks owning whole words send their per-step counts with their
            // bits (local bits then counts in one buffer), so the global lists
            // are assembled rank slice by rank slice
            P.rankCounts = P.nwGlobal > 32 && P.shardChunk % 32 == 0;
            const std::size_t exw = exchange_words(P);
            for (int b = 0; b < nSets; ++b) {
                if (P.rankCounts) {
                    uint32_t* lb = alloc<uint32_t>(exw);
                    P.kdev[b].bits = lb;
                    P.kdev[b].count = reinterpret_cast<int*>(lb + static_cast<std::size_t>(Wmax) * P.nwords);
                }
                P.gathered[b] = alloc<uint32_t>(static_cast<std::size_t>(world) * exw);
                auto& g = P.devb[b];
                g.n = P.nGlobal;
                g.nwords = P.nwGlobal;
                g.bits = alloc<uint32_t>(static_cast<std::size_t>(Wmax) * P.nwGlobal);
                g.list = alloc<int>(static_cast<std::size_t>(Wmax) * ng);
                g.count = alloc<int>(static_cast<std::size_t>(Wmax));
            }
        }
    }
    for (const auto& g : net.groups) {
        if (stepMode || net.pops[g.post].kind == kPoisson) continue;  // inputs via state
        auto& pp = pops[g.post].prePops;
        if (std::find(pp.begin(), pp.end(), g.pre) == pp.end()) pp.push_back(g.pre);
    }
    for (const auto& g : net.groups) {
        auto& c = pops[g.pre].consumers;
        if (std::find(c.begin(), c.end(), g.post) == c.end()) c.push_back(g.post);
        if (g.rowSplit) pops[g.pre].pipeSource = true;
        else pops[g.pre].globalUse = true;
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
        G.preN = pre.nGlobal;  // the pre population's (global) spike list stride
        G.preList = pre.dev.list;
        G.preCnt = pre.dev.count;
        if (g.dense) {
            G.W = upload<float>(g.W, static_cast<std::size_t>(g.nPre) * g.nPost);
            // TMA row gathers for wide-enough groups (launch_dense)
            if (rowTmaps.empty()) {
                rowTmaps.resize(net.groups.size());
                hasRowTmap.assign(net.groups.size(), 0);
            }
            if (tileTmaps.empty()) tileTmaps.resize(net.groups.size());
            if (g.nPost % 4 == 0 && g.nPost >= 32 && g.nPost <= ssbk::kChainMaxPost)
                hasRowTmap[gi] = encode_row_tmap(&rowTmaps[gi], G.W, g.preCount, g.nPost) &&
                                 encode_row_tmap(&tileTmaps[gi], G.W, g.preCount, g.nPost,
                                                 ssbk::kRsCols, ssbk::kRsBox);
            if (post.quad) {
                // the quad kernel's tile-major, column-permuted copy (quad.cuh)
                const int tn = post.tileN, nt = (g.nPost + tn - 1) / tn, rows = g.preCount + 1;
                std::vector<float> wq(static_cast<std::size_t>(nt) * rows * tn, 0.f);
                for (int t = 0; t < nt; ++t)
                    for (int r = 0; r < g.preCount; ++r) {
                        float* dst = wq.data() + (static_cast<std::size_t>(t) * rows + r) * tn;
                        const float* src = g.W + static_cast<std::size_t>(r) * g.nPost;
                        for (int c = 0; c < tn && t * tn + c < g.nPost; ++c) {
                            const float x = src[t * tn + c];
                            dst[ssbk::quad_perm(c, post.quad)] = x == 0.f ? 0.f : x;
                        }
                    }
                G.Wq = upload<float>(wq.data(), wq.size());
            }
        } else {
            G.segTile = post.kind != kPoisson ? post.tileN : 256;
            G.nTiles = (g.nPost + G.segTile - 1) / G.segTile;
            G.g = upload<float>(g.g, static_cast<std::size_t>(g.nnz));
            G.ind = upload<int>(g.ind, static_cast<std::size_t>(g.nnz));
            // every row holds every post (all-to-all stored sparse): the values
            // are the dense row-major matrix, entry for entry
            G.fullRows = g.nnz == static_cast<std::int64_t>(g.preCount) * g.nPost ? 1 : 0;
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
            // static CRS tile pack when the post kernel's plan stages one
            bool packed = false;
            for (int a = 0; a < 2 && post.kind != kPoisson; ++a)
                for (int k = 0; k < post.acc[a].ng; ++k)
                    if (post.accGroups[a][k] == static_cast<int>(gi) &&
                        post.stage[a].g[k].tpackWords > 0)
                        packed = true;
            if (packed) {
                std::vector<std::uint32_t> words;
                std::vector<long long> offs;
                tile_pack(g, post.tileN, &words, &offs, post.quad);
                G.tpack = upload<std::uint32_t>(words.data(), words.size());
                G.tpackOff = upload<long long>(offs.data(), offs.size());
                G.nwT = post.tileN / 32;
            }
        }
        HostGroup meta;
        meta.name = g.name;
        meta.pre = g.pre;
        meta.post = g.post;
        meta.dense = g.dense;
        meta.preCount = g.preCount;
        meta.nPost = g.nPost;
        meta.rowSplit = g.rowSplit;
        groupMeta.push_back(meta);
        if (g.rowSplit) {  // rank pipeline: partial sums per window-buffer set
            PipeRt L;
            L.gi = static_cast<int>(gi);
            L.post = g.post;
            L.a = g.inhibitory ? 1 : 0;
            L.nPost = g.nPost;
            L.name = g.name;
            for (int b = 0; b < nSets; ++b) {
                L.buf[b] = alloc<float>(static_cast<std::size_t>(Wmax + 1) * g.nPost);
                L.dev[b] = G;
                L.dev[b].preList = pops[g.pre].kdev[b].list;  // this rank's own spikes,
                L.dev[b].preCnt = pops[g.pre].kdev[b].count;  // local indices
                L.dev[b].preN = pops[g.pre].n;
            }
            pipes.push_back(L);
        }
    }
    for (auto& P : pops)
        for (int a = 0; a < 2; ++a)
            for (int k = 0; k < P.acc[a].ng; ++k) {
                const int gi = P.accGroups[a][k];
                P.acc[a].g[k] = groupDev[gi];
                for (int b = 0; b < nSets; ++b) {
                    ssbk::GroupDev G = groupDev[gi];
                    G.preList = pops[net.groups[gi].pre].devb[b].list;
                    G.preCnt = pops[net.groups[gi].pre].devb[b].count;
                    P.accb[b][a].g[k] = G;
                }
            }
    for (std::size_t gi = 0; gi < net.groups.size(); ++gi) {
        const auto& g = net.groups[gi];
        if (!g.plastic) continue;
        StdpRt L;
        L.gi = static_cast<int>(gi);
        L.smem = (g.nPost + (g.nPost + 31) / 32) * 4;
        if (L.smem > 200 * 1024)
            throw synscale::SpecError("plastic group '" + g.name + "': too many post neurons");
        if (L.smem > 48 * 1024)
            allow_smem(reinterpret_cast<const void*>(&ssbk::stdp_update_kernel), L.smem);
        const int nGroups = (g.nPre + 31) / 32;
        L.grid = std::max(1, std::min((nGroups + 7) / 8, 8 * smCount));
        ssbk::StdpDev D{};
        D.W = const_cast<float*>(groupDev[gi].W);
        D.x = alloc<float>(static_cast<std::size_t>(g.nPre));
        D.y = alloc<float>(static_cast<std::size_t>(g.nPost));
        D.preFlag = alloc<uint32_t>(static_cast<std::size_t>(nGroups));
        D.ticket = alloc<unsigned>(1);
        D.nPre = g.nPre;
        D.nPost = g.nPost;
        D.preOffset = g.preOffset;
        D.aPlus = g.aPlus;
        D.aMinus = g.aMinus;
        D.decPlus = g.decPlus;
        D.decMinus = g.decMinus;
        D.wMax = g.wMax;
        for (int b = 0; b < nSets; ++b) {
            L.dev[b] = D;
            L.dev[b].preList = pops[g.pre].devb[b].list;
            L.dev[b].preCnt = pops[g.pre].devb[b].count;
            L.dev[b].postList = pops[g.post].devb[b].list;
            L.dev[b].postCnt = pops[g.post].devb[b].count;
        }
        auto& Q = pops[g.post];
        if (Q.tailGroup == static_cast<int>(gi)) {
            L.tail = true;
            ssbk::TailDev T{};
            T.nSink = (g.nPost + ssbk::kSinkCols - 1) / ssbk::kSinkCols;
            // dynamic shared memory: the ring of L + 2 steps' pre spike bits
            L.tailSmem = (ssbk::kSinkRing * pops[g.pre].nwords + 3) / 4 * 16 + ssbk::kSinkLearnBytes +
                         ssbk::kSinkIdxBytes;
            allow_smem(reinterpret_cast<const void*>(&ssbk::sink_step_kernel), L.tailSmem);
            int perSm = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perSm, ssbk::sink_step_kernel,
                                                             ssbk::kSinkThreads, L.tailSmem));
            // sink blocks plus background blocks, every block co-resident
            int want = std::max(T.nSink + 1, smCount);
            if (const char* e = std::getenv("SSB_TAIL_GRID")) want = std::max(T.nSink + 1, std::atoi(e));
            L.tailGrid = std::min(want, perSm * smCount);
            if (L.tailGrid <= T.nSink)
                throw synscale::SpecError("plastic group '" + g.name + "': too many post neurons");
            // the weights transposed [nPost][nPre] (the potentiation walks post
            // columns); ssb_group_weights transposes back
            std::vector<float> wt(static_cast<std::size_t>(g.nPre) * g.nPost);
            for (int r = 0; r < g.nPre; ++r)
                for (int j = 0; j < g.nPost; ++j)
                    wt[static_cast<std::size_t>(j) * g.nPre + r] = g.W[static_cast<std::size_t>(r) * g.nPost + j];
            L.WT = upload<float>(wt.data(), wt.size());
            T.WT = L.WT;
            T.x = D.x;
            T.y = D.y;
            T.xd = alloc<float>(static_cast<std::size_t>(Wmax) * g.nPre);
            T.sinkDone = alloc<int>(static_cast<std::size_t>(Wmax));
            T.bgDone = alloc<int>(static_cast<std::size_t>(Wmax));
            T.nPre = g.nPre;
            T.nPost = g.nPost;
            T.preOffset = g.preOffset;
            T.aPlus = g.aPlus;
            T.aMinus = g.aMinus;
            T.decPlus = g.decPlus;
            T.decMinus = g.decMinus;
            T.wMax = g.wMax;
            if (const char* e = std::getenv("SSB_TAIL_SKIP")) T.skip = std::atoi(e);
            if (std::getenv("SSB_SINK_WATCH") && !watchHost) {  // diagnostic: each role's progress
                CK(cudaHostAlloc(&watchHost, 4 * (3 * T.nSink + 1) * sizeof(int), cudaHostAllocMapped));
                int* dw = nullptr;
                CK(cudaHostGetDevicePointer(&dw, watchHost, 0));
                CK(cudaMemcpyToSymbol(ssbk::g_watch, &dw, sizeof(dw)));
                const int ns = T.nSink;
                int* hw = watchHost;
                watchThread = std::thread([this, hw, ns] {
                    while (!watchStop.load()) {
                        std::this_thread::sleep_for(std::chrono::milliseconds(2000));
                        volatile int* v = hw;
                        std::fprintf(stderr, "watch: bg %d | chains", v[3 * ns]);
                        for (int b = 0; b < std::min(ns, 4); ++b) std::fprintf(stderr, " %d/%d", v[2 * b], v[2 * b + 1]);
                        std::fprintf(stderr, " | producers");
                        for (int b = 0; b < std::min(ns, 4); ++b) std::fprintf(stderr, " %d", v[2 * ns + b]);
                        std::fprintf(stderr, "\n");
                    }
                });
            }
            for (int b = 0; b < nSets; ++b) {
                L.tdev[b] = T;
                L.tdev[b].P = Q.devb[b];
                L.tdev[b].preList = pops[g.pre].devb[b].list;
                L.tdev[b].preCnt = pops[g.pre].devb[b].count;
                L.tdev[b].preBits = pops[g.pre].devb[b].bits;
                L.tdev[b].preN = pops[g.pre].n;
                L.tdev[b].preWords = pops[g.pre].nwords;
            }
        }
        stdp.push_back(L);
    }

    if (cycBlock) {  // the block kernel's view of the network, per window-buffer set
        ssbk::CycDev C{};
        C.nPops = nPops;
        C.nGroups = static_cast<int>(net.groups.size());
        int base = 0, acc = 0;
        for (int pi = 0; pi < nPops; ++pi) {
            C.pops[pi].base = base;
            base += (pops[pi].n + 31) / 32 * 32;
            for (int a = 0; a < 2; ++a) {
                bool any = false;
                for (const auto& g : net.groups)
                    any = any || (g.post == pi && (g.inhibitory ? 1 : 0) == a &&
                                  pops[pi].kind != kPoisson);
                C.pops[pi].acc[a] = any ? acc : -1;
                if (any) acc += pops[pi].n;
            }
        }
        C.nPad = base;
        C.nAcc = acc;
        for (std::size_t gi = 0; gi < net.groups.size(); ++gi) {
            const auto& g = net.groups[gi];
            auto& Q = C.groups[gi];
            Q.pre = g.pre;
            Q.post = g.post;
            Q.preOffset = g.preOffset;
            Q.preCount = g.preCount;
            Q.nPost = g.nPost;
            Q.accBase = C.pops[g.post].acc[g.inhibitory ? 1 : 0];
            Q.W = groupDev[gi].W;
            if (!g.dense) {
                // CRS as dense rows (absent entries +0.0f): the post-by-post
                // fold over the spiking rows (the block bounds the size)
                std::vector<float> dw(static_cast<std::size_t>(g.preCount) * g.nPost, 0.f);
                for (int r = 0; r < g.preCount; ++r)
                    for (std::int64_t k = g.rowStart[r]; k < g.rowStart[r + 1]; ++k)
                        dw[static_cast<std::size_t>(r) * g.nPost + g.ind[k]] = g.g[k];
                Q.W = upload<float>(dw.data(), dw.size());
            }
        }
        for (int b = 0; b < nSets; ++b) {
            for (int pi = 0; pi < nPops; ++pi) C.pops[pi].P = pops[pi].kdev[b];
            cycDev[b] = upload<ssbk::CycDev>(&C, 1);
        }
        allow_smem(reinterpret_cast<const void*>(&ssbk::cyclic_block_kernel), ssbk::kCycSmem);
    }

    // raster arena
    raster.nPops = nPops;
    // a local raster reads a split population's local lists (indices + lo) and
    // on ranks other than 0 records nothing of the replicated ones
    int* zeroCounts = rasterLocal ? alloc<int>(static_cast<std::size_t>(Wmax)) : nullptr;
    auto raster_src = [&](ssbk::RasterDev& r, int pi, int b) {
        const auto& P = pops[pi];
        r.n[pi] = P.nGlobal;
        r.add[pi] = 0;
        r.bits[pi] = P.devb[b].bits;
        r.nw[pi] = P.sharded ? P.nwGlobal : P.nwords;
        if (!rasterLocal) return;
        if (P.sharded) {
            r.n[pi] = P.n;
            r.add[pi] = P.lo;
            r.bits[pi] = P.kdev[b].bits;
            r.nw[pi] = P.nwords;
        } else if (cfg.rank != 0) {
            r.bits[pi] = nullptr;  // recorded by rank 0
        }
    };
    for (int pi = 0; pi < nPops; ++pi) raster_src(raster, pi, 0);
    raster.rowWords = 0;
    for (int pi = 0; pi < nPops; ++pi) {
        raster.popOff[pi] = raster.rowWords;
        raster.rowWords += raster.nw[pi];
    }
    // arena (words): 2% of the device memory (config 3 on a B200: ~29
    // simulated seconds, so a run's raster stays on the device until it is
    // drained or collected, as in the device-timed bench), at least two
    // launches of windows; rasterCapacity overrides it.  The fill never
    // depends on the activity.
    const std::int64_t perLaunch =
        static_cast<std::int64_t>(Wmax) * graphWindows * std::max(raster.rowWords, 1);
    std::int64_t capDefault = 0;
    {
        std::size_t freeB = 0, totalB = 0;
        if (cudaMemGetInfo(&freeB, &totalB) == cudaSuccess)
            capDefault = static_cast<std::int64_t>(0.02 * static_cast<double>(totalB)) / 4;
        else
            cudaGetLastError();
        // and never more than the whole run needs
        capDefault = std::min<std::int64_t>(
            capDefault, (stepsTotal + static_cast<std::int64_t>(Wmax) * graphWindows) *
                            std::max(raster.rowWords, 1));
    }
    rasterCap = std::max<std::int64_t>(cfg.rasterCapacity > 0 ? cfg.rasterCapacity : capDefault,
                                       2 * perLaunch);
    maxArenaSteps = rasterCap / std::max(raster.rowWords, 1) + 1;
    raster.arena[0] = alloc<int>(static_cast<std::size_t>(rasterCap), false);
    raster.arena[1] = alloc<int>(static_cast<std::size_t>(rasterCap), false);
    evStageCap = kEvStage;
    evStage = alloc<int>(evStageCap, false);
    CK(cudaEventCreateWithFlags(&flushEv, cudaEventDisableTiming));
    CK(cudaMallocHost(&pinnedConst, 4 * sizeof(long long)));
    pinnedConst[0] = 0;
    pinnedConst[1] = 1;
    pinnedConst[2] = 0;
    rowOffDev = alloc<long long>(static_cast<std::size_t>(maxArenaSteps), false);
    evOffDev = alloc<long long>(static_cast<std::size_t>(maxArenaSteps) * nPops, false);
    arenaSelDev = alloc<int>(1);
    raster.arenaSel = arenaSelDev;
    CK(cudaStreamCreateWithFlags(&copyStream, cudaStreamNonBlocking));
    for (auto& p : pinned) CK(cudaMallocHost(&p, kPinnedInts * 4));
    if (cfg.rasterPinnedMB > 0) {
        pinPool = std::make_shared<PinnedPool>();
        const std::size_t blocks = (static_cast<std::size_t>(cfg.rasterPinnedMB) * (1u << 20) +
                                    kPoolBlockInts * 4 - 1) / (kPoolBlockInts * 4);
        for (std::size_t i = 0; i < blocks; ++i) {
            std::int32_t* p = nullptr;
            CK(cudaMallocHost(&p, kPoolBlockInts * 4));
            pinPool->all.push_back(p);
            pinPool->free.push_back(p);
        }
    }
    raster.cursor = alloc<long long>(2);
    raster.countsAll = alloc<int>(static_cast<std::size_t>(std::max<std::int64_t>(stepsTotal, 1)) *
                                  nPops);
    raster.stepCounter = alloc<long long>(1);
    raster.windowCounter = alloc<long long>(1);
    raster.doneCounter = alloc<unsigned>(1);
    for (int b = 0; b < nSets; ++b) {
        rasterb[b] = raster;
        for (int pi = 0; pi < nPops; ++pi) raster_src(rasterb[b], pi, b);
    }
    // capture streams: one per population, one for deliver + raster
    // 3 per population, the raster's, then a second group stream per population
    auxStreams.resize(4 * nPops + 1);
    int leastPrio = 0;
    CK(cudaDeviceGetStreamPriorityRange(&leastPrio, &prioHigh));
    usePriority = !std::getenv("SSB_PRIORITY") || std::string(std::getenv("SSB_PRIORITY")) != "0";
    usePdl = std::getenv("SSB_PDL") && std::string(std::getenv("SSB_PDL")) == "1";
    if (const char* e = std::getenv("SSB_CHAIN_BLOCKS")) chainBlocks = std::atoi(e);
    for (auto& s : auxStreams) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));

    // kernels with large dynamic shared tiles (the limit is per function and
    // process-wide: only ever raised, several engines may share a device)
    int maxSmem = 0;
    for (const auto& P : pops) maxSmem = std::max(maxSmem, P.smemBytes);
    auto allow = allow_smem;
    allow(reinterpret_cast<const void*>(&ssbk::condlif_window_kernel), std::max(maxSmem, 4096));
    allow(reinterpret_cast<const void*>(&ssbk::condlif_quad_window_kernel), std::max(maxSmem, 4096));
    allow(reinterpret_cast<const void*>(&ssbk::condlif_pair_window_kernel), std::max(maxSmem, 4096));
    allow(reinterpret_cast<const void*>(&ssbk::izh_window_kernel), std::max(maxSmem, 4096));
    allow(reinterpret_cast<const void*>(&ssbk::hh_window_kernel), std::max(maxSmem, 4096));
    allow(reinterpret_cast<const void*>(&ssbk::dense_window_warp_kernel), kWarpRingBytes);
    allow(reinterpret_cast<const void*>(&ssbk::dense_window_pipe_kernel), ring_smem());
    for (int np = 4; np <= ssbk::kChainMaxPost; np += 4)
        allow(reinterpret_cast<const void*>(chain_kernel(np)), ssbk::kChainSmem);
    if (const char* e = std::getenv("SSB_DENSE_KERNEL")) {
        const std::string k = e;
        usePipe = k == "pipe";
        useTmaGather = k == "tma";
        useLdgGather = k == "ldg";
        useRowStream = k == "rowstream";
    }
    allow(reinterpret_cast<const void*>(&ssbk::dense_window_rowstream_kernel), ssbk::kRsSmem);
    allow(reinterpret_cast<const void*>(&ssbk::dense_window_tma_kernel),
          ssbk::tma_smem_bytes(ssbk::kChainMaxPost));
    if (const char* e = std::getenv("SSB_TIMELINE")) timelinePath = e;
    if (const char* e = std::getenv("SSB_TRACE")) {  // per-block trace (scripts/trace_kc.py)
        tracePath = e;
        const unsigned cap = 1u << 22;
        traceBuf = alloc<unsigned long long>(4ull * cap);
        unsigned long long* p = traceBuf;
        const unsigned zero = 0;
        CK(cudaMemcpyToSymbol(ssbk::g_trace, &p, sizeof(p)));
        CK(cudaMemcpyToSymbol(ssbk::g_traceN, &zero, sizeof(zero)));
        CK(cudaMemcpyToSymbol(ssbk::g_traceCap, &cap, sizeof(cap)));
    }
    CK(cudaStreamSynchronize(stream));
}

// One population's kernels for one window on stream s, window-buffer set b.
void DeviceEngine::Impl::enqueue_pop(int pi, int W, int b, cudaStream_t sg, cudaStream_t sm,
                                     cudaStream_t sp) {
    auto& P = pops[pi];
    const ssbk::PopDev& D = P.devb[b];
    if (P.kind == kPoisson) {
        launchStream = sm;
        launch("poisson_window:" + P.name, [&] {
            const int bitsBytes = W * P.nwords * 4;
            const int inSmem = bitsBytes <= 32 * 1024;
            ssbk::poisson_window_kernel<<<1, 320, inSmem ? bitsBytes : 0, sm>>>(
                D, W, P.acc[0].mode, P.acc[1].mode, inSmem);
        });
        edge(sm, sp);
        return;
    }
    if (P.tailGroup >= 0) {  // plastic sink: the window's steps in two kernels (plastic.cuh)
        for (const auto& L : stdp) {
            if (L.gi != P.tailGroup) continue;
            launchStream = sm;
            const auto& T = L.tdev[b];
            launch("sink_trace:" + P.name, [&] {
                ssbk::sink_trace_kernel<<<(T.nPre + 255) / 256, 256, 0, sm>>>(T, W);
            });
            launch("sink_step:" + P.name, [&] {
                cudaLaunchConfig_t lc{};
                lc.gridDim = dim3(L.tailGrid);
                lc.blockDim = dim3(ssbk::kSinkThreads);
                lc.dynamicSmemBytes = L.tailSmem;
                lc.stream = sm;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeCooperative;
                at[0].val.cooperative = 1;
                lc.attrs = at;
                lc.numAttrs = 1;
                CK(cudaLaunchKernelEx(&lc, ssbk::sink_step_kernel, T, W));
            });
        }
        edge(sm, sp);
        return;
    }
    if (P.n > 0) {
        launchStream = sg;
        bool groups = false;
        for (int a = 0; a < 2; ++a) {
            const auto& A = P.accb[b][a];
            if (A.mode != ssbk::kAccBuffered) continue;
            for (int k = 0; k < A.ng; ++k) {
                const auto& G = A.g[k];
                const int gi = P.accGroups[a][k];
                if (groupMeta[gi].rowSplit) continue;  // the rank pipeline fills it
                float* out = A.buf + P.n;  // row w = 1
                groups = true;
                if (G.dense || G.fullRows) {
                    ssbk::GroupDev D = G;
                    if (!G.dense) D.W = G.g;  // full CRS rows = dense rows
                    const CUtensorMap* tm =
                        G.dense && gi < static_cast<int>(hasRowTmap.size()) && hasRowTmap[gi]
                            ? &rowTmaps[gi]
                            : nullptr;
                    launch_dense(D, groupMeta[gi].name, "dense_window:", out, P.n, 1, W, k == 0, sg,
                                 tm, tm ? &tileTmaps[gi] : nullptr);
                } else {
                    dim3 grid(G.nTiles, W);
                    launch("sparse_window:" + groupMeta[gi].name, [&] {
                        ssbk::sparse_window_kernel<<<grid, G.segTile, 0, sg>>>(
                            G, out, P.n, 1, k == 0);
                    });
                }
            }
        }
        if (groups) edge(sg, sm);
        launchStream = sm;
        const ssbk::PopDev& K = P.kdev[b];
        const bool wide = is_wide(P.grid, P.smemBytes);
        if (wide) before_wide(sm);
        auto update = [&](const char* tag, auto kernel) {
            launch(tag + P.name, [&] {
                // multi-block updates launch at the highest priority (a launch
                // attribute, kept by the graph's kernel node): when a window's
                // update ends, the next one's blocks take the freed SMs ahead of
                // the gather blocks queued behind them -- otherwise its last
                // blocks start 15-45 us late (device trace, scripts/trace_kc.py)
                cudaLaunchConfig_t lc{};
                lc.gridDim = dim3(P.grid);
                lc.blockDim = dim3(P.block);
                lc.dynamicSmemBytes = P.smemBytes;
                lc.stream = sm;
                cudaLaunchAttribute at[2];
                int na = 0;
                if (P.grid > 1 && usePriority) {
                    at[na].id = cudaLaunchAttributePriority;
                    at[na++].val.priority = prioHigh;
                }
                // programmatic dependent launch: the stream's previous kernel
                // (the previous window's update) lets this grid launch in its
                // last chunk, and this grid waits for it to complete with
                // griddepcontrol.wait before anything else (kernels.cuh
                // window_body) -- whatever the previous kernel is, so the
                // stream order stays a full dependency
                if (P.grid > 1 && usePdl) {
                    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                    at[na++].val.programmaticStreamSerializationAllowed = 1;
                }
                lc.attrs = at;
                lc.numAttrs = na;
                CK(cudaLaunchKernelEx(&lc, kernel, K, P.accb[b][0], P.accb[b][1], P.stage[0],
                                      P.stage[1], W, P.tileN, P.chunk, P.offIn, P.offBits));
            });
        };
        if (P.kind == kIzhikevich) {
            launch("gaussian_draw:" + P.name, [&] {
                ssbk::gaussian_draw_kernel<<<1, 320, 0, sm>>>(K, W);
            });
            launch("gaussian_transform:" + P.name, [&] {
                ssbk::gaussian_transform_kernel<<<gauss_grid(P.n, W), 256, 0, sm>>>(K, W);
            });
            update("izh_window:", ssbk::izh_window_kernel);
        } else if (P.kind == kTraubMiles) {
            update("hh_window:", ssbk::hh_window_kernel);
        } else {
            update("condlif_window:", P.quad == 4   ? ssbk::condlif_quad_window_kernel
                                      : P.quad == 2 ? ssbk::condlif_pair_window_kernel
                                                    : ssbk::condlif_window_kernel);
        }
        // the next wide kernel may start right after the update: compaction
        // (on sp) feeds only this window's consumers
        if (wide) after_wide(sm);
        edge(sm, sp);
        launchStream = sp;
        // (split: the local raster's lists, or the counts the exchange carries)
        if (P.grid > 1 && (!P.sharded || rasterLocal || P.rankCounts || P.pipeSource)) {
            const int bs = std::min(1024, round_up((P.nwords + ssbk::kCompactK - 1) / ssbk::kCompactK, 32));
            launch("compact_window:" + P.name, [&] {
                ssbk::compact_window_kernel<<<W, bs, 0, sp>>>(K.bits, P.nwords, P.n, K.list, K.count);
            });
        }
    } else {
        edge(sm, sp);
    }
    // a split population's global spikes are needed by its consumers and a
    // global raster; a local raster of a sink population (DN) needs none
    if (P.sharded && (!rasterLocal || P.globalUse)) {
        // the window's exchange: every rank's local bits, in rank order
        if (comm) {
            // collectives of one communicator must run in the same order on
            // every rank: chain them (the enqueue order is identical on all
            // ranks; independent streams could otherwise reorder them)
            if (multiStream && lastCollective) CK(cudaStreamWaitEvent(sp, lastCollective, 0));
            comm->allgather_u32(P.kdev[b].bits, P.gathered[b], exchange_words(P, W), sp);
            if (multiStream) {
                lastCollective = capture_event();
                CK(cudaEventRecord(lastCollective, sp));
            }
        } else if (emulateExchange) {
            const std::size_t bytes = exchange_words(P, W) * 4;
            for (int r = 0; r < world; ++r)
                CK(cudaMemcpyAsync(reinterpret_cast<char*>(P.gathered[b]) + r * bytes,
                                   P.kdev[b].bits, bytes, cudaMemcpyDeviceToDevice, sp));
        }
        if (!virtualShard) assemble_compact(pi, W, b, sp);  // virtual: after the shard copies
    }
}

// Global bitmask and ordered spike lists of a split population from the
// gathered local bitmasks (rank order = ascending neuron order).
void DeviceEngine::Impl::assemble_compact(int pi, int W, int b, cudaStream_t s) {
    launchStream = s;
    auto& P = pops[pi];
    const ssbk::PopDev& D = P.devb[b];
    if (P.nwGlobal <= 32) {  // small population: a block per step, a thread per neuron
        launch("assemble_compact:" + P.name, [&] {
            ssbk::assemble_compact_small_kernel<<<W, 32 * P.nwGlobal, 0, s>>>(
                P.gathered[b], W, P.nwords, P.shardChunk, P.nGlobal, P.nwGlobal, D.bits, D.list,
                D.count);
        });
        return;
    }
    if (P.rankCounts) {
        const int bsr = std::min(1024, round_up((P.nwords + ssbk::kCompactK - 1) / ssbk::kCompactK, 32));
        launch("assemble_compact:" + P.name, [&] {
            ssbk::assemble_compact_ranks_kernel<<<dim3(W, world), bsr, 0, s>>>(
                P.gathered[b], Wmax, P.nwords, P.nwGlobal, P.nGlobal, D.bits, D.list, D.count);
        });
        return;
    }
    const int bs = std::min(1024, round_up((P.nwGlobal + ssbk::kCompactK - 1) / ssbk::kCompactK, 32));
    launch("assemble_compact:" + P.name, [&] {
        ssbk::assemble_compact_kernel<<<W, bs, 0, s>>>(P.gathered[b], W, P.nwords, P.shardChunk,
                                                       P.nGlobal, P.nwGlobal, D.bits, D.list,
                                                       D.count);
    });
}

// Accumulators written after every population advanced (cyclic graphs,
// Poisson targets: inputs of the next step from the last step's spikes), then
// the window's raster.
void DeviceEngine::Impl::enqueue_tail(int W, int b, cudaStream_t s) {
    launchStream = s;
    for (auto& P : pops) {
        for (int a = 0; a < 2; ++a) {
            const auto& A = P.accb[b][a];
            if (A.mode != ssbk::kAccDeliver) continue;
            float* out = a == 0 ? P.dev.excIn : P.dev.inhIn;
            for (int k = 0; k < A.ng; ++k) {
                const auto& G = A.g[k];
                const int gi = P.accGroups[a][k];
                if (G.dense) {
                    launch_dense(G, groupMeta[gi].name, "dense_deliver:", out, 0, W, 1, k == 0, s);
                } else {
                    dim3 grid(G.nTiles, 1);
                    launch("sparse_deliver:" + groupMeta[gi].name, [&] {
                        ssbk::sparse_window_kernel<<<grid, G.segTile, 0, s>>>(G, out, 0,
                                                                                         W, k == 0);
                    });
                }
            }
        }
    }
    // extension F2: learning after the step's propagation (step mode, W = 1)
    for (const auto& L : stdp) {
        if (L.tail) continue;
        const auto& D = L.dev[b];
        const std::string& nm = groupMeta[L.gi].name;
        launch("stdp_mark:" + nm, [&] { ssbk::stdp_mark_kernel<<<8, 256, 0, s>>>(D); });
        launch("stdp_update:" + nm,
               [&] { ssbk::stdp_update_kernel<<<L.grid, 256, L.smem, s>>>(D); });
    }
    launch("raster_window", [&] {
        ssbk::raster_window_kernel<<<W * raster.nPops, 256, 0, s>>>(rasterb[b], W);
    });
}

// Rank pipeline (ShardPlan::pipeSink): this rank's fold of a row-split group
// over its own spiking pre rows, into its partial-sum buffer (first: from +0,
// else continuing the partial sums already there).
void DeviceEngine::Impl::pipe_gather(const PipeRt& L, int W, int b, int first, cudaStream_t s) {
    launchStream = s;
    launch_dense(L.dev[b], L.name, "pipe_gather:", L.buf[b] + L.nPost, L.nPost, 1, W, first, s);
}

// One window of the rank pipeline into population pi (real or emulated
// world; virtual shards chain in lockstep): receive the previous rank's
// partial sums, continue them over this rank's rows, pass them on; the last
// rank hands the finished inputs to rank 0, which owns the population.
void DeviceEngine::Impl::enqueue_pipes(int pi, int W, int b, cudaStream_t sg, cudaStream_t sm) {
    const int R = world, rank = cfg.rank;
    for (const auto& L : pipes) {
        if (L.post != pi) continue;
        const std::size_t cnt = static_cast<std::size_t>(W) * L.nPost;
        float* rows = L.buf[b] + L.nPost;
        if (chainComm && rank > 0) chainComm->recv_f32(rows, cnt, rank - 1, sg);
        pipe_gather(L, W, b, rank == 0 ? 1 : 0, sg);
        auto& P = pops[pi];
        float* dst = P.accb[b][L.a].buf + P.n;
        if (chainComm) {
            if (rank < R - 1) chainComm->send_f32(rows, cnt, rank + 1, sg);
            else finalComm->send_f32(rows, cnt, 0, sg);
            if (rank == 0) finalComm->recv_f32(dst, cnt, R - 1, sm);
        } else if (rank == 0 && P.n > 0) {  // emulated exchange (timing): own partials
            CK(cudaMemcpyAsync(dst, rows, cnt * 4, cudaMemcpyDeviceToDevice, sg));
            edge(sg, sm);
        }
    }
}

// M consecutive windows.  Each population's kernels run on its own stream;
// cross-stream edges carry exactly the data dependencies: the pre
// populations' spike lists of the same window, the reuse of a window-buffer
// set two windows later (all readers done), deliver-before-next-window in
// step mode, and raster order.  So PN / LHI of window m+1 overlap KC of
// window m, and kc_dn / DN of window m overlap KC of window m+1.
void DeviceEngine::Impl::enqueue_windows(int W, int M) {
    const int nPops = static_cast<int>(pops.size());
    const bool multi = !cfg.profile && !serial;  // profile / virtual shards: one stream
    // (the diagnostic timeline keeps the multi-stream schedule)
    // streams: 3 per population (groups, update, compaction), then the raster
    const int rs = 3 * nPops;
    auto S = [&](int idx) { return multi ? auxStreams[idx] : stream; };
    evUsed = 0;
    multiStream = multi;
    lastWide = nullptr;
    lastWideStream = nullptr;
    lastCollective = nullptr;
    auto mark = [&](int sidx) -> cudaEvent_t {
        if (!multi) return nullptr;
        cudaEvent_t e = capture_event();
        CK(cudaEventRecord(e, S(sidx)));
        return e;
    };
    auto after = [&](int sidx, cudaEvent_t e) {
        if (multi && e) CK(cudaStreamWaitEvent(S(sidx), e, 0));
    };
    if (cycBlock) {
        multiStream = false;
        enqueue_cyclic(W, M);
        return;
    }
    if (multi) {
        cudaEvent_t fork = capture_event();
        CK(cudaEventRecord(fork, stream));
        for (auto s : auxStreams) CK(cudaStreamWaitEvent(s, fork, 0));
    }
    std::vector<std::vector<cudaEvent_t>> kdone(nPops, std::vector<cudaEvent_t>(M, nullptr));
    std::vector<cudaEvent_t> rdone(M, nullptr);
    for (int m = 0; m < M; ++m) {
        const int b = m % nSets;
        for (int pi : order) {
            auto& P = pops[pi];
            // extra streams only where they carry work (a graph's branches share
            // a few hardware queues: unused parallelism costs false dependencies)
            const int sm = 3 * pi + 1;
            const bool buffered =
                P.acc[0].mode == ssbk::kAccBuffered || P.acc[1].mode == ssbk::kAccBuffered;
            // narrow gathers (a rank's few DN columns) are latency-bound chains
            // with a block per step: consecutive windows' gathers write
            // different buffer sets, so they alternate between two streams
            // and overlap
            const bool narrow = buffered && P.n > 0 && P.n <= ssbk::kChainMaxPost;
            const int sg = !buffered ? sm : (narrow && (m & 1)) ? rs + 1 + pi : 3 * pi;
            const int sp = (P.grid > 1 && P.n > 0) || P.sharded ? 3 * pi + 2 : sm;
            for (int x : {sg, sm}) {
                for (int q : P.prePops) after(x, kdone[q][m]);
                if (m >= nSets) {  // buffer set b was last read by window m-nSets's consumers
                    for (int c : P.consumers) after(x, kdone[c][m - nSets]);
                    after(x, rdone[m - nSets]);
                    after(x, kdone[pi][m - nSets]);
                }
                if (stepMode && m >= 1) after(x, rdone[m - 1]);
            }
            if (!pipes.empty() && !virtualShard) enqueue_pipes(pi, W, b, S(sg), S(sm));
            enqueue_pop(pi, W, b, S(sg), S(sm), S(sp));
            kdone[pi][m] = mark(sp);
        }
        for (int pi = 0; pi < nPops; ++pi) after(rs, kdone[pi][m]);
        enqueue_tail(W, b, S(rs));
        rdone[m] = mark(rs);
    }
    if (multi)
        for (auto s : auxStreams) {
            cudaEvent_t e = capture_event();
            CK(cudaEventRecord(e, s));
            CK(cudaStreamWaitEvent(stream, e, 0));
        }
}

// Small recurrent networks (cycBlock): per window, the Poisson spikes and the
// Izhikevich noise of the window (in the reference's stream order), the block
// kernel over every population, then the raster -- one stream.
void DeviceEngine::Impl::enqueue_cyclic(int W, int M) {
    // the draws run one window ahead on a side stream (window-buffer sets
    // keep them apart); the block kernel and the raster on the main stream
    const bool multi = !cfg.profile && !serial && !auxStreams.empty();
    cudaStream_t gs = multi ? auxStreams[0] : stream;
    if (multi) {
        cudaEvent_t fork = capture_event();
        CK(cudaEventRecord(fork, stream));
        CK(cudaStreamWaitEvent(gs, fork, 0));
    }
    std::vector<cudaEvent_t> done(M, nullptr);
    for (int m = 0; m < M; ++m) {
        const int b = m % nSets;
        if (multi && m >= nSets) CK(cudaStreamWaitEvent(gs, done[m - nSets], 0));
        launchStream = gs;
        for (auto& P : pops) {
            const ssbk::PopDev& K = P.kdev[b];
            if (P.kind == kPoisson && P.n > 0) {
                launch("poisson_window:" + P.name, [&] {
                    const int bitsBytes = W * P.nwords * 4;
                    const int inSmem = bitsBytes <= 32 * 1024;
                    ssbk::poisson_window_kernel<<<1, 320, inSmem ? bitsBytes : 0, gs>>>(
                        K, W, ssbk::kAccNone, ssbk::kAccNone, inSmem);
                });
            } else if (P.kind == kIzhikevich && P.n > 0) {
                launch("gaussian_draw:" + P.name, [&] {
                    ssbk::gaussian_draw_kernel<<<1, 320, 0, gs>>>(K, W);
                });
                launch("gaussian_transform:" + P.name, [&] {
                    ssbk::gaussian_transform_kernel<<<gauss_grid(P.n, W), 256, 0, gs>>>(K, W);
                });
            }
        }
        if (multi) {
            cudaEvent_t e = capture_event();
            CK(cudaEventRecord(e, gs));
            CK(cudaStreamWaitEvent(stream, e, 0));
        }
        launchStream = stream;
        launch("cyclic_block", [&] {
            ssbk::cyclic_block_kernel<<<1, ssbk::kCycThreads, ssbk::kCycSmem, stream>>>(cycDev[b], W);
        });
        launch("raster_window", [&] {
            ssbk::raster_window_kernel<<<W * raster.nPops, 256, 0, stream>>>(rasterb[b], W);
        });
        if (multi) {
            done[m] = capture_event();
            CK(cudaEventRecord(done[m], stream));
        }
    }
    if (multi) {
        cudaEvent_t e = capture_event();
        CK(cudaEventRecord(e, gs));
        CK(cudaStreamWaitEvent(stream, e, 0));
    }
}

// Switches the device to the other arena and drains the full one in the
// background (wait = true: drain synchronously, e.g. to collect results): the
// recorded bitmask rows are decoded into events on the device (copy stream,
// chunks of at most kEvStage events) and copied to host memory -- straight
// into the pinned pool's blocks when enough are free, else through pinned
// staging into huge-page host memory.
void DeviceEngine::Impl::flush_raster(bool wait) {
    // the switch is enqueued on the stream (no host wait): windows enqueued
    // before it fill the full arena, later ones the other; the drain waits
    // for flushEv, recorded right after the switch
    join_copier();  // the other arena must be drained before it is reused
    const int parity = static_cast<int>(windowsLaunched & 1);
    const int full = arenaSel;
    arenaSel ^= 1;
    // pinnedConst holds 0 and 1 as long longs: their low words are the int selector
    CK(cudaMemcpyAsync(arenaSelDev, reinterpret_cast<const int*>(pinnedConst + arenaSel),
                       sizeof(int), cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(raster.cursor + parity, pinnedConst + 2, sizeof(long long),
                       cudaMemcpyHostToDevice, stream));
    CK(cudaEventRecord(flushEv, stream));
    auto wins = std::make_shared<std::vector<int>>();
    wins->swap(arenaWins);
    const std::int64_t step0 = arenaStep0;
    arenaStep0 = stepsDone;
    cursorHost = 0;
    if (wins->empty() || rasterDiscarded) {
        if (wait) CK(cudaEventSynchronize(flushEv));
        return;
    }
    const int nP = raster.nPops;
    const int dev = cfg.device;
    cudaStream_t cs = copyStream;
    cudaEvent_t ready = flushEv;
    std::int32_t* stage[2] = {pinned[0], pinned[1]};
    const uint32_t* arena = reinterpret_cast<const uint32_t*>(raster.arena[full]);
    const ssbk::RasterDev R = raster;
    int* ev = evStage;
    const std::size_t evCap = evStageCap;
    long long* rowD = rowOffDev;
    long long* evD = evOffDev;
    const int* countsDev = raster.countsAll + step0 * nP;
    std::shared_ptr<PinnedPool> pool = pinPool;
    auto* chunks = &hostChunks;
    auto drain = [=] {
        cudaSetDevice(dev);
        cudaEventSynchronize(ready);
        // per-step arena offsets and per-(step, pop) event offsets
        std::int64_t nSteps = 0;
        for (int w : *wins) nSteps += w;
        std::vector<int> cnt(static_cast<std::size_t>(nSteps) * nP);
        cudaMemcpyAsync(cnt.data(), countsDev, cnt.size() * 4, cudaMemcpyDeviceToHost, cs);
        cudaStreamSynchronize(cs);
        std::vector<long long> rowOff(static_cast<std::size_t>(nSteps)), evOff(cnt.size() + 1);
        std::size_t total = 0;
        std::vector<std::int64_t> cuts{0};  // chunks of steps whose events fit the stage
        std::size_t acc = 0;
        for (std::int64_t st = 0; st < nSteps; ++st) {
            rowOff[st] = st * R.rowWords;
            std::size_t e = 0;
            for (int p = 0; p < nP; ++p) {
                evOff[st * nP + p] = static_cast<long long>(total);
                total += static_cast<std::size_t>(cnt[st * nP + p]);
                e += static_cast<std::size_t>(cnt[st * nP + p]);
            }
            if (acc + e > evCap && st > 0) {
                cuts.push_back(st);
                acc = 0;
            }
            acc += e;
        }
        evOff[cnt.size()] = static_cast<long long>(total);
        cuts.push_back(nSteps);
        if (total == 0) return;
        // destination segments (host memory, in event order)
        std::vector<std::pair<std::int32_t*, std::size_t>> segs;
        bool pooled = false;
        if (pool) {
            const std::size_t need = (total + kPoolBlockInts - 1) / kPoolBlockInts;
            std::lock_guard<std::mutex> lk(pool->mu);
            if (pool->free.size() >= need) {
                std::vector<std::int32_t*> blocks(pool->free.end() - need, pool->free.end());
                pool->free.resize(pool->free.size() - need);
                for (std::size_t i = 0; i < blocks.size(); ++i) {
                    const std::size_t len = std::min(kPoolBlockInts, total - i * kPoolBlockInts);
                    chunks->emplace_back(std::shared_ptr<std::int32_t>(blocks[i], [pool](std::int32_t* q) {
                                             std::lock_guard<std::mutex> lk2(pool->mu);
                                             pool->free.push_back(q);
                                         }),
                                         len);
                    segs.emplace_back(blocks[i], len);
                }
                pooled = true;
            }
        }
        if (!pooled) {
            auto chunk = host_events(total);
            segs.emplace_back(chunk.get(), total);
            chunks->emplace_back(std::move(chunk), total);
        }
        cudaMemcpyAsync(rowD, rowOff.data(), rowOff.size() * 8, cudaMemcpyHostToDevice, cs);
        std::vector<long long> rel(cnt.size());
        std::size_t out = 0;  // events written to the destination so far
        for (std::size_t c = 0; c + 1 < cuts.size(); ++c) {
            const std::int64_t a = cuts[c], b = cuts[c + 1];
            if (a == b) continue;
            const long long base = evOff[a * nP];
            const std::size_t n = static_cast<std::size_t>(evOff[b * nP] - base);
            for (std::int64_t i = a * nP; i < b * nP; ++i) rel[i] = evOff[i] - base;
            cudaMemcpyAsync(evD + a * nP, rel.data() + a * nP, (b - a) * nP * 8,
                            cudaMemcpyHostToDevice, cs);
            ssbk::raster_decode_kernel<<<static_cast<unsigned>((b - a) * nP), 256, 0, cs>>>(
                arena, rowD + a, evD + a * nP, R, countsDev + a * nP, ev);
            // device stage -> destination segments
            std::size_t done = 0;
            while (done < n) {
                std::size_t o = out + done, si = 0;
                while (o >= segs[si].second) o -= segs[si++].second;
                const std::size_t len = std::min(n - done, segs[si].second - o);
                if (pooled) {
                    cudaMemcpyAsync(segs[si].first + o, ev + done, len * 4, cudaMemcpyDeviceToHost, cs);
                } else {
                    // pinned staging, host copy of the previous piece meanwhile
                    std::size_t prevOff = 0, prevLen = 0;
                    int k = 0;
                    for (std::size_t p0 = 0; p0 < len || prevLen; p0 += kPinnedInts, k ^= 1) {
                        const std::size_t l = p0 < len ? std::min(kPinnedInts, len - p0) : 0;
                        if (l)
                            cudaMemcpyAsync(stage[k], ev + done + p0, l * 4, cudaMemcpyDeviceToHost, cs);
                        if (prevLen) parallel_copy(segs[si].first + o + prevOff, stage[k ^ 1], prevLen * 4);
                        cudaStreamSynchronize(cs);
                        prevOff = p0;
                        prevLen = l;
                    }
                }
                done += len;
            }
            cudaStreamSynchronize(cs);  // the stage is reused by the next chunk
            out += n;
        }
    };
    if (wait) drain();
    else copier = std::thread(drain);
}

// Raster bookkeeping before a launch of M windows of W steps: flush the
// arena if they would not fit (their size is fixed).  Returns their words.
std::int64_t DeviceEngine::Impl::pre_launch(int W, int M) {
    const std::int64_t add = static_cast<std::int64_t>(W) * M * raster.rowWords;
    if (cursorHost + add > rasterCap) flush_raster();
    return add;
}

void DeviceEngine::Impl::post_launch(int W, int M, std::int64_t add) {
    windowsLaunched += M;
    stepsDone += static_cast<std::int64_t>(W) * M;
    cursorHost += add;
    for (int i = 0; i < M; ++i) arenaWins.push_back(W);
    ++launchesDone;
}

void DeviceEngine::Impl::run_windows(int W, int M) {
    const std::int64_t add = pre_launch(W, M);
    const int key = W * 64 + M;  // M <= kMaxSets < 64
    if (cfg.useGraphs && !timed() && !serial) {
        auto it = graphs.find(key);
        if (it == graphs.end()) {
            cudaGraph_t g;
            CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
            enqueued = 0;
            enqueue_windows(W, M);
            kernelsPerLaunch[key] = enqueued;
            CK(cudaStreamEndCapture(stream, &g));
            cudaGraphExec_t exec;
            CK(cudaGraphInstantiate(&exec, g, 0));
            CK(cudaGraphDestroy(g));
            it = graphs.emplace(key, exec).first;
        }
        CK(cudaGraphLaunch(it->second, stream));
        kernelLaunches += kernelsPerLaunch[key];
    } else {
        enqueued = 0;
        enqueue_windows(W, M);
        kernelLaunches += enqueued;
        harvest();
    }
    post_launch(W, M, add);
}

// ---------------------------------------------------------------------------

DeviceEngine::DeviceEngine(const HostNet& net, const EngineConfig& cfgIn)
    : impl_(std::make_unique<Impl>()) {
    EngineConfig cfg = cfgIn;
    if (cfg.heavyPreThreshold <= 0) cfg.heavyPreThreshold = 1024;
    if (cfg.window <= 0) cfg.window = 64;
    if (device_count() == 0) throw DeviceError("no CUDA device is visible (the engine has no CPU path)");
    CK(cudaSetDevice(cfg.device));
    const bool virt = cfg.virtualWorld > 1;
    const int R = virt ? cfg.virtualWorld : std::max(1, cfg.world);
    // diagnostic (SSB_EMULATE_EXCHANGE=1): one rank of a world of R on its own,
    // the all-gather replaced by R copies of the local bits -- the rank's
    // real per-window work (global spike lists R x as long) with meaningless
    // dynamics, for timing weak scaling on one GPU
    const bool emulate = !virt && R > 1 && !cfg.hasCommId && std::getenv("SSB_EMULATE_EXCHANGE") &&
                         std::string(std::getenv("SSB_EMULATE_EXCHANGE")) == "1";
    if (!virt && R > 1 && !cfg.hasCommId && !emulate)
        throw synscale::SpecError("a multi-GPU run needs a communicator id (ssb_comm_unique_id)");
    if (!virt && R > 1 && (cfg.rank < 0 || cfg.rank >= R))
        throw synscale::SpecError("rank " + std::to_string(cfg.rank) + " outside a world of " +
                                  std::to_string(R));
    // a communicator id with a world of one rank still runs the split path
    // (exchange included) on a one-rank communicator
    const bool split = R > 1 || (!virt && cfg.hasCommId);
    for (const auto& g : net.groups)
        if (g.plastic && split)
            throw synscale::SpecError("plastic group '" + g.name +
                                      "': learning runs on one GPU (split worlds are not supported)");
    const bool pipeline = !(std::getenv("SSB_PIPELINE") && std::string(std::getenv("SSB_PIPELINE")) == "0");
    const ShardPlan plan =
        split ? plan_shards(net, R, cfg.shardMinSize, true,
                            cfg.heavyPreThreshold > 0 ? cfg.heavyPreThreshold : 1024, pipeline)
              : ShardPlan{};
    const int smCount = device_props(cfg.device).smCount;
    auto init = [&](Impl& m, int rank, cudaStream_t shared) {
        m.cfg = cfg;
        m.cfg.rank = rank;
        m.world = R;
        m.smCount = smCount;
        m.virtualShard = virt;
        m.rasterLocal = cfg.rasterLocal && split && !virt;
        m.emulateExchange = emulate;
        if (virt) {  // lockstep across shards on one stream
            m.serial = true;
            m.cfg.useGraphs = false;
        }
        if (shared) {
            m.stream = shared;
            m.ownsStream = false;
        } else {
            CK(cudaStreamCreateWithFlags(&m.stream, cudaStreamNonBlocking));
        }
        try {
            ShardStore store;
            const HostNet local = split ? shard_net(net, plan, rank, store) : HostNet{};
            if (split && !virt && !emulate) m.comm = std::make_unique<Comm>(R, rank, cfg.commId.data());
            m.build(split ? local : net);
            if (m.comm && !m.pipes.empty()) {
                m.chainComm = m.comm->split();
                m.finalComm = m.comm->split();
            }
        } catch (...) {
            m.release();
            throw;
        }
    };
    init(*impl_, virt ? 0 : (R > 1 ? cfg.rank : 0), nullptr);
    if (virt) {
        try {
            for (int r = 1; r < R; ++r) {
                shards_.push_back(std::make_unique<Impl>());
                init(*shards_.back(), r, impl_->stream);
                shards_.back()->rasterDiscarded = true;  // shard 0 keeps the (identical) raster
            }
        } catch (...) {
            for (auto& sh : shards_) sh->release();
            shards_.clear();
            impl_->release();
            throw;
        }
    }
}

// Virtual shards: window W of every shard on the shared stream, population by
// population in topological order; a split population's local bitmasks are
// copied into every shard's gather buffer (the all-gather of a real world)
// before each shard assembles its global lists.
void DeviceEngine::lockstep(int W) {
    std::vector<Impl*> all{impl_.get()};
    for (auto& sh : shards_) all.push_back(sh.get());
    const int R = static_cast<int>(all.size());
    std::vector<std::int64_t> add(R);
    for (int r = 0; r < R; ++r) add[r] = all[r]->pre_launch(W, 1);
    Impl& m0 = *impl_;
    const int b = static_cast<int>(m0.windowsLaunched % m0.nSets);
    for (auto* m : all) {
        m->enqueued = 0;
        m->evUsed = 0;
        m->multiStream = false;
        m->lastWide = nullptr;
    }
    for (int pi : m0.order) {
        // rank pipeline: shard r continues shard r-1's partial sums over its
        // own rows; the last shard's are shard 0's (the owner's) inputs
        for (std::size_t k = 0; k < m0.pipes.size(); ++k) {
            if (m0.pipes[k].post != pi) continue;
            const auto& L0 = m0.pipes[k];
            const std::size_t cnt = static_cast<std::size_t>(W) * L0.nPost;
            for (int r = 0; r < R; ++r) {
                auto& L = all[r]->pipes[k];
                if (r > 0)
                    CK(cudaMemcpyAsync(L.buf[b] + L.nPost, all[r - 1]->pipes[k].buf[b] + L.nPost,
                                       cnt * 4, cudaMemcpyDeviceToDevice, m0.stream));
                all[r]->pipe_gather(L, W, b, r == 0 ? 1 : 0, m0.stream);
            }
            auto& P0 = m0.pops[pi];
            CK(cudaMemcpyAsync(P0.accb[b][L0.a].buf + P0.n, all[R - 1]->pipes[k].buf[b] + L0.nPost,
                               cnt * 4, cudaMemcpyDeviceToDevice, m0.stream));
        }
        for (auto* m : all) m->enqueue_pop(pi, W, b, m0.stream);
        if (!m0.pops[pi].sharded) continue;
        const std::size_t words = m0.exchange_words(m0.pops[pi], W);
        for (int src = 0; src < R; ++src)
            for (int dst = 0; dst < R; ++dst)
                CK(cudaMemcpyAsync(all[dst]->pops[pi].gathered[b] + src * words,
                                   all[src]->pops[pi].kdev[b].bits, words * 4,
                                   cudaMemcpyDeviceToDevice, m0.stream));
        for (auto* m : all) m->assemble_compact(pi, W, b, m0.stream);
    }
    for (auto* m : all) {
        m->enqueue_tail(W, b, m0.stream);
        m->kernelLaunches += m->enqueued;
        m->harvest();
    }
    for (int r = 0; r < R; ++r) all[r]->post_launch(W, 1, add[r]);
}

void DeviceEngine::Impl::release() {
    join_copier();
    if (watchThread.joinable()) {
        watchStop = true;
        watchThread.join();
    }
    if (watchHost) {
        int* nul = nullptr;
        cudaMemcpyToSymbol(ssbk::g_watch, &nul, sizeof(nul));
        cudaFreeHost(watchHost);
        watchHost = nullptr;
    }
    if (traceBuf && !tracePath.empty()) {
        cudaDeviceSynchronize();
        unsigned n = 0;
        cudaMemcpyFromSymbol(&n, ssbk::g_traceN, sizeof(n));
        n = std::min(n, 1u << 22);
        std::vector<unsigned long long> h(4ull * n);
        cudaMemcpy(h.data(), traceBuf, h.size() * 8, cudaMemcpyDeviceToHost);
        if (FILE* f = std::fopen(tracePath.c_str(), "wb")) {
            std::fwrite(h.data(), 8, h.size(), f);
            std::fclose(f);
        }
        unsigned long long* nul = nullptr;
        cudaMemcpyToSymbol(ssbk::g_trace, &nul, sizeof(nul));
        tracePath.clear();
    }
    if (copyStream) cudaStreamDestroy(copyStream), copyStream = nullptr;
    for (auto& p : pinned)
        if (p) cudaFreeHost(p), p = nullptr;
    if (stream) cudaStreamSynchronize(stream);
    for (auto& [w, g] : graphs) cudaGraphExecDestroy(g);
    graphs.clear();
    for (auto& [n, ev] : pending) {
        cudaEventDestroy(ev.first);
        cudaEventDestroy(ev.second);
    }
    pending.clear();
    for (cudaEvent_t e : eventPool) cudaEventDestroy(e);
    eventPool.clear();
    for (cudaEvent_t e : capEvents) cudaEventDestroy(e);
    capEvents.clear();
    if (flushEv) cudaEventDestroy(flushEv), flushEv = nullptr;
    if (pinnedConst) cudaFreeHost(pinnedConst), pinnedConst = nullptr;
    for (void* p : allocations) cudaFree(p);
    allocations.clear();
    for (cudaStream_t s : auxStreams) cudaStreamDestroy(s);
    auxStreams.clear();
    comm.reset();
    if (stream && ownsStream) cudaStreamDestroy(stream);
    stream = nullptr;
}

DeviceEngine::~DeviceEngine() {
    cudaSetDevice(impl_->cfg.device);
    for (auto& sh : shards_) sh->release();  // they borrow shard 0's stream
    impl_->release();
}

void DeviceEngine::step(std::int64_t n) {
    auto& m = *impl_;
    CK(cudaSetDevice(m.cfg.device));
    if (!shards_.empty()) {
        while (n > 0) {
            const int W = static_cast<int>(std::min<std::int64_t>(m.Wmax, n));
            lockstep(W);
            n -= W;
        }
        return;
    }
    const std::int64_t full = static_cast<std::int64_t>(m.Wmax) * m.graphWindows;
    while (n >= full && m.graphWindows > 1) {
        m.run_windows(m.Wmax, m.graphWindows);
        n -= full;
    }
    if (n <= 0) return;
    if (m.graphWindows == 1) {
        while (n > 0) {
            const int W = static_cast<int>(std::min<std::int64_t>(m.Wmax, n));
            m.run_windows(W, 1);
            n -= W;
        }
        return;
    }
    // the rest as ceil(n / Wmax) near-equal windows in at most two graph
    // launches (cached like the full ones), so a remainder still overlaps
    // populations across windows instead of running window by window
    const int k = static_cast<int>((n + m.Wmax - 1) / m.Wmax);
    const int w = static_cast<int>(n / k), r = static_cast<int>(n % k);
    if (k - r > 0) m.run_windows(w, k - r);
    if (r > 0) m.run_windows(w + 1, r);
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
    case kFieldM: return d.hm;
    case kFieldH: return d.hh;
    case kFieldN: return d.hn;
    case kFieldFlagged: esz = 8; return d.flagged;
    }
    return nullptr;
}
}  // namespace

// State of a split population is assembled to the whole population on the
// way out and split on the way in, so callers see the unsplit engine: a
// real world all-gathers the chunk-padded local slices over NCCL, virtual
// shards are read one by one.  FLAGGED (the NaN counter) is summed.
namespace {
struct Slice {
    void* ptr;
    std::size_t esz;
};
}  // namespace

void DeviceEngine::pull(int pop, int field, void* dst, std::int64_t count) {
    auto& m = *impl_;
    CK(cudaSetDevice(m.cfg.device));
    std::size_t esz;
    void* src = field_ptr(m.pops.at(pop).dev, field, esz);
    if (!src) throw synscale::SpecError("unknown state field " + std::to_string(field));
    CK(cudaStreamSynchronize(m.stream));
    const auto& P = m.pops.at(pop);
    if (!P.sharded) {
        CK(cudaMemcpy(dst, src, esz * static_cast<std::size_t>(count), cudaMemcpyDeviceToHost));
        return;
    }
    if (field == kFieldFlagged) {
        unsigned long long total = 0, part = 0;
        if (!shards_.empty()) {
            CK(cudaMemcpy(&total, P.dev.flagged, 8, cudaMemcpyDeviceToHost));
            for (auto& sh : shards_) {
                CK(cudaMemcpy(&part, sh->pops.at(pop).dev.flagged, 8, cudaMemcpyDeviceToHost));
                total += part;
            }
        } else {
            auto* tmp = reinterpret_cast<unsigned long long*>(m.comm_scratch(8));
            CK(cudaMemcpyAsync(tmp, P.dev.flagged, 8, cudaMemcpyDeviceToDevice, m.stream));
            m.comm->allreduce_sum_u64(tmp, 1, m.stream);
            CK(cudaStreamSynchronize(m.stream));
            CK(cudaMemcpy(&total, tmp, 8, cudaMemcpyDeviceToHost));
        }
        std::memcpy(dst, &total, 8);
        return;
    }
    const std::int64_t n = std::min<std::int64_t>(count, P.nGlobal);
    char* out = static_cast<char*>(dst);
    if (!shards_.empty()) {
        for (Impl* sh : [&] {
                 std::vector<Impl*> v{impl_.get()};
                 for (auto& x : shards_) v.push_back(x.get());
                 return v;
             }()) {
            const auto& Q = sh->pops.at(pop);
            std::size_t e2;
            void* s2 = field_ptr(Q.dev, field, e2);
            const std::int64_t k = std::max<std::int64_t>(0, std::min<std::int64_t>(Q.n, n - Q.lo));
            if (k > 0)
                CK(cudaMemcpy(out + esz * Q.lo, s2, esz * k, cudaMemcpyDeviceToHost));
        }
        return;
    }
    // one process per GPU: all-gather chunk-padded slices (chunk*esz is a
    // multiple of 4 bytes: chunks are multiples of 4 neurons)
    const std::size_t sliceBytes = esz * static_cast<std::size_t>(P.shardChunk);
    char* send = m.comm_scratch(sliceBytes * (m.world + 1));
    char* recv = send + sliceBytes;
    if (P.n) CK(cudaMemcpyAsync(send, src, esz * P.n, cudaMemcpyDeviceToDevice, m.stream));
    m.comm->allgather_u32(send, recv, sliceBytes / 4, m.stream);
    CK(cudaStreamSynchronize(m.stream));
    CK(cudaMemcpy(out, recv, esz * n, cudaMemcpyDeviceToHost));
}

void DeviceEngine::push(int pop, int field, const void* src, std::int64_t count) {
    auto& m = *impl_;
    CK(cudaSetDevice(m.cfg.device));
    std::size_t esz;
    void* dst = field_ptr(m.pops.at(pop).dev, field, esz);
    if (!dst) throw synscale::SpecError("unknown state field " + std::to_string(field));
    CK(cudaStreamSynchronize(m.stream));
    std::vector<Impl*> all{impl_.get()};
    for (auto& x : shards_) all.push_back(x.get());
    const char* in = static_cast<const char*>(src);
    for (Impl* sh : all) {
        const auto& Q = sh->pops.at(pop);
        std::size_t e2;
        void* d2 = field_ptr(Q.dev, field, e2);
        if (Q.sharded && field == kFieldFlagged) {
            // a split population's NaN counter is a sum over shards: the value
            // goes to shard / rank 0, the others restart from 0
            const bool first = sh == impl_.get() && (shards_.size() > 0 || m.cfg.rank == 0);
            const unsigned long long zero = 0;
            CK(cudaMemcpy(d2, first ? src : &zero, 8, cudaMemcpyHostToDevice));
            continue;
        }
        if (!Q.sharded) {  // whole populations are replicated on every shard
            CK(cudaMemcpy(d2, in, esz * static_cast<std::size_t>(count), cudaMemcpyHostToDevice));
            continue;
        }
        const std::int64_t k = std::max<std::int64_t>(0, std::min<std::int64_t>(Q.n, count - Q.lo));
        if (k > 0) CK(cudaMemcpy(d2, in + esz * Q.lo, esz * k, cudaMemcpyHostToDevice));
    }
}

void DeviceEngine::shard_range(int pop, int& lo, int& n, int& nGlobal) const {
    const auto& P = impl_->pops.at(pop);
    lo = P.sharded ? P.lo : 0;
    n = P.n;
    nGlobal = P.nGlobal;
}

int DeviceEngine::world() const { return impl_->world; }

void DeviceEngine::collect_raster(std::vector<std::int32_t>& counts,
                                  std::vector<std::int32_t>& neurons) {
    auto& m = *impl_;
    CK(cudaSetDevice(m.cfg.device));
    if (m.rasterDiscarded)
        throw synscale::SpecError("the raster was discarded (ssb_raster_discard)");
    m.flush_raster(true);
    m.join_copier();
    const std::size_t nc = static_cast<std::size_t>(m.stepsDone) * m.pops.size();
    counts.resize(nc);
    if (nc)
        CK(cudaMemcpy(counts.data(), m.raster.countsAll, nc * 4, cudaMemcpyDeviceToHost));
    std::size_t total = 0;
    for (const auto& c : m.hostChunks) total += c.second;
    neurons.resize(total);
    std::size_t at = 0;
    for (const auto& c : m.hostChunks) {
        std::copy(c.first.get(), c.first.get() + c.second, neurons.data() + at);
        at += c.second;
    }
}

std::int64_t DeviceEngine::drain_raster(bool wait) {
    auto& m = *impl_;
    CK(cudaSetDevice(m.cfg.device));
    if (!wait) {
        // hand the events recorded so far to the background copier and
        // return: the steps enqueued next overlap the device-to-host copy
        if (!m.rasterDiscarded) m.flush_raster(false);
        return -1;
    }
    if (!m.rasterDiscarded) m.flush_raster(true);
    m.join_copier();
    std::int64_t n = 0;
    for (const auto& c : m.hostChunks) n += static_cast<std::int64_t>(c.second);
    return n;
}

void DeviceEngine::discard_raster() {
    auto& m = *impl_;
    m.flush_raster(true);
    m.join_copier();
    m.hostChunks.clear();
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

void DeviceEngine::global_spike_totals(std::vector<std::int64_t>& perPop) {
    spike_totals(perPop);
    auto& m = *impl_;
    if (!m.rasterLocal || !m.comm || perPop.empty()) return;
    const std::size_t bytes = perPop.size() * 8;
    auto* tmp = reinterpret_cast<unsigned long long*>(m.comm_scratch(bytes));
    CK(cudaMemcpyAsync(tmp, perPop.data(), bytes, cudaMemcpyHostToDevice, m.stream));
    m.comm->allreduce_sum_u64(tmp, perPop.size(), m.stream);
    CK(cudaMemcpyAsync(perPop.data(), tmp, bytes, cudaMemcpyDeviceToHost, m.stream));
    CK(cudaStreamSynchronize(m.stream));
}

bool DeviceEngine::raster_discarded() const { return impl_->rasterDiscarded; }

bool DeviceEngine::pull_weights(int group, float* dst, std::int64_t count) {
    auto& m = *impl_;
    for (const auto& L : m.stdp) {
        if (L.gi != group) continue;
        const auto& g = m.groupMeta[group];
        if (count != static_cast<std::int64_t>(g.preCount) * g.nPost)
            throw synscale::SpecError("wrong buffer size");
        CK(cudaSetDevice(m.cfg.device));
        CK(cudaStreamSynchronize(m.stream));
        if (L.tail) {  // the tail kernel's transposed copy holds the current weights
            std::vector<float> wt(static_cast<std::size_t>(count));
            CK(cudaMemcpy(wt.data(), L.WT, wt.size() * 4, cudaMemcpyDeviceToHost));
            for (int r = 0; r < g.preCount; ++r)
                for (int j = 0; j < g.nPost; ++j)
                    dst[static_cast<std::size_t>(r) * g.nPost + j] =
                        wt[static_cast<std::size_t>(j) * g.preCount + r];
            return true;
        }
        CK(cudaMemcpy(dst, L.dev[0].W, static_cast<std::size_t>(count) * 4, cudaMemcpyDeviceToHost));
        return true;
    }
    return false;
}

void* DeviceEngine::stream() const { return impl_->stream; }
int DeviceEngine::window() const { return impl_->Wmax; }
int DeviceEngine::block_size(int pop) const { return impl_->pops.at(pop).block; }
int DeviceEngine::grid_size(int pop) const { return impl_->pops.at(pop).grid; }
bool DeviceEngine::step_mode() const { return impl_->stepMode; }
std::int64_t DeviceEngine::device_bytes() const { return impl_->bytes; }
std::int64_t DeviceEngine::kernel_launches() const { return impl_->kernelLaunches; }

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
