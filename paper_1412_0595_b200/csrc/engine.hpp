// engine.hpp — internal interface between the host library (C++20) and the
// device engine (CUDA, sm_100a).  No CUDA types appear here so the host
// sources compile with plain g++.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace ssb {

enum PopKind : int { kIzhikevich = 0, kPoisson = 1, kCondLif = 2, kTraubMiles = 3 };

// One population, compiled for the device: constants already cast to the
// storage precision exactly as Simulation's constructor does
// (reference engine.cpp:163-210).
struct HostPop {
    std::string name;
    int kind = kCondLif;
    int n = 0;
    // CondLif constants (fp32, engine.cpp:192-198)
    float tauM = 0, eLeak = 0, eExc = 0, eInh = 0, vThresh = 0, vReset = 0, synDecay = 0;
    // Poisson (engine.cpp:186): p in fp64
    double p = 0.0;
    // Izhikevich per-neuron parameters (fp32) and drives (fp64)
    std::vector<float> a, b, c, d;
    std::vector<double> noise, bias;
    // Traub-Miles (extension): conductances fp32, sub-step length dt/substeps
    float gNa = 0, ENa = 0, gK = 0, EK = 0, gl = 0, El = 0, Cm = 0, mdt = 0;
    int substeps = 0;
    // RNG stream ("<name>/source" or "<name>/noise"): MT19937-64 state
    std::array<std::uint64_t, 312> mt{};
    int mtPos = 312;
    // shard of a population split across ranks: neurons [lo, lo + n) of
    // nGlobal, ranks own chunk neurons each (nGlobal == 0: not split)
    int nGlobal = 0, lo = 0, chunk = 0;
};

// One synapse group after gen_fixed_outdegree, gScale and StorageMode.
struct HostGroup {
    std::string name;
    int pre = 0, post = 0;
    int preOffset = 0, preCount = 0;
    bool inhibitory = false;
    bool dense = false;
    int nPre = 0, nPost = 0;
    int outDegree = 0;
    // non-owning views of the host matrices (kept by the caller)
    const float* W = nullptr;              // dense [nPre*nPost]
    const float* g = nullptr;              // CRS gValues [nnz]
    const std::int32_t* ind = nullptr;     // CRS postInd [nnz]
    const std::int64_t* rowStart = nullptr;  // CRS [nPre+1]
    std::int64_t nnz = 0;
    // extension F2: STDP (fp32 constants; trace decays float(exp(-dt/tau)))
    bool plastic = false;
    float aPlus = 0, aMinus = 0, decPlus = 0, decMinus = 0, wMax = 0;
    // multi-GPU (ShardPlan::rowSplit): this rank holds the rows of its own
    // pre-neuron range [preLo, preLo + nPre) and every post column; the fold
    // continues rank by rank (DeviceEngine, rank pipeline)
    bool rowSplit = false;
    int preLo = 0;
};

struct HostNet {
    std::vector<HostPop> pops;
    std::vector<HostGroup> groups;
    float dtS = 0.f;
    double dtMs = 0.0;
    double durationMs = 0.0;
    std::int64_t steps = 0;
};

struct EngineConfig {
    int device = 0;
    int window = 64;
    int blockSize = 0;
    int blockPolicy = 0;
    bool useGraphs = true;
    int heavyPreThreshold = 1024;
    std::int64_t rasterCapacity = 0;  // 0 = automatic
    bool profile = false;
    bool forceStepMode = false;
    // multi-GPU: this process is rank `rank` of `world` (NCCL communicator
    // from commId, one process per GPU).  virtualWorld > 1 instead runs that
    // many shards inside this engine on one device (exchange by device
    // copies) -- the same kernels, for testing the sharded path on one GPU.
    int rank = 0, world = 1, virtualWorld = 0;
    int shardMinSize = 64;  // CondLif populations at least this large are split
    bool hasCommId = false;
    std::array<unsigned char, 128> commId{};
    int rasterPinnedMB = 0;  // pinned host pool for raster drains (0 = none)
    bool rasterLocal = false;  // split runs: record this rank's neurons only (see the C ABI)
};

// Which populations a world of R ranks splits, and where (host, no CUDA).
// bounds[p] is empty for a whole population, else R+1 offsets: rank r owns
// neurons [bounds[p][r], bounds[p][r+1]).  Split populations are CondLif
// populations of at least max(minSize, R) neurons; ranges are multiples of
// 32 neurons (whole spike-bitmask words) for populations of >= 1024*R
// neurons, of 4 otherwise.  Requires a feed-forward population graph.
struct ShardPlan {
    int world = 1;
    std::vector<std::vector<int>> bounds;
    std::vector<int> chunk;  // bounds[p][r] = min(r * chunk[p], n)
    // rank pipeline: a sink population fed only by heavy dense groups from
    // split populations is owned whole by rank 0 (chunk = n); each rank folds
    // those groups over its own pre rows, continuing the previous rank's
    // partial sums (ascending rows = the reference's order), the last rank
    // hands the result to rank 0 -- no spike exchange for the pre population
    std::vector<char> pipeSink;  // per population
    std::vector<char> rowSplit;  // per group
    bool split(int p) const { return !bounds[p].empty(); }
};
// force: split even a world of one rank (a one-rank NCCL communicator runs
// the whole exchange path; used to test it on one GPU)
ShardPlan plan_shards(const HostNet& net, int world, int minSize, bool force = false,
                      int heavyThreshold = 1024, bool pipeline = true);

// Matrices owned by a rank's local network (column slices).
struct ShardStore {
    std::vector<std::vector<float>> f;
    std::vector<std::vector<std::int32_t>> i32;
    std::vector<std::vector<std::int64_t>> i64;
};
// The local network of one rank: split populations shrink to the rank's
// range (nGlobal / lo set); a group into a split population keeps the post
// columns of that range (dense: row-major [nPre][nLocal]; CRS: entries with
// postInd in range, rebased), rows are untouched -- its pre population's
// spike list is global after the exchange.
HostNet shard_net(const HostNet& net, const ShardPlan& plan, int rank, ShardStore& store);

// NCCL unique id for a new communicator (libnccl loaded on first use).
std::array<unsigned char, 128> comm_unique_id();
// One-rank communicator on `device`: all-gather and sum, plain and inside a
// captured CUDA graph; throws DeviceError on any mismatch or NCCL failure.
void comm_selftest(int device);

struct KernelStat {
    std::string name;
    std::int64_t launches = 0;
    double totalMs = 0.0;
    double bytes = 0.0;
};

enum StateField : int {
    kFieldV = 0, kFieldU, kFieldGExc, kFieldGInh, kFieldExcIn, kFieldInhIn, kFieldNanFlag,
    kFieldFlagged, kFieldM, kFieldH, kFieldN
};

// Thrown for CUDA failures (maps to SSB_ERR_INTERNAL).
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

class DeviceEngine {
public:
    DeviceEngine(const HostNet& net, const EngineConfig& cfg);
    ~DeviceEngine();
    DeviceEngine(const DeviceEngine&) = delete;
    DeviceEngine& operator=(const DeviceEngine&) = delete;

    // Advances n steps (n <= steps remaining; checked by the caller).
    void step(std::int64_t n);
    void sync();
    std::int64_t steps_done() const;

    // State access (count elements; FLAGGED is one int64).
    void pull(int pop, int field, void* dst, std::int64_t count);
    void push(int pop, int field, const void* src, std::int64_t count);

    // Raster: flushes device events to the host store and returns it.
    // counts: [steps_done * nPops] spikes per (step, pop); neurons: ids in
    // (step, pop, neuron) order.
    void collect_raster(std::vector<std::int32_t>& counts, std::vector<std::int32_t>& neurons);
    void discard_raster();
    // Flush of the recorded events to the host store: wait = true returns the
    // events held once everything is on the host; wait = false starts the copy
    // in the background and returns -1.
    std::int64_t drain_raster(bool wait = true);
    void spike_totals(std::vector<std::int64_t>& perPop);
    // spike_totals summed over the ranks of a split run that records local
    // rasters (one all-reduce); otherwise spike_totals.
    void global_spike_totals(std::vector<std::int64_t>& perPop);
    bool raster_discarded() const;
    // A plastic group's current weights (false: the group is static).
    bool pull_weights(int group, float* dst, std::int64_t count);

    // Neurons of population pop held by this process: [lo, lo + n) of
    // nGlobal.  State pull/push of a split population move that local slice
    // (virtual shards: the whole population); FLAGGED is the global sum.
    void shard_range(int pop, int& lo, int& n, int& nGlobal) const;
    int world() const;

    void* stream() const;
    int window() const;
    int block_size(int pop) const;
    int grid_size(int pop) const;
    bool step_mode() const;
    std::int64_t device_bytes() const;
    std::int64_t kernel_launches() const;  // kernels launched by step() so far
    std::vector<KernelStat> kernel_stats();
    void reset_kernel_stats();

    struct Impl;

private:
    std::unique_ptr<Impl> impl_;                 // rank / shard 0
    std::vector<std::unique_ptr<Impl>> shards_;  // virtual shards 1..R-1
    void lockstep(int W);
};

// Standalone kernels over caller host arrays (reference propagate /
// detect_nans, engine.cpp:27-80).  Throw DeviceError on CUDA failure.
void device_propagate_dense(const float* w, int nPre, int nPost, const std::int32_t* spikes,
                            std::int64_t nSpikes, float* acc);
void device_propagate_crs(const float* g, const std::int32_t* ind, const std::int64_t* rowStart,
                          int nPre, int nPost, const std::int32_t* spikes, std::int64_t nSpikes,
                          float* acc);
std::int64_t device_detect_nans(int kind, const float* v, const float* u, const float* gExc,
                                const float* gInh, std::uint8_t* flag, std::int64_t n);

// Device-pointer entry points (bench / kernel-level sweeps).
void device_propagate_dense_dev(const float* w, int nPre, int nPost, const std::int32_t* spikes,
                                int nSpikes, float* acc, void* stream);
void device_crs_segments_dev(const std::int32_t* ind, const std::int64_t* rowStart, int nPre,
                             int nPost, int tile, std::int32_t* seg, void* stream);
// Column slices of a CRS matrix (ssb_crs_slices); returns the entries incl.
// padding (rows / vals may be null: sizes only).  Throws SpecError.
std::int64_t crs_slices(const float* g, const std::int32_t* ind, const std::int64_t* rowStart,
                        int nPre, int nPost, std::int64_t* sliceOff, std::int32_t* rows,
                        float* vals, std::int64_t cap);
void device_propagate_crs_sliced_dev(const std::int32_t* rows, const float* vals,
                                     const std::int64_t* sliceOff, int nPre, int nPost,
                                     const std::int32_t* spikes, int nSpikes, float* acc,
                                     void* stream);
void device_propagate_crs_dev(const float* g, const std::int32_t* ind, const std::int32_t* seg,
                              int tile, int nPre, int nPost, const std::int32_t* spikes,
                              int nSpikes, float* acc, void* stream);

int device_count();
struct DeviceProps {
    std::string name;
    int smCount = 0, warpSize = 32, maxThreadsPerSM = 0, maxBlocksPerSM = 0,
        maxThreadsPerBlock = 0, regsPerSM = 0;
    std::int64_t sharedPerSM = 0, sharedPerBlockOptin = 0;
};
DeviceProps device_props(int device);
// numRegs / static shared bytes / max threads of an engine kernel by name.
bool kernel_attributes(const std::string& name, int& regs, int& sharedBytes, int& maxThreads);

}  // namespace ssb
