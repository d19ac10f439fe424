// synscale/synscale.hpp — C++ API of the B200-native engine.
//
// Same namespace, type and function names as the reference's public headers
// (/root/reference/proj/include/synscale/{common,random,matrix,network,
// engine,occupancy}.hpp) so existing callers recompile unchanged; the
// per-topic headers next to this one simply include it.  The simulation
// engine behind `Simulation` runs on the GPU (C ABI: include/synscale_b200.h,
// kernels: paper_1412_0595_b200/csrc/device/).  Host-side pieces (spec
// validation, builders, connectivity generation, the occupancy model) are
// re-implemented here in C++20 and reproduce the reference's RNG consumption
// exactly, because the connectivity they produce is an input of the parity
// contract.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <variant>
#include <vector>

namespace synscale {

// ---- common (reference common.hpp:9-23) -----------------------------------

using scalar = float;  // fp32 state and weights; the device kernels are fp32-only

// User-caused contract violation (bad spec, misuse, out-of-range argument).
// The C ABI maps it to SSB_ERR_SPEC (2); anything else is internal (1).
class SpecError : public std::runtime_error {
public:
    explicit SpecError(const std::string& what) : std::runtime_error(what) {}
};

// ---- random streams (reference random.hpp:11-83) --------------------------

constexpr std::uint64_t fnv1a64(std::string_view text) {
    // NB: the reference's basis (random.hpp:12) is 1469598103934665603, one
    // digit short of the published FNV-1a offset basis; streams depend on it.
    std::uint64_t h = 1469598103934665603ull;
    for (unsigned char ch : text) h = (h ^ ch) * 0x100000001b3ull;
    return h;
}

constexpr std::uint64_t splitmix64(std::uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

inline std::uint64_t derive_seed(std::uint64_t parent, std::string_view label) {
    return splitmix64(splitmix64(parent) ^ fnv1a64(label));
}

// 64-bit Mersenne twister with the parameters of std::mt19937_64.  Written
// out (rather than using the standard class) because the device engine needs
// the raw 312-word state to continue the same stream on the GPU.
class Mt19937_64 {
public:
    static constexpr int kN = 312;
    explicit Mt19937_64(std::uint64_t seed = 5489u) { reseed(seed); }
    void reseed(std::uint64_t seed);
    std::uint64_t operator()();
    const std::array<std::uint64_t, kN>& state() const { return s_; }
    int position() const { return pos_; }

private:
    void regenerate();
    std::array<std::uint64_t, kN> s_{};
    int pos_ = kN;
};

// Seed of the stream RandomStream(globalSeed, entitySeed, label) would use.
inline std::uint64_t stream_seed(std::uint64_t globalSeed, std::uint64_t entitySeed,
                                 std::string_view label) {
    return splitmix64(splitmix64(globalSeed) ^ splitmix64(~entitySeed) ^ fnv1a64(label));
}

class RandomStream {
public:
    RandomStream(std::uint64_t globalSeed, std::uint64_t entitySeed, std::string_view label)
        : mt_(stream_seed(globalSeed, entitySeed, label)) {}

    std::uint64_t next_u64() { return mt_(); }
    double uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + uniform01() * (hi - lo); }
    std::uint32_t below(std::uint32_t n) {
        const unsigned __int128 wide = static_cast<unsigned __int128>(next_u64()) * n;
        return static_cast<std::uint32_t>(wide >> 64);
    }
    double gaussian();
    const Mt19937_64& engine() const { return mt_; }

private:
    Mt19937_64 mt_;
    bool cached_ = false;
    double cache_ = 0.0;
};

// ---- connectivity (reference matrix.hpp:14-81) -----------------------------

struct WeightDist {
    enum class Kind { Constant, Uniform };
    Kind kind = Kind::Constant;
    double lo = 0.0;
    double hi = 0.0;
    double value = 0.0;

    static WeightDist uniform(double lo, double hi);
    static WeightDist constant(double value);
};

struct DenseMatrix {
    std::int32_t nPre = 0;
    std::int32_t nPost = 0;
    std::vector<scalar> weights;  // row-major [nPre][nPost]; 0 = no synapse

    scalar at(std::int32_t i, std::int32_t j) const {
        return weights[static_cast<std::size_t>(i) * static_cast<std::size_t>(nPost) + j];
    }
    std::int64_t nnz() const;
};

struct CrsMatrix {
    std::int32_t nPre = 0;
    std::int32_t nPost = 0;
    std::vector<scalar> gValues;        // GeNN's g
    std::vector<std::int32_t> postInd;  // GeNN's ind; strictly increasing per row
    std::vector<std::int64_t> rowStart; // GeNN's indInG; nPre + 1 entries

    std::int64_t nnz() const { return static_cast<std::int64_t>(gValues.size()); }
};

bool operator==(const DenseMatrix& a, const DenseMatrix& b);
bool operator==(const CrsMatrix& a, const CrsMatrix& b);
void check_crs(const CrsMatrix& m);
void check_dense(const DenseMatrix& m);
DenseMatrix gen_fixed_outdegree(std::int32_t nPre, std::int32_t nPost, std::int32_t k,
                                const WeightDist& dist, int sign, std::uint64_t seed);
CrsMatrix to_sparse(const DenseMatrix& d);
DenseMatrix to_dense(const CrsMatrix& s);
std::uint64_t mem_sparse_elements(std::uint64_t nNZ, std::uint64_t nPostSynN);
std::uint64_t mem_dense_elements(std::uint64_t nPreSynN, std::uint64_t nPostSynN);
DenseMatrix scale(const DenseMatrix& m, double gScale);
CrsMatrix scale(const CrsMatrix& m, double gScale);

// ---- network model (reference network.hpp:12-144) --------------------------

enum class ModelKind { Izhikevich, PoissonSource, CondLif, TraubMiles };
enum class SynapseSign { Excitatory, Inhibitory };
enum class StorageKind { Dense, Sparse };

// Extension F2 (not in the reference): pair-based STDP on a dense
// all-to-all excitatory group.  After step t's propagation, with traces
// decayed once (x *= decPlus, y *= decMinus): a spiking pre row takes
// w -= aMinus * y[j] on every column, a spiking post column takes
// w += aPlus * x[row] on every row, a touched w is clipped to [0, wMax];
// then spiking rows / columns add 1 to their trace.  fp32, no FMA.
struct StdpRule {
    bool enabled = false;
    double aPlus = 0.0, aMinus = 0.0, tauPlusMs = 20.0, tauMinusMs = 20.0, wMax = 0.0;
};

struct IzhikevichParams {
    std::vector<double> a, b, c, d;
    std::vector<double> noiseAmplitude;
    std::vector<double> biasCurrent;
};

struct PoissonParams {
    double rateHz = 0.0;
};

struct CondLifParams {
    double tauMMs = 10.0;
    double eLeakMV = -60.0;
    double vThreshMV = -45.0;
    double vResetMV = -60.0;
    double eExcMV = 0.0;
    double eInhMV = -80.0;
    double tauSynMs = 5.0;
};

// B200 extension (not in the reference): the Traub-Miles
// Hodgkin-Huxley neuron of the paper's mushroom-body KCs (GeNN's TraubMiles:
// Na / K / leak currents, `substeps` explicit-Euler sub-steps of dt/substeps
// per step, spike on the upward crossing of 0 mV) with the same conductance
// synapses as CondLif (decay exp(-dt/tauSyn), reversal eExc / eInh).
struct TraubMilesParams {
    double gNa = 7.15;     // uS
    double ENa = 50.0;     // mV
    double gK = 1.43;
    double EK = -95.0;
    double gl = 0.02672;
    double El = -63.563;
    double C = 0.143;      // nF
    double eExcMV = 0.0;
    double eInhMV = -92.0;
    double tauSynMs = 3.0;
    std::int32_t substeps = 25;
};

struct NeuronPopulation {
    std::string name;
    std::int32_t size = 0;
    ModelKind model = ModelKind::Izhikevich;
    std::uint64_t seed = 0;
    std::variant<IzhikevichParams, PoissonParams, CondLifParams, TraubMilesParams> params;
};

struct SynapseGroupSpec {
    std::string name;
    std::string pre;
    std::string post;
    SynapseSign sign = SynapseSign::Excitatory;
    std::int32_t outDegree = 0;
    WeightDist baseWeight;
    double gScale = 1.0;
    StorageKind storage = StorageKind::Sparse;
    std::int32_t preOffset = 0;
    std::int32_t preCount = -1;
    StdpRule stdp;  // extension F2
};

struct NetworkSpec {
    std::vector<NeuronPopulation> populations;
    std::vector<SynapseGroupSpec> synapses;
    double dtMs = 1.0;
    double durationMs = 1000.0;
    std::uint64_t globalSeed = 0;

    const NeuronPopulation* find_population(const std::string& name) const;
};

struct Violation {
    std::string field;
    std::string message;
};

std::vector<Violation> validate(const NetworkSpec& spec);
void require_valid(const NetworkSpec& spec);
std::int32_t group_pre_count(const SynapseGroupSpec& g, std::int32_t preSize);

struct IzhBuildOptions {
    double dtMs = 1.0;
    double durationMs = 1000.0;
    double noiseExc = 5.0;
    double noiseInh = 2.0;
    double excWeightHi = 0.5;
    double inhWeightHi = 1.0;
    double biasCurrent = 0.0;
    StorageKind storage = StorageKind::Sparse;
};

NetworkSpec build_izhikevich_net(std::int32_t nNeurons, std::int32_t nConn, double excFraction,
                                 double gScale, std::uint64_t seed,
                                 const IzhBuildOptions& opt = {});

struct MBodyBuildOptions {
    double dtMs = 1.0;
    double durationMs = 1000.0;
    double pnRateHz = 50.0;
    double pnKcOutFraction = 0.5;
    CondLifParams lif{};
    double pnKcWeightHi = 0.02;
    double pnLhiWeight = 0.02;
    double lhiKcWeight = 0.01;
    double kcDnWeight = 0.01;
    // extension: the KC model (CondLif as the reference, or Traub-Miles HH)
    ModelKind kcModel = ModelKind::CondLif;
    TraubMilesParams kcHH{};
};

NetworkSpec build_mbody_net(std::int32_t nPN, std::int32_t nLHI, std::int32_t nKC, std::int32_t nDN,
                            const std::map<std::string, double>& gScales, std::uint64_t seed,
                            const MBodyBuildOptions& opt = {});

// ---- engine (reference engine.hpp:14-104) ----------------------------------

// Auto (B200 extension): each group takes dense storage when its connection
// density outDegree / nPost is at least auto_dense_threshold() (measured
// crossover of the device kernels), CRS below it.  Like the
// reference's modes it never changes results (engine.hpp:15-18).
enum class StorageMode { FromSpec, ForceDense, ForceSparse, Auto };
double auto_dense_threshold();

struct SpikeEvent {
    std::int64_t step;
    std::int32_t population;
    std::int32_t neuron;
};

struct Raster {
    struct PopulationInfo {
        std::string name;
        std::int32_t size;
    };
    std::vector<PopulationInfo> populations;
    std::vector<SpikeEvent> events;  // (step, population, neuron) ascending
};

struct RunResult {
    Raster raster;
    std::map<std::string, double> avgSpike;
    std::int64_t sumNaNs = 0;
    std::int64_t steps = 0;
    double durationMs = 0.0;
    double wallTimeMs = 0.0;
};

// Host mirror of one population's device state.  The arrays a model does not
// use are empty, as in the reference.
struct PopulationState {
    std::vector<scalar> v, u;
    std::vector<scalar> gExc, gInh;
    std::vector<scalar> excIn, inhIn;
    std::vector<std::uint8_t> nanFlag;
    std::int64_t flagged = 0;
    std::vector<scalar> m, h, n;  // Traub-Miles gating variables (extension)
};

// Both run on the GPU over the caller's host arrays (no CPU path).
std::int64_t detect_nans(PopulationState& st, ModelKind model);
void propagate(const DenseMatrix& m, std::span<const std::int32_t> spikes, std::span<scalar> acc);
void propagate(const CrsMatrix& m, std::span<const std::int32_t> spikes, std::span<scalar> acc);

double avg_spike(const Raster& raster, const std::string& population, double durationMs);

// B200 engine knobs (no reference counterpart).  Zero fields take defaults.
struct EngineOptions {
    int device = 0;
    int window = 0;           // steps fused per launch window (default 64)
    int blockSize = 0;        // neuron-update block size (0 = occupancy policy)
    int blockPolicy = 0;      // 0 = occupancy model + SM fill, 1 = paper model only
    bool useGraphs = true;
    int heavyPreThreshold = 0;
    std::int64_t rasterCapacity = 0;
    bool profile = false;
    bool forceStepMode = false;
    // multi-GPU (one process per GPU): rank of world, NCCL id from
    // comm_unique_id() on rank 0 shared by the caller; virtualWorld > 1 runs
    // that many shards in this process on one GPU instead
    int rank = 0, world = 1, virtualWorld = 0, shardMinSize = 0;
    bool hasCommId = false;
    std::array<unsigned char, 128> commId{};
    int rasterPinnedMB = 0;  // pinned host pool for raster drains (B200 extension)
    bool rasterLocal = false;  // split runs: each rank records its own neurons only
};

// NCCL unique id for EngineOptions::commId (B200 extension).
std::array<unsigned char, 128> comm_unique_id();

class Simulation {
public:
    Simulation(const NetworkSpec& spec, StorageMode mode = StorageMode::FromSpec);
    Simulation(const NetworkSpec& spec, StorageMode mode, const EngineOptions& options);
    ~Simulation();
    Simulation(Simulation&&) noexcept;
    Simulation& operator=(Simulation&&) noexcept;

    void step();
    // B200 extension: n steps in one call (fused into launch windows).
    void step(std::int64_t n);
    std::int64_t steps_total() const;
    std::int64_t steps_done() const;

    // Live host mirrors: once handed out, a population's mirror is refreshed
    // after every step, and the mutable overload's edits are pushed to the
    // device before the next step (the reference's aliasing semantics).
    const PopulationState& population_state(const std::string& name) const;
    PopulationState& population_state(const std::string& name);

    const DenseMatrix* group_dense(const std::string& name) const;
    const CrsMatrix* group_sparse(const std::string& name) const;

    RunResult finish();

    struct Impl;

private:
    std::unique_ptr<Impl> impl_;
};

RunResult run(const NetworkSpec& spec, StorageMode mode = StorageMode::FromSpec);
// B200 extension: run with engine options.
RunResult run(const NetworkSpec& spec, StorageMode mode, const EngineOptions& options);

// ---- calibration sweep (reference calibration.hpp:12-42), the hot path's caller ----
// Cells run as independent device simulations, up to `parallelism` in flight,
// advanced round-robin by one host thread (each Simulation owns its streams,
// so in-flight cells overlap on the GPU); specs are built on host threads ahead.

struct SweepRow {
    std::int32_t nConn = 0;
    double gScale = 0.0;
    double avgSpike = 0.0;
    std::int64_t sumNaNs = 0;
    bool failed = false;
    std::string error;
};

using TemplateBuilder = std::function<NetworkSpec(std::int32_t nConn, double gScale)>;

struct SweepRequest {
    std::vector<std::int32_t> nConnValues;
    std::vector<double> gScaleValues;
    std::string targetPopulation;
    int parallelism = 1;
    StorageMode storage = StorageMode::FromSpec;
    std::function<void(const SweepRow&, std::size_t done, std::size_t total)> onCell;
    EngineOptions engine;  // B200 extension
};

std::vector<SweepRow> sweep(const TemplateBuilder& builder, const SweepRequest& req);

// ---- occupancy model (reference occupancy.hpp:10-70) -----------------------

struct DeviceSpec {
    std::string name;
    std::int64_t warpSize = 32;
    std::int64_t maxWarpsPerSM = 64;
    std::int64_t maxBlocksPerSM = 16;
    std::int64_t maxThreadsPerBlock = 1024;
    std::int64_t sharedMemPerSM = 49152;
    std::int64_t regsPerSM = 65536;
    std::int64_t regAllocUnit = 256;
    std::int64_t sharedAllocUnit = 256;
};

struct KernelSpec {
    std::int64_t threadsPerBlock = 0;
    std::int64_t regsPerThread = 0;
    std::int64_t sharedMemPerBlock = 0;
};

enum class Limiter { Warps, Blocks, SharedMem, Registers };
std::string to_string(Limiter l);

struct OccupancyResult {
    std::int64_t warpsPerBlock = 0;
    std::int64_t limitWarps = 0;
    std::int64_t limitBlocks = 0;
    std::int64_t limitShared = 0;
    std::int64_t limitRegs = 0;
    std::int64_t activeBlocks = 0;
    std::int64_t activeWarps = 0;
    double occupancy = 0.0;
    std::vector<Limiter> limiters;
};

inline constexpr std::int64_t kUnlimited = INT64_MAX;

void check_device(const DeviceSpec& dev);
OccupancyResult occupancy(const DeviceSpec& dev, const KernelSpec& kernel);
std::pair<std::int64_t, OccupancyResult> recommend_block_size(const DeviceSpec& dev,
                                                              std::int64_t regsPerThread,
                                                              std::int64_t sharedMemPerBlock);
DeviceSpec device_preset(const std::string& name);
std::vector<std::string> device_preset_names();

// ---- output formats (reference io.hpp:16-48, the parity artefacts only) ----

std::string format_double(double v);
std::string raster_to_csv(const Raster& raster);
std::string run_summary_to_json(const NetworkSpec& spec, const RunResult& result,
                                StorageMode mode);

}  // namespace synscale
