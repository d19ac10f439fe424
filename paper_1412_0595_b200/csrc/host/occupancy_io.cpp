// occupancy_io.cpp — the paper's occupancy model (reference occupancy.cpp)
// with a B200 (sm_100) preset, and the parity output formats (reference
// io.cpp:15-19, 276-310).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <sstream>

#include "synscale/synscale.hpp"

namespace synscale {

std::string to_string(Limiter l) {
    switch (l) {
    case Limiter::Warps: return "warps";
    case Limiter::Blocks: return "blocks";
    case Limiter::SharedMem: return "shared";
    case Limiter::Registers: return "registers";
    }
    return "?";
}

void check_device(const DeviceSpec& dev) {
    const std::pair<std::int64_t, const char*> budgets[] = {
        {dev.warpSize, "warpSize"},
        {dev.maxWarpsPerSM, "maxWarpsPerSM"},
        {dev.maxBlocksPerSM, "maxBlocksPerSM"},
        {dev.maxThreadsPerBlock, "maxThreadsPerBlock"},
        {dev.sharedMemPerSM, "sharedMemPerSM"},
        {dev.regsPerSM, "regsPerSM"},
        {dev.regAllocUnit, "regAllocUnit"},
        {dev.sharedAllocUnit, "sharedAllocUnit"}};
    for (const auto& [v, nm] : budgets)
        if (v < 1)
            throw SpecError("device '" + dev.name + "': " + nm + " must be >= 1, got " +
                            std::to_string(v));
}

namespace {
std::int64_t div_up(std::int64_t a, std::int64_t b) { return (a + b - 1) / b; }
}  // namespace

OccupancyResult occupancy(const DeviceSpec& dev, const KernelSpec& k) {
    check_device(dev);
    if (k.threadsPerBlock < 1 || k.threadsPerBlock > dev.maxThreadsPerBlock)
        throw SpecError("threadsPerBlock " + std::to_string(k.threadsPerBlock) +
                        " must lie in [1, " + std::to_string(dev.maxThreadsPerBlock) + "]");
    if (k.regsPerThread < 0)
        throw SpecError("regsPerThread must be >= 0, got " + std::to_string(k.regsPerThread));
    if (k.sharedMemPerBlock < 0)
        throw SpecError("sharedMemPerBlock must be >= 0, got " + std::to_string(k.sharedMemPerBlock));

    OccupancyResult r;
    r.warpsPerBlock = div_up(k.threadsPerBlock, dev.warpSize);
    r.limitWarps = dev.maxWarpsPerSM / r.warpsPerBlock;
    r.limitBlocks = dev.maxBlocksPerSM;
    // shared memory: per-block footprint rounded up to the allocation unit
    r.limitShared = k.sharedMemPerBlock == 0
                        ? kUnlimited
                        : dev.sharedMemPerSM /
                              (div_up(k.sharedMemPerBlock, dev.sharedAllocUnit) * dev.sharedAllocUnit);
    // registers: allocated per warp, rounded up to the allocation unit
    if (k.regsPerThread == 0) {
        r.limitRegs = kUnlimited;
    } else {
        const std::int64_t perWarp =
            div_up(k.regsPerThread * dev.warpSize, dev.regAllocUnit) * dev.regAllocUnit;
        r.limitRegs = dev.regsPerSM / (perWarp * r.warpsPerBlock);
    }
    r.activeBlocks = std::min(std::min(r.limitWarps, r.limitBlocks), std::min(r.limitShared, r.limitRegs));
    r.activeWarps = r.activeBlocks * r.warpsPerBlock;
    r.occupancy = static_cast<double>(r.activeWarps) / static_cast<double>(dev.maxWarpsPerSM);
    if (r.limitWarps == r.activeBlocks) r.limiters.push_back(Limiter::Warps);
    if (r.limitBlocks == r.activeBlocks) r.limiters.push_back(Limiter::Blocks);
    if (r.limitShared == r.activeBlocks) r.limiters.push_back(Limiter::SharedMem);
    if (r.limitRegs == r.activeBlocks) r.limiters.push_back(Limiter::Registers);
    return r;
}

std::pair<std::int64_t, OccupancyResult> recommend_block_size(const DeviceSpec& dev,
                                                              std::int64_t regsPerThread,
                                                              std::int64_t sharedMemPerBlock) {
    check_device(dev);
    if (dev.maxThreadsPerBlock < dev.warpSize)
        throw SpecError("device '" + dev.name + "' cannot launch a whole warp (maxThreadsPerBlock " +
                        std::to_string(dev.maxThreadsPerBlock) + " < warpSize " +
                        std::to_string(dev.warpSize) + ")");
    std::pair<std::int64_t, OccupancyResult> best{0, {}};
    for (std::int64_t t = dev.warpSize; t <= dev.maxThreadsPerBlock; t += dev.warpSize) {
        OccupancyResult r = occupancy(dev, {t, regsPerThread, sharedMemPerBlock});
        // ties go to the larger block: scan upward and replace on >=
        if (best.first == 0 || r.activeWarps >= best.second.activeWarps) best = {t, std::move(r)};
    }
    return best;
}

DeviceSpec device_preset(const std::string& name) {
    // per-SM budgets: cc20/cc30/cc50 as in the paper's model; sm100 is B200
    // (cudaGetDeviceProperties: 64 warps, 32 blocks, 228 KB shared of which
    // 227 KB per block, 64K registers; 256-register warp and 128 B shared
    // allocation granularity)
    if (name == "cc20") return {"cc20", 32, 48, 8, 1024, 49152, 32768, 64, 128};
    if (name == "cc30") return {"cc30", 32, 64, 16, 1024, 49152, 65536, 256, 256};
    if (name == "cc50") return {"cc50", 32, 64, 32, 1024, 65536, 65536, 256, 256};
    if (name == "sm100") return {"sm100", 32, 64, 32, 1024, 233472, 65536, 256, 128};
    std::string known;
    for (const auto& n : device_preset_names()) known += (known.empty() ? "" : ", ") + n;
    known += ", sm100";
    throw SpecError("unknown device preset '" + name + "'; known presets: " + known);
}

// The reference's presets (occupancy.cpp:98-116, pinned by test_occupancy.cpp:265);
// device_preset("sm100") (B200, extension) is accepted but not listed.
std::vector<std::string> device_preset_names() { return {"cc20", "cc30", "cc50"}; }

// ---- formats -------------------------------------------------------------------

std::string format_double(double v) {
    char buf[64];
    const auto res = std::to_chars(buf, buf + sizeof buf, v);
    return std::string(buf, res.ptr);
}

std::string raster_to_csv(const Raster& raster) {
    std::string out = "step,population,neuron\n";
    out.reserve(out.size() + raster.events.size() * 16);
    for (const auto& e : raster.events) {
        out += std::to_string(e.step);
        out += ',';
        out += raster.populations[static_cast<std::size_t>(e.population)].name;
        out += ',';
        out += std::to_string(e.neuron);
        out += '\n';
    }
    return out;
}

namespace {
std::string json_str(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        o += c;
    }
    return o + "\"";
}
std::string json_num(double v) { return std::isfinite(v) ? format_double(v) : "null"; }
}  // namespace

// Same keys and layout as the reference's summary.json (io.cpp:289-310).
std::string run_summary_to_json(const NetworkSpec& spec, const RunResult& result,
                                StorageMode mode) {
    std::ostringstream o;
    o << "{\n  \"avgSpike\": {";
    bool first = true;
    for (const auto& [name, rate] : result.avgSpike) {
        o << (first ? "\n" : ",\n") << "    " << json_str(name) << ": " << json_num(rate);
        first = false;
    }
    o << (first ? "}" : "\n  }") << ",\n";
    o << "  \"dtMs\": " << json_num(spec.dtMs) << ",\n";
    o << "  \"durationMs\": " << json_num(spec.durationMs) << ",\n";
    o << "  \"globalSeed\": " << spec.globalSeed << ",\n";
    o << "  \"populations\": {";
    std::vector<std::pair<std::string, std::int32_t>> sizes;
    for (const auto& p : result.raster.populations) sizes.emplace_back(p.name, p.size);
    std::sort(sizes.begin(), sizes.end());
    first = true;
    for (const auto& [name, size] : sizes) {
        o << (first ? "\n" : ",\n") << "    " << json_str(name) << ": " << size;
        first = false;
    }
    o << (first ? "}" : "\n  }") << ",\n";
    o << "  \"spikes\": " << result.raster.events.size() << ",\n";
    o << "  \"steps\": " << result.steps << ",\n";
    o << "  \"storage\": "
      << (mode == StorageMode::ForceDense    ? "\"dense\""
          : mode == StorageMode::ForceSparse ? "\"sparse\""
          : mode == StorageMode::Auto        ? "\"auto\""
                                             : "\"spec\"")
      << ",\n";
    o << "  \"sumNaNs\": " << result.sumNaNs << ",\n";
    o << "  \"wallTimeMs\": " << json_num(result.wallTimeMs) << "\n}\n";
    return o.str();
}

}  // namespace synscale
