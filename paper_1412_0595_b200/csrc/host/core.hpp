// core.hpp — SimCore: one simulation = validated spec + host connectivity +
// device engine + collected results.  Shared by the C++ facade
// (synscale::Simulation) and the C ABI (ssb_sim).
#pragma once

#include <chrono>
#include <memory>
#include <optional>
#include <vector>

#include "../engine.hpp"
#include "synscale/synscale.hpp"

namespace ssb {

// Connectivity of synapse group `gi` exactly as the reference Simulation
// constructor builds it (engine.cpp:214-244): gen_fixed_outdegree from
// derive_seed(globalSeed, name), gScale in fp64, dense or CRS per `mode`.
// Exactly one of dense/sparse is set on return.
void build_group_matrix(const synscale::NetworkSpec& spec, synscale::StorageMode mode, int gi,
                        std::optional<synscale::DenseMatrix>& dense,
                        std::optional<synscale::CrsMatrix>& sparse);

class SimCore {
public:
    SimCore(const synscale::NetworkSpec& spec, synscale::StorageMode mode, const EngineConfig& cfg);

    void step(std::int64_t n);  // SpecError on misuse
    void finish();              // SpecError when called twice
    std::int64_t steps_total() const { return net_.steps; }
    std::int64_t steps_done() const { return done_; }
    bool finished() const { return finished_; }

    int pop_index(const std::string& name) const;    // SpecError if unknown
    int group_index(const std::string& name) const;  // SpecError if unknown
    int n_pops() const { return static_cast<int>(spec_.populations.size()); }
    int n_groups() const { return static_cast<int>(spec_.synapses.size()); }
    int pop_size(int pop) const { return spec_.populations.at(pop).size; }
    synscale::ModelKind pop_model(int pop) const { return spec_.populations.at(pop).model; }

    const synscale::DenseMatrix* dense(int g) const { return dense_.at(g) ? &*dense_[g] : nullptr; }
    const synscale::CrsMatrix* sparse(int g) const { return sparse_.at(g) ? &*sparse_[g] : nullptr; }

    DeviceEngine& engine() { return *engine_; }
    const DeviceEngine& engine() const { return *engine_; }
    const synscale::NetworkSpec& spec() const { return spec_; }
    synscale::StorageMode mode() const { return mode_; }

    // results (valid after finish)
    const std::vector<std::int32_t>& counts() const { return counts_; }
    const std::vector<std::int32_t>& neurons() const { return neurons_; }
    const std::vector<double>& rates() const { return rates_; }
    std::int64_t sum_nans() const { return sumNaNs_; }
    double wall_ms() const { return wallMs_; }
    synscale::RunResult run_result() const;  // expands the raster

private:
    synscale::NetworkSpec spec_;
    synscale::StorageMode mode_;
    HostNet net_;
    std::vector<std::optional<synscale::DenseMatrix>> dense_;
    std::vector<std::optional<synscale::CrsMatrix>> sparse_;
    std::unique_ptr<DeviceEngine> engine_;
    std::int64_t done_ = 0;
    bool finished_ = false;
    std::chrono::steady_clock::time_point t0_;
    std::vector<std::int32_t> counts_, neurons_;
    std::vector<double> rates_;
    std::int64_t sumNaNs_ = 0;
    double wallMs_ = 0.0;
};

}  // namespace ssb
