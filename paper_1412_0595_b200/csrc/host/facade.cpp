// facade.cpp — the reference's C++ engine API (engine.hpp:59-104) on top of
// the device engine: Simulation with live host mirrors, run(), and the free
// functions propagate()/detect_nans()/avg_spike().
#include <cmath>

#include "core.hpp"

namespace synscale {

namespace {

ssb::EngineConfig to_config(const EngineOptions& o) {
    ssb::EngineConfig c;
    c.device = o.device;
    if (o.window > 0) c.window = o.window;
    c.blockSize = o.blockSize;
    c.blockPolicy = o.blockPolicy;
    c.useGraphs = o.useGraphs;
    if (o.heavyPreThreshold > 0) c.heavyPreThreshold = o.heavyPreThreshold;
    c.rasterCapacity = o.rasterCapacity;
    c.profile = o.profile;
    c.forceStepMode = o.forceStepMode;
    c.rank = o.rank;
    c.world = std::max(1, o.world);
    c.virtualWorld = o.virtualWorld;
    if (o.shardMinSize > 0) c.shardMinSize = o.shardMinSize;
    c.hasCommId = o.hasCommId;
    c.commId = o.commId;
    c.rasterPinnedMB = std::max(0, o.rasterPinnedMB);
    c.rasterLocal = o.rasterLocal;
    return c;
}

}  // namespace

struct Simulation::Impl {
    ssb::SimCore core;
    mutable std::vector<PopulationState> mirror;
    mutable std::vector<char> observed;  // refresh after every step
    mutable std::vector<char> writable;  // push before every step

    Impl(const NetworkSpec& spec, StorageMode mode, const EngineOptions& opt)
        : core(spec, mode, to_config(opt)),
          mirror(spec.populations.size()),
          observed(spec.populations.size(), 0),
          writable(spec.populations.size(), 0) {}

    static constexpr int kMirrored[] = {ssb::kFieldV,     ssb::kFieldU,     ssb::kFieldGExc,
                                        ssb::kFieldGInh,  ssb::kFieldExcIn, ssb::kFieldInhIn,
                                        ssb::kFieldM,     ssb::kFieldH,     ssb::kFieldN};
    // fields a model keeps (the others stay empty, as in the reference)
    static bool uses(ModelKind m, int field) {
        switch (field) {
        case ssb::kFieldV: return m != ModelKind::PoissonSource;
        case ssb::kFieldU: return m == ModelKind::Izhikevich;
        case ssb::kFieldGExc:
        case ssb::kFieldGInh: return m == ModelKind::CondLif || m == ModelKind::TraubMiles;
        case ssb::kFieldM:
        case ssb::kFieldH:
        case ssb::kFieldN: return m == ModelKind::TraubMiles;
        default: return true;
        }
    }
    static std::vector<scalar>* vec(PopulationState& s, int field) {
        switch (field) {
        case ssb::kFieldV: return &s.v;
        case ssb::kFieldU: return &s.u;
        case ssb::kFieldGExc: return &s.gExc;
        case ssb::kFieldGInh: return &s.gInh;
        case ssb::kFieldExcIn: return &s.excIn;
        case ssb::kFieldInhIn: return &s.inhIn;
        case ssb::kFieldM: return &s.m;
        case ssb::kFieldH: return &s.h;
        case ssb::kFieldN: return &s.n;
        }
        return nullptr;
    }

    void refresh(int p) const {
        auto& s = mirror[p];
        const ModelKind m = core.pop_model(p);
        const std::int64_t n = core.pop_size(p);
        auto& eng = const_cast<ssb::SimCore&>(core).engine();
        for (int f : kMirrored) {
            if (!uses(m, f)) continue;
            auto* v = vec(s, f);
            v->resize(static_cast<std::size_t>(n));
            eng.pull(p, f, v->data(), n);
        }
        s.nanFlag.resize(static_cast<std::size_t>(n));
        eng.pull(p, ssb::kFieldNanFlag, s.nanFlag.data(), n);
        eng.pull(p, ssb::kFieldFlagged, &s.flagged, 1);
    }

    void push_edits() {
        for (std::size_t p = 0; p < mirror.size(); ++p) {
            if (!writable[p]) continue;
            auto& s = mirror[p];
            const ModelKind m = core.pop_model(static_cast<int>(p));
            const std::int64_t n = core.pop_size(static_cast<int>(p));
            auto& eng = core.engine();
            for (int f : kMirrored) {
                if (!uses(m, f)) continue;
                auto* v = vec(s, f);
                if (static_cast<std::int64_t>(v->size()) != n)
                    throw SpecError("population state array was resized");
                eng.push(static_cast<int>(p), f, v->data(), n);
            }
            if (static_cast<std::int64_t>(s.nanFlag.size()) != n)
                throw SpecError("population nanFlag array was resized");
            eng.push(static_cast<int>(p), ssb::kFieldNanFlag, s.nanFlag.data(), n);
            eng.push(static_cast<int>(p), ssb::kFieldFlagged, &s.flagged, 1);
        }
    }

    void refresh_observed() const {
        for (std::size_t p = 0; p < mirror.size(); ++p)
            if (observed[p]) refresh(static_cast<int>(p));
    }
};

Simulation::Simulation(const NetworkSpec& spec, StorageMode mode)
    : Simulation(spec, mode, EngineOptions{}) {}

Simulation::Simulation(const NetworkSpec& spec, StorageMode mode, const EngineOptions& options)
    : impl_(std::make_unique<Impl>(spec, mode, options)) {}

Simulation::~Simulation() = default;
Simulation::Simulation(Simulation&&) noexcept = default;
Simulation& Simulation::operator=(Simulation&&) noexcept = default;

void Simulation::step() { step(1); }

void Simulation::step(std::int64_t n) {
    auto& m = *impl_;
    if (m.core.finished()) throw SpecError("simulation already finished");
    m.push_edits();
    // observed populations need the mirror after every single step
    const bool perStep = std::any_of(m.observed.begin(), m.observed.end(), [](char c) { return c; });
    if (perStep) {
        for (std::int64_t i = 0; i < n; ++i) {
            m.core.step(1);
            m.refresh_observed();
        }
    } else {
        m.core.step(n);
    }
}

std::int64_t Simulation::steps_total() const { return impl_->core.steps_total(); }
std::int64_t Simulation::steps_done() const { return impl_->core.steps_done(); }

const PopulationState& Simulation::population_state(const std::string& name) const {
    const int p = impl_->core.pop_index(name);
    if (!impl_->observed[p]) {
        impl_->observed[p] = 1;
        impl_->refresh(p);
    }
    return impl_->mirror[p];
}

PopulationState& Simulation::population_state(const std::string& name) {
    const int p = impl_->core.pop_index(name);
    if (!impl_->observed[p]) {
        impl_->observed[p] = 1;
        impl_->refresh(p);
    }
    impl_->writable[p] = 1;
    return impl_->mirror[p];
}

const DenseMatrix* Simulation::group_dense(const std::string& name) const {
    return impl_->core.dense(impl_->core.group_index(name));
}

const CrsMatrix* Simulation::group_sparse(const std::string& name) const {
    return impl_->core.sparse(impl_->core.group_index(name));
}

RunResult Simulation::finish() {
    auto& m = *impl_;
    if (m.core.finished()) throw SpecError("finish() may only be called once");
    const std::int64_t left = m.core.steps_total() - m.core.steps_done();
    if (left > 0) step(left);
    m.push_edits();
    m.core.finish();
    m.refresh_observed();
    return m.core.run_result();
}

RunResult run(const NetworkSpec& spec, StorageMode mode) { return run(spec, mode, EngineOptions{}); }

RunResult run(const NetworkSpec& spec, StorageMode mode, const EngineOptions& options) {
    const auto t0 = std::chrono::steady_clock::now();
    Simulation sim(spec, mode, options);
    RunResult r = sim.finish();
    r.wallTimeMs =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return r;
}

// ---- free functions -----------------------------------------------------------

namespace {
void check_spikes(std::span<const std::int32_t> spikes, std::int32_t nPre) {
    for (std::int32_t i : spikes)
        if (i < 0 || i >= nPre)
            throw SpecError("spike index " + std::to_string(i) + " outside [0, " +
                            std::to_string(nPre) + ")");
}
void check_acc(std::size_t len, std::int32_t nPost) {
    if (static_cast<std::int64_t>(len) != nPost)
        throw SpecError("accumulator length " + std::to_string(len) + " does not match nPost " +
                        std::to_string(nPost));
}
}  // namespace

void propagate(const DenseMatrix& m, std::span<const std::int32_t> spikes, std::span<scalar> acc) {
    check_acc(acc.size(), m.nPost);
    check_spikes(spikes, m.nPre);
    if (spikes.empty()) return;
    ssb::device_propagate_dense(m.weights.data(), m.nPre, m.nPost, spikes.data(),
                                static_cast<std::int64_t>(spikes.size()), acc.data());
}

void propagate(const CrsMatrix& m, std::span<const std::int32_t> spikes, std::span<scalar> acc) {
    check_acc(acc.size(), m.nPost);
    check_spikes(spikes, m.nPre);
    if (spikes.empty()) return;
    ssb::device_propagate_crs(m.gValues.data(), m.postInd.data(), m.rowStart.data(), m.nPre,
                              m.nPost, spikes.data(), static_cast<std::int64_t>(spikes.size()),
                              acc.data());
}

std::int64_t detect_nans(PopulationState& st, ModelKind model) {
    const std::int64_t n = static_cast<std::int64_t>(st.nanFlag.size());
    auto ptr = [&](const std::vector<scalar>& v) -> const float* {
        if (v.empty()) return nullptr;
        if (static_cast<std::int64_t>(v.size()) != n)
            throw SpecError("state arrays and nanFlag differ in length");
        return v.data();
    };
    const int kind = model == ModelKind::Izhikevich ? 0 : model == ModelKind::PoissonSource ? 1 : 2;
    if (kind == 1) return 0;  // sources hold no continuous state
    const std::int64_t newly = ssb::device_detect_nans(kind, ptr(st.v), ptr(st.u), ptr(st.gExc),
                                                       ptr(st.gInh), st.nanFlag.data(), n);
    st.flagged += newly;
    return newly;
}

double avg_spike(const Raster& raster, const std::string& population, double durationMs) {
    if (!std::isfinite(durationMs) || !(durationMs > 0.0))
        throw SpecError("durationMs must be finite and > 0");
    std::int32_t index = -1, size = 0;
    for (std::size_t i = 0; i < raster.populations.size(); ++i)
        if (raster.populations[i].name == population) {
            index = static_cast<std::int32_t>(i);
            size = raster.populations[i].size;
            break;
        }
    if (index < 0) throw SpecError("raster has no population named '" + population + "'");
    if (size < 1) throw SpecError("population '" + population + "' has a non-positive size");
    std::int64_t count = 0;
    for (const auto& e : raster.events) count += e.population == index;
    return static_cast<double>(count) / (static_cast<double>(size) * (durationMs / 1000.0));
}

}  // namespace synscale

namespace synscale {
std::array<unsigned char, 128> comm_unique_id() { return ssb::comm_unique_id(); }
}  // namespace synscale
