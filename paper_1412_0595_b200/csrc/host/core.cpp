// core.cpp — spec -> device network compile (reference Simulation ctor,
// engine.cpp:146-245), stepping contract (engine.cpp:316-319, 385-401) and
// result collection.
#include <cstdlib>
#include "core.hpp"

#include <atomic>
#include <cmath>
#include <exception>
#include <numeric>
#include <thread>

#include "connect_detail.hpp"

namespace ssb {

using namespace synscale;

namespace {

// step_count (reference engine.cpp:14-18)
std::int64_t step_count(double durationMs, double dtMs) {
    const auto n = static_cast<std::int64_t>(std::ceil(durationMs / dtMs - 1e-9));
    return std::max<std::int64_t>(n, 1);
}

double spike_rate(std::int64_t count, std::int32_t size, double durationMs) {
    return static_cast<double>(count) / (static_cast<double>(size) * (durationMs / 1000.0));
}

}  // namespace

}  // namespace ssb

namespace synscale {
// The density at and above which StorageMode::Auto stores a group dense: the
// crossover of the window kernels on B200 (profiles/r02_sweeps.md); the
// environment variable SSB_AUTO_DENSITY overrides it.
double auto_dense_threshold() {
    static const double t = [] {
        const char* e = std::getenv("SSB_AUTO_DENSITY");
        return e ? std::atof(e) : 0.25;
    }();
    return t;
}
}  // namespace synscale

namespace ssb {

void build_group_matrix(const NetworkSpec& spec, StorageMode mode, int gi,
                        std::optional<DenseMatrix>& dense, std::optional<CrsMatrix>& sparse) {
    const auto& gs = spec.synapses.at(gi);
    const NeuronPopulation* pre = spec.find_population(gs.pre);
    const NeuronPopulation* post = spec.find_population(gs.post);
    if (!pre || !post) throw SpecError("group '" + gs.name + "' names an unknown population");
    const std::int32_t nPre = group_pre_count(gs, pre->size), nPost = post->size;
    const bool inhibitory = gs.sign == SynapseSign::Inhibitory;
    const StorageKind eff =
        mode == StorageMode::ForceDense    ? StorageKind::Dense
        : mode == StorageMode::ForceSparse ? StorageKind::Sparse
        : mode == StorageMode::Auto
            ? (static_cast<double>(gs.outDegree) >= auto_dense_threshold() * nPost ? StorageKind::Dense
                                                                                   : StorageKind::Sparse)
            : gs.storage;
    detail::OutdegreeRows rows;
    rows.begin(nPre, nPost, gs.outDegree, gs.baseWeight, inhibitory ? -1 : +1,
               derive_seed(spec.globalSeed, gs.name));  // engine.cpp:223
    // gScale applied per nonzero in fp64 (engine.cpp:227-234); 0 blanks
    auto scaled = [&](scalar w) {
        const scalar s = static_cast<scalar>(static_cast<double>(w) * gs.gScale);
        if (!std::isfinite(s))
            throw SpecError("gScale " + std::to_string(gs.gScale) +
                            " overflows the weights of group '" + gs.name + "'");
        return s;
    };
    dense.reset();
    sparse.reset();
    if (eff == StorageKind::Dense) {
        DenseMatrix m;
        m.nPre = nPre;
        m.nPost = nPost;
        if (rows.full && gs.baseWeight.kind == WeightDist::Kind::Constant) {
            // all-to-all with one constant weight (lhi_kc, kc_dn, pn_lhi): every
            // entry is the same scaled value and no stream is drawn
            // (matrix.cpp:128-139 draws nothing for a constant distribution)
            scalar w = scalar(0);
            if (nPre > 0 && rows.next()) w = scaled(rows.vals[0]);
            m.weights.assign(static_cast<std::size_t>(nPre) * static_cast<std::size_t>(nPost), w);
            dense = std::move(m);
            return;
        }
        m.weights.assign(static_cast<std::size_t>(nPre) * static_cast<std::size_t>(nPost), scalar(0));
        for (std::int32_t r = 0; rows.next(); ++r) {
            scalar* dst = m.weights.data() + static_cast<std::size_t>(r) * nPost;
            for (std::int32_t j = 0; j < rows.k; ++j) dst[rows.cols[j]] = scaled(rows.vals[j]);
        }
        dense = std::move(m);
    } else {
        CrsMatrix m;  // to_sparse of the scaled rows (zeros dropped)
        m.nPre = nPre;
        m.nPost = nPost;
        m.rowStart.reserve(static_cast<std::size_t>(nPre) + 1);
        m.rowStart.push_back(0);
        const std::size_t est = static_cast<std::size_t>(nPre) * static_cast<std::size_t>(gs.outDegree);
        m.gValues.reserve(est);
        m.postInd.reserve(est);
        while (rows.next()) {
            for (std::int32_t j = 0; j < rows.k; ++j) {
                const scalar w = scaled(rows.vals[j]);
                if (w == scalar(0)) continue;
                m.postInd.push_back(rows.cols[j]);
                m.gValues.push_back(w);
            }
            m.rowStart.push_back(static_cast<std::int64_t>(m.gValues.size()));
        }
        sparse = std::move(m);
    }
}

SimCore::SimCore(const NetworkSpec& spec, StorageMode mode, const EngineConfig& cfg)
    : spec_(spec), mode_(mode), t0_(std::chrono::steady_clock::now()) {
    require_valid(spec_);
    net_.dtMs = spec_.dtMs;
    net_.dtS = static_cast<scalar>(spec_.dtMs);
    net_.durationMs = spec_.durationMs;
    net_.steps = step_count(spec_.durationMs, spec_.dtMs);

    for (const auto& ps : spec_.populations) {
        HostPop p;
        p.name = ps.name;
        p.n = ps.size;
        std::string label;
        switch (ps.model) {
        case ModelKind::PoissonSource:
            p.kind = kPoisson;
            p.p = std::get<PoissonParams>(ps.params).rateHz * spec_.dtMs / 1000.0;
            label = ps.name + "/source";
            break;
        case ModelKind::CondLif: {
            p.kind = kCondLif;
            const auto& c = std::get<CondLifParams>(ps.params);
            p.tauM = static_cast<scalar>(c.tauMMs);
            p.eLeak = static_cast<scalar>(c.eLeakMV);
            p.eExc = static_cast<scalar>(c.eExcMV);
            p.eInh = static_cast<scalar>(c.eInhMV);
            p.vThresh = static_cast<scalar>(c.vThreshMV);
            p.vReset = static_cast<scalar>(c.vResetMV);
            p.synDecay = static_cast<scalar>(std::exp(-spec_.dtMs / c.tauSynMs));
            break;
        }
        case ModelKind::TraubMiles: {  // extension (F1)
            p.kind = kTraubMiles;
            const auto& h = std::get<TraubMilesParams>(ps.params);
            p.gNa = static_cast<scalar>(h.gNa);
            p.ENa = static_cast<scalar>(h.ENa);
            p.gK = static_cast<scalar>(h.gK);
            p.EK = static_cast<scalar>(h.EK);
            p.gl = static_cast<scalar>(h.gl);
            p.El = static_cast<scalar>(h.El);
            p.Cm = static_cast<scalar>(h.C);
            p.eExc = static_cast<scalar>(h.eExcMV);
            p.eInh = static_cast<scalar>(h.eInhMV);
            p.substeps = h.substeps;
            p.mdt = static_cast<scalar>(spec_.dtMs / h.substeps);
            p.synDecay = static_cast<scalar>(std::exp(-spec_.dtMs / h.tauSynMs));
            break;
        }
        case ModelKind::Izhikevich: {
            p.kind = kIzhikevich;
            const auto& z = std::get<IzhikevichParams>(ps.params);
            for (std::size_t i = 0; i < z.a.size(); ++i) {
                p.a.push_back(static_cast<scalar>(z.a[i]));
                p.b.push_back(static_cast<scalar>(z.b[i]));
                p.c.push_back(static_cast<scalar>(z.c[i]));
                p.d.push_back(static_cast<scalar>(z.d[i]));
            }
            p.noise = z.noiseAmplitude;
            p.bias = z.biasCurrent;
            label = ps.name + "/noise";
            break;
        }
        }
        if (!label.empty()) {
            Mt19937_64 mt(stream_seed(spec_.globalSeed, ps.seed, label));
            p.mt = mt.state();
            p.mtPos = mt.position();
        }
        net_.pops.push_back(std::move(p));
    }

    dense_.resize(spec_.synapses.size());
    sparse_.resize(spec_.synapses.size());
    {
        // groups are independent (own derived seeds and streams): build them
        // on host threads, largest first
        const std::size_t ng = spec_.synapses.size();
        std::vector<std::size_t> todo(ng);
        std::iota(todo.begin(), todo.end(), 0);
        auto work = [&](std::size_t gi) {
            const auto& gs = spec_.synapses[gi];
            const auto* post = spec_.find_population(gs.post);
            return static_cast<double>(gs.outDegree) *
                   (spec_.find_population(gs.pre) ? spec_.find_population(gs.pre)->size : 0) +
                   (post ? post->size : 0);
        };
        std::sort(todo.begin(), todo.end(), [&](auto a, auto b) { return work(a) > work(b); });
        std::atomic<std::size_t> next{0};
        std::vector<std::exception_ptr> errs(ng);
        auto run = [&] {
            for (std::size_t i; (i = next.fetch_add(1)) < ng;) {
                try {
                    build_group_matrix(spec_, mode_, static_cast<int>(todo[i]), dense_[todo[i]],
                                       sparse_[todo[i]]);
                } catch (...) {
                    errs[todo[i]] = std::current_exception();
                }
            }
        };
        const unsigned nt = static_cast<unsigned>(std::min<std::size_t>(
            ng, std::max(1u, std::min(8u, std::thread::hardware_concurrency()))));
        std::vector<std::thread> pool;
        for (unsigned t = 1; t < nt; ++t) pool.emplace_back(run);
        run();
        for (auto& t : pool) t.join();
        for (auto& e : errs)  // the first failing group in spec order, as sequentially
            if (e) std::rethrow_exception(e);
    }
    for (std::size_t gi = 0; gi < spec_.synapses.size(); ++gi) {
        const auto& gs = spec_.synapses[gi];
        HostGroup g;
        g.name = gs.name;
        g.pre = pop_index(gs.pre);
        g.post = pop_index(gs.post);
        g.preOffset = gs.preOffset;
        g.preCount = group_pre_count(gs, spec_.populations[g.pre].size);
        g.inhibitory = gs.sign == SynapseSign::Inhibitory;
        g.nPre = g.preCount;
        g.nPost = spec_.populations[g.post].size;
        g.outDegree = gs.outDegree;
        g.dense = dense_[gi].has_value();
        if (gs.stdp.enabled) {  // extension F2
            if (!g.dense) throw SpecError("plastic group '" + gs.name + "' must be stored dense");
            g.plastic = true;
            g.aPlus = static_cast<float>(gs.stdp.aPlus);
            g.aMinus = static_cast<float>(gs.stdp.aMinus);
            g.decPlus = static_cast<float>(std::exp(-spec_.dtMs / gs.stdp.tauPlusMs));
            g.decMinus = static_cast<float>(std::exp(-spec_.dtMs / gs.stdp.tauMinusMs));
            g.wMax = static_cast<float>(gs.stdp.wMax);
        }
        if (g.dense) {
            g.W = dense_[gi]->weights.data();
        } else {
            g.g = sparse_[gi]->gValues.data();
            g.ind = sparse_[gi]->postInd.data();
            g.rowStart = sparse_[gi]->rowStart.data();
            g.nnz = sparse_[gi]->nnz();
        }
        net_.groups.push_back(std::move(g));
    }
    engine_ = std::make_unique<DeviceEngine>(net_, cfg);
}

int SimCore::pop_index(const std::string& name) const {
    for (std::size_t i = 0; i < spec_.populations.size(); ++i)
        if (spec_.populations[i].name == name) return static_cast<int>(i);
    throw SpecError("unknown population '" + name + "'");
}

int SimCore::group_index(const std::string& name) const {
    for (std::size_t i = 0; i < spec_.synapses.size(); ++i)
        if (spec_.synapses[i].name == name) return static_cast<int>(i);
    throw SpecError("unknown synapse group '" + name + "'");
}

void SimCore::step(std::int64_t n) {
    if (finished_) throw SpecError("simulation already finished");
    if (n < 0) throw SpecError("step count must be >= 0, got " + std::to_string(n));
    if (done_ + n > net_.steps)
        throw SpecError(done_ >= net_.steps ? "simulation already ran all its steps"
                                            : "only " + std::to_string(net_.steps - done_) +
                                                  " steps remain, " + std::to_string(n) + " requested");
    engine_->step(n);
    done_ += n;
}

void SimCore::finish() {
    if (finished_) throw SpecError("finish() may only be called once");
    if (done_ < net_.steps) step(net_.steps - done_);
    engine_->sync();
    // the raster (unless discarded by ssb_raster_discard) and the rates: the
    // rates come from the device's per-step counts, summed over the ranks of a
    // split run that records local rasters, so they never depend on the raster
    std::vector<std::int32_t> counts, neurons;
    if (!engine_->raster_discarded()) engine_->collect_raster(counts, neurons);
    std::vector<std::int64_t> perPop;
    engine_->global_spike_totals(perPop);
    const std::size_t np = spec_.populations.size();
    std::vector<double> rates(np);
    std::int64_t nans = 0;
    for (std::size_t p = 0; p < np; ++p) {
        rates[p] = spike_rate(perPop.at(p), spec_.populations[p].size, spec_.durationMs);
        std::int64_t f = 0;
        engine_->pull(static_cast<int>(p), kFieldFlagged, &f, 1);
        nans += f;
    }
    counts_ = std::move(counts);
    neurons_ = std::move(neurons);
    rates_ = std::move(rates);
    sumNaNs_ = nans;
    wallMs_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count();
    finished_ = true;
}

RunResult SimCore::run_result() const {
    RunResult r;
    r.steps = net_.steps;
    r.durationMs = spec_.durationMs;
    r.sumNaNs = sumNaNs_;
    r.wallTimeMs = wallMs_;
    const std::size_t np = spec_.populations.size();
    for (std::size_t p = 0; p < np; ++p) {
        r.raster.populations.push_back({spec_.populations[p].name, spec_.populations[p].size});
        r.avgSpike[spec_.populations[p].name] = rates_[p];
    }
    r.raster.events.reserve(neurons_.size());
    std::size_t at = 0;
    for (std::size_t i = 0; i < counts_.size(); ++i) {
        const std::int64_t step = static_cast<std::int64_t>(i / np);
        const std::int32_t pop = static_cast<std::int32_t>(i % np);
        for (std::int32_t k = 0; k < counts_[i]; ++k)
            r.raster.events.push_back({step, pop, neurons_[at++]});
    }
    return r;
}

}  // namespace ssb
