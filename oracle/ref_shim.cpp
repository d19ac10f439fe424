// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.  A C ABI over the UNMODIFIED
// reference library (compiled by oracle/Makefile from the sources under
// /root/reference/proj into oracle/_ref/libsynscale_ref.so).  It lets the
// Python tests and bench.py's reference arm drive the reference's own
// Simulation / run / propagate / gen_fixed_outdegree through its public C++
// API (include/synscale/*.hpp), to pin the oracle restatement and to time the
// reference CPU path.  Nothing here is product code.
#include <chrono>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "synscale/engine.hpp"
#include "synscale/matrix.hpp"
#include "synscale/network.hpp"
#include "synscale/random.hpp"

#include "../include/synscale_b200.h"

#define REF_API extern "C" __attribute__((visibility("default")))

using namespace synscale;

namespace {

NetworkSpec to_spec(const ssb_net_desc* d) {
    NetworkSpec s;
    s.dtMs = d->dt_ms;
    s.durationMs = d->duration_ms;
    s.globalSeed = d->global_seed;
    for (int i = 0; i < d->n_pops; ++i) {
        const ssb_pop_desc& p = d->pops[i];
        NeuronPopulation np;
        np.name = p.name;
        np.size = p.size;
        np.seed = p.seed;
        if (p.model == SSB_MODEL_POISSON) {
            np.model = ModelKind::PoissonSource;
            np.params = PoissonParams{p.rate_hz};
        } else if (p.model == SSB_MODEL_CONDLIF) {
            np.model = ModelKind::CondLif;
            CondLifParams c;
            c.tauMMs = p.tau_m_ms;
            c.eLeakMV = p.e_leak_mv;
            c.vThreshMV = p.v_thresh_mv;
            c.vResetMV = p.v_reset_mv;
            c.eExcMV = p.e_exc_mv;
            c.eInhMV = p.e_inh_mv;
            c.tauSynMs = p.tau_syn_ms;
            np.params = c;
        } else {
            np.model = ModelKind::Izhikevich;
            IzhikevichParams z;
            const std::size_t n = static_cast<std::size_t>(p.size);
            z.a.assign(p.izh_a, p.izh_a + n);
            z.b.assign(p.izh_b, p.izh_b + n);
            z.c.assign(p.izh_c, p.izh_c + n);
            z.d.assign(p.izh_d, p.izh_d + n);
            z.noiseAmplitude.assign(p.izh_noise, p.izh_noise + n);
            z.biasCurrent.assign(p.izh_bias, p.izh_bias + n);
            np.params = std::move(z);
        }
        s.populations.push_back(std::move(np));
    }
    for (int i = 0; i < d->n_groups; ++i) {
        const ssb_group_desc& g = d->groups[i];
        SynapseGroupSpec sg;
        sg.name = g.name;
        sg.pre = g.pre;
        sg.post = g.post;
        sg.sign = g.sign == SSB_SIGN_INH ? SynapseSign::Inhibitory : SynapseSign::Excitatory;
        sg.outDegree = g.out_degree;
        if (g.weight_kind == SSB_WEIGHT_UNIFORM) {
            sg.baseWeight.kind = WeightDist::Kind::Uniform;
            sg.baseWeight.lo = g.weight_lo;
            sg.baseWeight.hi = g.weight_hi;
        } else {
            sg.baseWeight.kind = WeightDist::Kind::Constant;
            sg.baseWeight.value = g.weight_value;
        }
        sg.gScale = g.g_scale;
        sg.storage = g.storage == SSB_STORAGE_DENSE ? StorageKind::Dense : StorageKind::Sparse;
        sg.preOffset = g.pre_offset;
        sg.preCount = g.pre_count;
        s.synapses.push_back(std::move(sg));
    }
    return s;
}

StorageMode to_mode(int m) {
    return m == SSB_MODE_FORCE_DENSE    ? StorageMode::ForceDense
           : m == SSB_MODE_FORCE_SPARSE ? StorageMode::ForceSparse
                                        : StorageMode::FromSpec;
}

int fail(const std::exception& e, char* err, std::size_t errlen) {
    if (err && errlen) {
        std::strncpy(err, e.what(), errlen - 1);
        err[errlen - 1] = 0;
    }
    return dynamic_cast<const SpecError*>(&e) ? 2 : 1;
}

struct RefSim {
    NetworkSpec spec;
    std::unique_ptr<Simulation> sim;
    std::vector<std::string> popNames;
    std::vector<std::string> groupNames;
    RunResult result;
    bool finished = false;
};

}  // namespace

REF_API RefSim* ref_create(const ssb_net_desc* d, int mode, char* err, std::size_t errlen) {
    try {
        auto r = std::make_unique<RefSim>();
        r->spec = to_spec(d);
        r->sim = std::make_unique<Simulation>(r->spec, to_mode(mode));
        for (const auto& p : r->spec.populations) r->popNames.push_back(p.name);
        for (const auto& g : r->spec.synapses) r->groupNames.push_back(g.name);
        return r.release();
    } catch (const std::exception& e) {
        fail(e, err, errlen);
        return nullptr;
    }
}

REF_API void ref_destroy(RefSim* r) { delete r; }

REF_API int ref_step(RefSim* r, long long n) {
    try {
        for (long long i = 0; i < n; ++i) r->sim->step();
        return 0;
    } catch (const std::exception& e) {
        return fail(e, nullptr, 0);
    }
}

REF_API long long ref_steps_total(RefSim* r) { return r->sim->steps_total(); }
REF_API long long ref_steps_done(RefSim* r) { return r->sim->steps_done(); }

REF_API int ref_finish(RefSim* r) {
    try {
        r->result = r->sim->finish();
        r->finished = true;
        return 0;
    } catch (const std::exception& e) {
        return fail(e, nullptr, 0);
    }
}

REF_API long long ref_n_events(RefSim* r) {
    return static_cast<long long>(r->result.raster.events.size());
}

REF_API int ref_raster(RefSim* r, int64_t* step, int32_t* pop, int32_t* neuron, long long cap) {
    const auto& ev = r->result.raster.events;
    if (static_cast<long long>(ev.size()) > cap) return 2;
    for (std::size_t i = 0; i < ev.size(); ++i) {
        step[i] = ev[i].step;
        pop[i] = ev[i].population;
        neuron[i] = ev[i].neuron;
    }
    return 0;
}

REF_API int ref_rates(RefSim* r, double* out, int n) {
    for (int i = 0; i < n; ++i) out[i] = r->result.avgSpike.at(r->popNames[i]);
    return 0;
}

REF_API long long ref_sum_nans(RefSim* r) { return r->result.sumNaNs; }

REF_API int ref_get_state(RefSim* r, int pop, int field, void* dst, long long n) {
    try {
        auto& st = r->sim->population_state(r->popNames.at(pop));
        const std::vector<float>* src = nullptr;
        switch (field) {
        case SSB_FIELD_V: src = &st.v; break;
        case SSB_FIELD_U: src = &st.u; break;
        case SSB_FIELD_GEXC: src = &st.gExc; break;
        case SSB_FIELD_GINH: src = &st.gInh; break;
        case SSB_FIELD_EXCIN: src = &st.excIn; break;
        case SSB_FIELD_INHIN: src = &st.inhIn; break;
        case SSB_FIELD_NANFLAG:
            if (static_cast<long long>(st.nanFlag.size()) != n) return 2;
            std::memcpy(dst, st.nanFlag.data(), st.nanFlag.size());
            return 0;
        case SSB_FIELD_FLAGGED: *static_cast<int64_t*>(dst) = st.flagged; return 0;
        default: return 2;
        }
        // arrays a model does not use are empty in the reference
        if (src->empty()) {
            std::memset(dst, 0, sizeof(float) * static_cast<std::size_t>(n));
            return 0;
        }
        if (static_cast<long long>(src->size()) != n) return 2;
        std::memcpy(dst, src->data(), sizeof(float) * src->size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e, nullptr, 0);
    }
}

REF_API int ref_set_state(RefSim* r, int pop, int field, const void* src, long long n) {
    try {
        auto& st = r->sim->population_state(r->popNames.at(pop));
        std::vector<float>* dst = nullptr;
        switch (field) {
        case SSB_FIELD_V: dst = &st.v; break;
        case SSB_FIELD_U: dst = &st.u; break;
        case SSB_FIELD_GEXC: dst = &st.gExc; break;
        case SSB_FIELD_GINH: dst = &st.gInh; break;
        case SSB_FIELD_EXCIN: dst = &st.excIn; break;
        case SSB_FIELD_INHIN: dst = &st.inhIn; break;
        case SSB_FIELD_FLAGGED: st.flagged = *static_cast<const int64_t*>(src); return 0;
        default: return 2;
        }
        if (static_cast<long long>(dst->size()) != n) return 2;
        std::memcpy(dst->data(), src, sizeof(float) * dst->size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e, nullptr, 0);
    }
}

REF_API int ref_group_info(RefSim* r, int g, int32_t* dense, int32_t* nPre, int32_t* nPost,
                           int64_t* nnz) {
    const auto& name = r->groupNames.at(g);
    if (const DenseMatrix* d = r->sim->group_dense(name)) {
        *dense = 1;
        *nPre = d->nPre;
        *nPost = d->nPost;
        *nnz = -1;
    } else {
        const CrsMatrix* s = r->sim->group_sparse(name);
        *dense = 0;
        *nPre = s->nPre;
        *nPost = s->nPost;
        *nnz = s->nnz();
    }
    return 0;
}

REF_API int ref_group_dense(RefSim* r, int g, float* out) {
    const DenseMatrix* d = r->sim->group_dense(r->groupNames.at(g));
    if (!d) return 2;
    std::memcpy(out, d->weights.data(), sizeof(float) * d->weights.size());
    return 0;
}

REF_API int ref_group_sparse(RefSim* r, int g, float* gv, int32_t* ind, int64_t* rs) {
    const CrsMatrix* s = r->sim->group_sparse(r->groupNames.at(g));
    if (!s) return 2;
    std::memcpy(gv, s->gValues.data(), sizeof(float) * s->gValues.size());
    std::memcpy(ind, s->postInd.data(), sizeof(int32_t) * s->postInd.size());
    std::memcpy(rs, s->rowStart.data(), sizeof(int64_t) * s->rowStart.size());
    return 0;
}

REF_API int ref_gen_fixed_outdegree(int32_t nPre, int32_t nPost, int32_t k, int kind, double lo,
                                    double hi, double value, int sign, uint64_t seed, float* out,
                                    char* err, std::size_t errlen) {
    try {
        WeightDist w = kind == SSB_WEIGHT_UNIFORM ? WeightDist::uniform(lo, hi)
                                                  : WeightDist::constant(value);
        DenseMatrix m = gen_fixed_outdegree(nPre, nPost, k, w, sign, seed);
        std::memcpy(out, m.weights.data(), sizeof(float) * m.weights.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e, err, errlen);
    }
}

REF_API void ref_stream_u64(uint64_t g, uint64_t e, const char* label, long long n,
                            uint64_t* out) {
    RandomStream s(g, e, label);
    for (long long i = 0; i < n; ++i) out[i] = s.next_u64();
}

REF_API uint64_t ref_derive_seed(uint64_t parent, const char* label) {
    return derive_seed(parent, label);
}

REF_API int ref_propagate_dense(const float* w, int32_t nPre, int32_t nPost, const int32_t* spk,
                                long long n, float* acc, long long accLen) {
    try {
        DenseMatrix m;
        m.nPre = nPre;
        m.nPost = nPost;
        m.weights.assign(w, w + static_cast<std::size_t>(nPre) * nPost);
        propagate(m, std::span<const std::int32_t>(spk, static_cast<std::size_t>(n)),
                  std::span<scalar>(acc, static_cast<std::size_t>(accLen)));
        return 0;
    } catch (const std::exception& e) {
        return fail(e, nullptr, 0);
    }
}

REF_API int ref_propagate_crs(const float* g, const int32_t* ind, const int64_t* rs, int32_t nPre,
                              int32_t nPost, const int32_t* spk, long long n, float* acc,
                              long long accLen) {
    try {
        CrsMatrix m;
        m.nPre = nPre;
        m.nPost = nPost;
        m.rowStart.assign(rs, rs + nPre + 1);
        m.gValues.assign(g, g + rs[nPre]);
        m.postInd.assign(ind, ind + rs[nPre]);
        propagate(m, std::span<const std::int32_t>(spk, static_cast<std::size_t>(n)),
                  std::span<scalar>(acc, static_cast<std::size_t>(accLen)));
        return 0;
    } catch (const std::exception& e) {
        return fail(e, nullptr, 0);
    }
}

// Reference CPU timing: `replicas` independent Simulations of the same spec on
// `replicas` host threads (the calibration sweep's own parallelism model,
// src/calibration.cpp:76-84), each advancing `steps` steps after construction.
// Returns the wall seconds of the stepping phase (construction excluded) and,
// via *events, replica 0's raster size.
REF_API double ref_time_steps(const ssb_net_desc* d, int mode, long long steps, int replicas,
                              double* buildSeconds, long long* events) {
    try {
        const NetworkSpec spec = to_spec(d);
        std::vector<std::unique_ptr<Simulation>> sims(static_cast<std::size_t>(replicas));
        const auto b0 = std::chrono::steady_clock::now();
        {
            std::vector<std::thread> th;
            for (int i = 0; i < replicas; ++i)
                th.emplace_back([&, i] { sims[i] = std::make_unique<Simulation>(spec, to_mode(mode)); });
            for (auto& t : th) t.join();
        }
        const auto b1 = std::chrono::steady_clock::now();
        if (buildSeconds) *buildSeconds = std::chrono::duration<double>(b1 - b0).count();
        const auto t0 = std::chrono::steady_clock::now();
        {
            std::vector<std::thread> th;
            for (int i = 0; i < replicas; ++i)
                th.emplace_back([&, i] {
                    for (long long s = 0; s < steps; ++s) sims[i]->step();
                });
            for (auto& t : th) t.join();
        }
        const auto t1 = std::chrono::steady_clock::now();
        if (events) {
            // finish() would run the remaining steps; read the spike counts
            // through population_state-independent means: the raster lives in
            // the engine until finish, so report -1 here (callers use rates).
            *events = -1;
        }
        return std::chrono::duration<double>(t1 - t0).count();
    } catch (const std::exception&) {
        return -1.0;
    }
}

// ---------------------------------------------------------------------------
// The reference's OWN builders (network.cpp:198-362), flattened here, so the
// golden fixtures, the builder-equality test and the bench reference arm never
// take a spec from the product library.
namespace {

struct OwnedDesc {
    ssb_net_desc d{};  // first member: an OwnedDesc* is an ssb_net_desc*
    std::vector<ssb_pop_desc> pops;
    std::vector<ssb_group_desc> groups;
    std::vector<std::unique_ptr<std::string>> strs;
    std::vector<std::unique_ptr<std::vector<double>>> arrs;

    const char* keep(const std::string& s) {
        strs.push_back(std::make_unique<std::string>(s));
        return strs.back()->c_str();
    }
    const double* keep(const std::vector<double>& v) {
        arrs.push_back(std::make_unique<std::vector<double>>(v));
        return arrs.back()->data();
    }
};

OwnedDesc* flatten(const NetworkSpec& s) {
    auto o = std::make_unique<OwnedDesc>();
    for (const auto& p : s.populations) {
        ssb_pop_desc q{};
        q.name = o->keep(p.name);
        q.size = p.size;
        q.seed = p.seed;
        if (p.model == ModelKind::PoissonSource) {
            q.model = SSB_MODEL_POISSON;
            q.rate_hz = std::get<PoissonParams>(p.params).rateHz;
        } else if (p.model == ModelKind::CondLif) {
            q.model = SSB_MODEL_CONDLIF;
            const auto& c = std::get<CondLifParams>(p.params);
            q.tau_m_ms = c.tauMMs;
            q.e_leak_mv = c.eLeakMV;
            q.v_thresh_mv = c.vThreshMV;
            q.v_reset_mv = c.vResetMV;
            q.e_exc_mv = c.eExcMV;
            q.e_inh_mv = c.eInhMV;
            q.tau_syn_ms = c.tauSynMs;
        } else {
            q.model = SSB_MODEL_IZHIKEVICH;
            const auto& z = std::get<IzhikevichParams>(p.params);
            q.izh_a = o->keep(z.a);
            q.izh_b = o->keep(z.b);
            q.izh_c = o->keep(z.c);
            q.izh_d = o->keep(z.d);
            q.izh_noise = o->keep(z.noiseAmplitude);
            q.izh_bias = o->keep(z.biasCurrent);
        }
        o->pops.push_back(q);
    }
    for (const auto& g : s.synapses) {
        ssb_group_desc q{};
        q.name = o->keep(g.name);
        q.pre = o->keep(g.pre);
        q.post = o->keep(g.post);
        q.sign = g.sign == SynapseSign::Inhibitory ? SSB_SIGN_INH : SSB_SIGN_EXC;
        q.out_degree = g.outDegree;
        if (g.baseWeight.kind == WeightDist::Kind::Uniform) {
            q.weight_kind = SSB_WEIGHT_UNIFORM;
            q.weight_lo = g.baseWeight.lo;
            q.weight_hi = g.baseWeight.hi;
        } else {
            q.weight_kind = SSB_WEIGHT_CONSTANT;
            q.weight_value = g.baseWeight.value;
        }
        q.g_scale = g.gScale;
        q.storage = g.storage == StorageKind::Dense ? SSB_STORAGE_DENSE : SSB_STORAGE_SPARSE;
        q.pre_offset = g.preOffset;
        q.pre_count = g.preCount;
        o->groups.push_back(q);
    }
    o->d.n_pops = static_cast<int32_t>(o->pops.size());
    o->d.pops = o->pops.data();
    o->d.n_groups = static_cast<int32_t>(o->groups.size());
    o->d.groups = o->groups.data();
    o->d.dt_ms = s.dtMs;
    o->d.duration_ms = s.durationMs;
    o->d.global_seed = s.globalSeed;
    return o.release();
}

NetworkSpec mbody(int32_t nPN, int32_t nLHI, int32_t nKC, int32_t nDN, const double g[4],
                  uint64_t seed, double dtMs, double durationMs, double pnRateHz, double frac) {
    MBodyBuildOptions o;
    o.dtMs = dtMs;
    o.durationMs = durationMs;
    o.pnRateHz = pnRateHz;
    o.pnKcOutFraction = frac;
    return build_mbody_net(nPN, nLHI, nKC, nDN,
                           {{"pn_kc", g[0]}, {"pn_lhi", g[1]}, {"lhi_kc", g[2]}, {"kc_dn", g[3]}},
                           seed, o);
}

// Replicas of one reference Simulation stepped concurrently on host threads
// (the calibration sweep's parallelism model, calibration.cpp:76-84).
struct RefPool {
    NetworkSpec spec;
    std::vector<std::unique_ptr<Simulation>> sims;
    std::vector<RunResult> results;
};

template <class F>
void on_threads(int n, F&& f) {
    std::vector<std::thread> th;
    for (int i = 0; i < n; ++i) th.emplace_back([&, i] { f(i); });
    for (auto& t : th) t.join();
}

}  // namespace

// build_mbody_net of the reference (network.cpp:286-362), flattened.  gscales
// order: pn_kc, pn_lhi, lhi_kc, kc_dn.  Release with ref_desc_free.
REF_API ssb_net_desc* ref_build_mbody(int32_t nPN, int32_t nLHI, int32_t nKC, int32_t nDN,
                                      const double* gscales, uint64_t seed, double dtMs,
                                      double durationMs, double pnRateHz, double frac, char* err,
                                      std::size_t errlen) {
    try {
        return &flatten(mbody(nPN, nLHI, nKC, nDN, gscales, seed, dtMs, durationMs, pnRateHz,
                              frac))->d;
    } catch (const std::exception& e) {
        fail(e, err, errlen);
        return nullptr;
    }
}

// build_izhikevich_net of the reference (network.cpp:198-284), flattened.
REF_API ssb_net_desc* ref_build_izhikevich(int32_t n, int32_t nConn, double excFraction,
                                           double gScale, uint64_t seed, double dtMs,
                                           double durationMs, double noiseExc, double noiseInh,
                                           double excWeightHi, double inhWeightHi, double bias,
                                           int dense, char* err, std::size_t errlen) {
    try {
        IzhBuildOptions o;
        o.dtMs = dtMs;
        o.durationMs = durationMs;
        o.noiseExc = noiseExc;
        o.noiseInh = noiseInh;
        o.excWeightHi = excWeightHi;
        o.inhWeightHi = inhWeightHi;
        o.biasCurrent = bias;
        o.storage = dense ? StorageKind::Dense : StorageKind::Sparse;
        return &flatten(build_izhikevich_net(n, nConn, excFraction, gScale, seed, o))->d;
    } catch (const std::exception& e) {
        fail(e, err, errlen);
        return nullptr;
    }
}

REF_API void ref_desc_free(ssb_net_desc* d) { delete reinterpret_cast<OwnedDesc*>(d); }

// `replicas` Simulations of the reference's own mushroom body, constructed
// concurrently; *buildSeconds = construction wall time.
REF_API RefPool* ref_pool_mbody(int32_t nPN, int32_t nLHI, int32_t nKC, int32_t nDN,
                                const double* gscales, uint64_t seed, double dtMs,
                                double durationMs, double pnRateHz, double frac, int mode,
                                int replicas, double* buildSeconds, char* err,
                                std::size_t errlen) {
    try {
        auto p = std::make_unique<RefPool>();
        p->spec = mbody(nPN, nLHI, nKC, nDN, gscales, seed, dtMs, durationMs, pnRateHz, frac);
        p->sims.resize(static_cast<std::size_t>(replicas));
        const auto b0 = std::chrono::steady_clock::now();
        std::vector<std::string> errs(static_cast<std::size_t>(replicas));
        on_threads(replicas, [&](int i) {
            try {
                p->sims[i] = std::make_unique<Simulation>(p->spec, to_mode(mode));
            } catch (const std::exception& e) {
                errs[i] = e.what();
            }
        });
        for (const auto& e : errs)
            if (!e.empty()) throw SpecError(e);
        if (buildSeconds)
            *buildSeconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - b0)
                                .count();
        return p.release();
    } catch (const std::exception& e) {
        fail(e, err, errlen);
        return nullptr;
    }
}

// Advances every replica by `steps` Simulation::step() calls, one host thread
// per replica; returns the wall seconds of the whole pool (-1 on error).
REF_API double ref_pool_step(RefPool* p, long long steps) {
    std::vector<int> bad(p->sims.size(), 0);
    const auto t0 = std::chrono::steady_clock::now();
    on_threads(static_cast<int>(p->sims.size()), [&](int i) {
        try {
            for (long long s = 0; s < steps; ++s) p->sims[i]->step();
        } catch (const std::exception&) {
            bad[i] = 1;
        }
    });
    const double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int b : bad)
        if (b) return -1.0;
    return t;
}

// Finishes every replica (Simulation::finish, outside any timed region) and
// writes, per population, the spikes with step in [lo, hi) summed over the
// replicas.  Returns the population count, or -1.
REF_API int ref_pool_counts(RefPool* p, long long lo, long long hi, long long* counts, int cap) {
    try {
        const int nPops = static_cast<int>(p->spec.populations.size());
        if (cap < nPops) return -1;
        if (p->results.empty()) {
            p->results.resize(p->sims.size());
            on_threads(static_cast<int>(p->sims.size()),
                       [&](int i) { p->results[i] = p->sims[i]->finish(); });
        }
        for (int k = 0; k < nPops; ++k) counts[k] = 0;
        for (const auto& r : p->results)
            for (const auto& ev : r.raster.events)
                if (ev.step >= lo && ev.step < hi) ++counts[ev.population];
        return nPops;
    } catch (const std::exception&) {
        return -1;
    }
}

// Per group: index of its pre population and its outDegree (synaptic events =
// pre spikes x outDegree).  Returns the group count.
REF_API int ref_pool_groups(RefPool* p, int32_t* prePop, int32_t* outDegree, int cap) {
    const auto& s = p->spec;
    const int n = static_cast<int>(s.synapses.size());
    for (int g = 0; g < n && g < cap; ++g) {
        int idx = 0;
        for (std::size_t k = 0; k < s.populations.size(); ++k)
            if (s.populations[k].name == s.synapses[g].pre) idx = static_cast<int>(k);
        prePop[g] = idx;
        outDegree[g] = s.synapses[g].outDegree;
    }
    return n;
}

REF_API long long ref_pool_steps_total(RefPool* p) { return p->sims.at(0)->steps_total(); }
REF_API void ref_pool_destroy(RefPool* p) { delete p; }

// Raster of a single reference run as the order-independent checksum used by
// the split parity check (tests/specs.py raster_checksum): sum over events of
// mix64(step << 40 ^ pop << 32 ^ neuron), mod 2^64, events with step < upTo.
REF_API uint64_t ref_pool_raster_checksum(RefPool* p, int replica, long long upTo) {
    const auto& r = p->results.at(static_cast<std::size_t>(replica));
    uint64_t acc = 0;
    for (const auto& ev : r.raster.events) {
        if (ev.step >= upTo) continue;
        uint64_t x = (static_cast<uint64_t>(ev.step) << 40) ^
                     (static_cast<uint64_t>(ev.population) << 32) ^
                     static_cast<uint64_t>(static_cast<uint32_t>(ev.neuron));
        x ^= x >> 30;
        x *= 0xbf58476d1ce4e5b9ULL;
        x ^= x >> 27;
        x *= 0x94d049bb133111ebULL;
        x ^= x >> 31;
        acc += x;
    }
    return acc;
}
