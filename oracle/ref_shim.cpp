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
