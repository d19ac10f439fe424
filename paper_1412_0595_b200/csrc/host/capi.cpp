// capi.cpp — extern "C" boundary (include/synscale_b200.h).  Converts flat
// descriptors to the C++ model, runs everything behind try/catch and maps
// SpecError -> SSB_ERR_SPEC, anything else -> SSB_ERR_INTERNAL.
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <vector>
#include <string>

#include "../../../include/synscale_b200.h"
#include "core.hpp"

using namespace synscale;

struct ssb_sim {
    std::unique_ptr<ssb::SimCore> core;
    std::string lastError;
};

namespace {

void put(char* dst, std::size_t len, const std::string& s) {
    if (!dst || !len) return;
    std::strncpy(dst, s.c_str(), len - 1);
    dst[len - 1] = 0;
}

template <typename F>
int guarded(char* err, std::size_t errlen, F&& f) {
    try {
        f();
        return SSB_OK;
    } catch (const SpecError& e) {
        put(err, errlen, e.what());
        return SSB_ERR_SPEC;
    } catch (const std::exception& e) {
        put(err, errlen, e.what());
        return SSB_ERR_INTERNAL;
    } catch (...) {
        put(err, errlen, "unknown error");
        return SSB_ERR_INTERNAL;
    }
}

template <typename F>
int on_sim(ssb_sim* s, F&& f) {
    if (!s) return SSB_ERR_SPEC;
    char buf[1024] = {0};
    const int rc = guarded(buf, sizeof buf, [&] { f(*s->core); });
    if (rc) s->lastError = buf;
    return rc;
}

std::string str(const char* s) { return s ? std::string(s) : std::string(); }

NetworkSpec to_spec(const ssb_net_desc* d) {
    if (!d) throw SpecError("network descriptor is NULL");
    NetworkSpec spec;
    spec.dtMs = d->dt_ms;
    spec.durationMs = d->duration_ms;
    spec.globalSeed = d->global_seed;
    if (d->n_pops < 0 || d->n_groups < 0) throw SpecError("negative population or group count");
    for (int i = 0; i < d->n_pops; ++i) {
        const ssb_pop_desc& p = d->pops[i];
        NeuronPopulation np;
        np.name = str(p.name);
        np.size = p.size;
        np.seed = p.seed;
        switch (p.model) {
        case SSB_MODEL_POISSON:
            np.model = ModelKind::PoissonSource;
            np.params = PoissonParams{p.rate_hz};
            break;
        case SSB_MODEL_CONDLIF: {
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
            break;
        }
        case SSB_MODEL_TRAUBMILES: {
            np.model = ModelKind::TraubMiles;
            TraubMilesParams h;
            h.gNa = p.hh_gna;
            h.ENa = p.hh_ena;
            h.gK = p.hh_gk;
            h.EK = p.hh_ek;
            h.gl = p.hh_gl;
            h.El = p.hh_el;
            h.C = p.hh_c;
            h.eExcMV = p.e_exc_mv;
            h.eInhMV = p.e_inh_mv;
            h.tauSynMs = p.tau_syn_ms;
            h.substeps = p.hh_substeps;
            np.params = h;
            break;
        }
        case SSB_MODEL_IZHIKEVICH: {
            np.model = ModelKind::Izhikevich;
            IzhikevichParams z;
            const std::size_t n = p.size > 0 ? static_cast<std::size_t>(p.size) : 0;
            auto take = [&](const double* src, std::vector<double>& dst) {
                if (src) dst.assign(src, src + n);
            };
            take(p.izh_a, z.a);
            take(p.izh_b, z.b);
            take(p.izh_c, z.c);
            take(p.izh_d, z.d);
            take(p.izh_noise, z.noiseAmplitude);
            take(p.izh_bias, z.biasCurrent);
            np.params = std::move(z);
            break;
        }
        default: throw SpecError("population '" + np.name + "' has an unknown model kind");
        }
        spec.populations.push_back(std::move(np));
    }
    for (int i = 0; i < d->n_groups; ++i) {
        const ssb_group_desc& g = d->groups[i];
        SynapseGroupSpec s;
        s.name = str(g.name);
        s.pre = str(g.pre);
        s.post = str(g.post);
        s.sign = g.sign == SSB_SIGN_INH ? SynapseSign::Inhibitory : SynapseSign::Excitatory;
        s.outDegree = g.out_degree;
        s.baseWeight.kind = g.weight_kind == SSB_WEIGHT_UNIFORM ? WeightDist::Kind::Uniform
                                                                : WeightDist::Kind::Constant;
        s.baseWeight.lo = g.weight_lo;
        s.baseWeight.hi = g.weight_hi;
        s.baseWeight.value = g.weight_value;
        s.gScale = g.g_scale;
        s.storage = g.storage == SSB_STORAGE_DENSE ? StorageKind::Dense : StorageKind::Sparse;
        s.preOffset = g.pre_offset;
        s.preCount = g.pre_count;
        s.stdp.enabled = g.plasticity == SSB_PLASTICITY_STDP;
        s.stdp.aPlus = g.stdp_a_plus;
        s.stdp.aMinus = g.stdp_a_minus;
        s.stdp.tauPlusMs = g.stdp_tau_plus_ms;
        s.stdp.tauMinusMs = g.stdp_tau_minus_ms;
        s.stdp.wMax = g.stdp_w_max;
        if (g.plasticity != SSB_PLASTICITY_NONE && g.plasticity != SSB_PLASTICITY_STDP)
            throw SpecError("group '" + s.name + "': unknown plasticity kind");
        spec.synapses.push_back(std::move(s));
    }
    return spec;
}

// An owning descriptor: the strings and arrays live right behind the structs.
struct OwnedDesc : ssb_net_desc {
    std::vector<ssb_pop_desc> popStore;
    std::vector<ssb_group_desc> groupStore;
    std::vector<std::string> strings;
    std::vector<std::vector<double>> arrays;
};

ssb_net_desc* to_desc(const NetworkSpec& spec) {
    auto* o = new OwnedDesc();
    static_cast<ssb_net_desc&>(*o) = ssb_net_desc{};
    o->strings.reserve(spec.populations.size() + 3 * spec.synapses.size());
    o->arrays.reserve(6 * spec.populations.size());
    auto keep = [&](const std::string& s) { return o->strings.emplace_back(s).c_str(); };
    for (const auto& p : spec.populations) {
        ssb_pop_desc d{};
        d.name = keep(p.name);
        d.size = p.size;
        d.seed = p.seed;
        if (p.model == ModelKind::PoissonSource) {
            d.model = SSB_MODEL_POISSON;
            d.rate_hz = std::get<PoissonParams>(p.params).rateHz;
        } else if (p.model == ModelKind::CondLif) {
            d.model = SSB_MODEL_CONDLIF;
            const auto& c = std::get<CondLifParams>(p.params);
            d.tau_m_ms = c.tauMMs;
            d.e_leak_mv = c.eLeakMV;
            d.v_thresh_mv = c.vThreshMV;
            d.v_reset_mv = c.vResetMV;
            d.e_exc_mv = c.eExcMV;
            d.e_inh_mv = c.eInhMV;
            d.tau_syn_ms = c.tauSynMs;
        } else if (p.model == ModelKind::TraubMiles) {
            d.model = SSB_MODEL_TRAUBMILES;
            const auto& h = std::get<TraubMilesParams>(p.params);
            d.hh_gna = h.gNa;
            d.hh_ena = h.ENa;
            d.hh_gk = h.gK;
            d.hh_ek = h.EK;
            d.hh_gl = h.gl;
            d.hh_el = h.El;
            d.hh_c = h.C;
            d.e_exc_mv = h.eExcMV;
            d.e_inh_mv = h.eInhMV;
            d.tau_syn_ms = h.tauSynMs;
            d.hh_substeps = h.substeps;
        } else {
            d.model = SSB_MODEL_IZHIKEVICH;
            const auto& z = std::get<IzhikevichParams>(p.params);
            d.izh_a = o->arrays.emplace_back(z.a).data();
            d.izh_b = o->arrays.emplace_back(z.b).data();
            d.izh_c = o->arrays.emplace_back(z.c).data();
            d.izh_d = o->arrays.emplace_back(z.d).data();
            d.izh_noise = o->arrays.emplace_back(z.noiseAmplitude).data();
            d.izh_bias = o->arrays.emplace_back(z.biasCurrent).data();
        }
        o->popStore.push_back(d);
    }
    for (const auto& g : spec.synapses) {
        ssb_group_desc d{};
        d.name = keep(g.name);
        d.pre = keep(g.pre);
        d.post = keep(g.post);
        d.sign = g.sign == SynapseSign::Inhibitory ? SSB_SIGN_INH : SSB_SIGN_EXC;
        d.out_degree = g.outDegree;
        d.weight_kind =
            g.baseWeight.kind == WeightDist::Kind::Uniform ? SSB_WEIGHT_UNIFORM : SSB_WEIGHT_CONSTANT;
        d.weight_lo = g.baseWeight.lo;
        d.weight_hi = g.baseWeight.hi;
        d.weight_value = g.baseWeight.value;
        d.g_scale = g.gScale;
        d.storage = g.storage == StorageKind::Dense ? SSB_STORAGE_DENSE : SSB_STORAGE_SPARSE;
        d.pre_offset = g.preOffset;
        d.pre_count = g.preCount;
        d.plasticity = g.stdp.enabled ? SSB_PLASTICITY_STDP : SSB_PLASTICITY_NONE;
        d.stdp_a_plus = g.stdp.aPlus;
        d.stdp_a_minus = g.stdp.aMinus;
        d.stdp_tau_plus_ms = g.stdp.tauPlusMs;
        d.stdp_tau_minus_ms = g.stdp.tauMinusMs;
        d.stdp_w_max = g.stdp.wMax;
        o->groupStore.push_back(d);
    }
    o->n_pops = static_cast<int32_t>(o->popStore.size());
    o->pops = o->popStore.data();
    o->n_groups = static_cast<int32_t>(o->groupStore.size());
    o->groups = o->groupStore.data();
    o->dt_ms = spec.dtMs;
    o->duration_ms = spec.durationMs;
    o->global_seed = spec.globalSeed;
    return o;
}

ssb::EngineConfig to_config(const ssb_engine_opts* o) {
    ssb::EngineConfig c;
    if (!o) return c;
    c.device = o->device;
    if (o->window > 0) c.window = o->window;
    c.blockSize = o->block_size;
    c.blockPolicy = o->block_policy;
    c.useGraphs = o->use_graphs >= 0;
    if (o->heavy_pre_threshold > 0) c.heavyPreThreshold = o->heavy_pre_threshold;
    c.rasterCapacity = o->raster_capacity;
    c.profile = o->profile != 0;
    c.forceStepMode = o->force_step_mode != 0;
    c.rank = o->rank;
    c.world = std::max(1, static_cast<int>(o->world_size));
    c.virtualWorld = o->virtual_world;
    if (o->shard_min_size > 0) c.shardMinSize = o->shard_min_size;
    c.hasCommId = o->has_comm_id != 0;
    std::memcpy(c.commId.data(), o->comm_id, 128);
    c.rasterPinnedMB = std::max(0, static_cast<int>(o->raster_pinned_mb));
    c.rasterLocal = o->raster_local != 0;
    return c;
}

// Population kinds, sizes and group endpoints of a spec (no matrices): what
// the shard plan reads.
// The host network without matrices: what plan_shards decides on (the
// storage each group gets under `mode`, its pre window and post size).
ssb::HostNet skeleton(const NetworkSpec& spec, StorageMode mode = StorageMode::FromSpec) {
    ssb::HostNet net;
    for (const auto& p : spec.populations) {
        ssb::HostPop hp;
        hp.name = p.name;
        hp.n = p.size;
        hp.kind = p.model == ModelKind::TraubMiles ? ssb::kTraubMiles
                  : p.model == ModelKind::CondLif ? ssb::kCondLif
                  : p.model == ModelKind::PoissonSource ? ssb::kPoisson
                                                         : ssb::kIzhikevich;
        net.pops.push_back(hp);
    }
    auto index = [&](const std::string& n) {
        for (std::size_t i = 0; i < spec.populations.size(); ++i)
            if (spec.populations[i].name == n) return static_cast<int>(i);
        throw SpecError("unknown population '" + n + "'");
    };
    for (const auto& g : spec.synapses) {
        ssb::HostGroup hg;
        hg.name = g.name;
        hg.pre = index(g.pre);
        hg.post = index(g.post);
        hg.preOffset = g.preOffset;
        hg.preCount = group_pre_count(g, spec.populations[hg.pre].size);
        hg.nPre = hg.preCount;
        hg.nPost = spec.populations[hg.post].size;
        hg.outDegree = g.outDegree;
        hg.inhibitory = g.sign == SynapseSign::Inhibitory;
        hg.plastic = g.stdp.enabled;
        hg.dense = mode == StorageMode::ForceDense    ? true
                   : mode == StorageMode::ForceSparse ? false
                   : mode == StorageMode::Auto
                       ? static_cast<double>(g.outDegree) >= auto_dense_threshold() * hg.nPost
                       : g.storage == StorageKind::Dense;
        net.groups.push_back(hg);
    }
    return net;
}

StorageMode to_mode(int m) {
    switch (m) {
    case SSB_MODE_FROM_SPEC: return StorageMode::FromSpec;
    case SSB_MODE_FORCE_DENSE: return StorageMode::ForceDense;
    case SSB_MODE_FORCE_SPARSE: return StorageMode::ForceSparse;
    case SSB_MODE_AUTO: return StorageMode::Auto;
    }
    throw SpecError("unknown storage mode " + std::to_string(m));
}

DeviceSpec from_c(const ssb_device_spec* d) {
    if (!d) throw SpecError("device spec is NULL");
    DeviceSpec s;
    s.name = std::string(d->name, strnlen(d->name, sizeof d->name));
    s.warpSize = d->warp_size;
    s.maxWarpsPerSM = d->max_warps_per_sm;
    s.maxBlocksPerSM = d->max_blocks_per_sm;
    s.maxThreadsPerBlock = d->max_threads_per_block;
    s.sharedMemPerSM = d->shared_mem_per_sm;
    s.regsPerSM = d->regs_per_sm;
    s.regAllocUnit = d->reg_alloc_unit;
    s.sharedAllocUnit = d->shared_alloc_unit;
    return s;
}

void to_c(const DeviceSpec& s, ssb_device_spec* d) {
    std::memset(d, 0, sizeof *d);
    std::strncpy(d->name, s.name.c_str(), sizeof d->name - 1);
    d->warp_size = s.warpSize;
    d->max_warps_per_sm = s.maxWarpsPerSM;
    d->max_blocks_per_sm = s.maxBlocksPerSM;
    d->max_threads_per_block = s.maxThreadsPerBlock;
    d->shared_mem_per_sm = s.sharedMemPerSM;
    d->regs_per_sm = s.regsPerSM;
    d->reg_alloc_unit = s.regAllocUnit;
    d->shared_alloc_unit = s.sharedAllocUnit;
}

void to_c(const OccupancyResult& r, ssb_occupancy_result* o) {
    o->warps_per_block = r.warpsPerBlock;
    o->limit_warps = r.limitWarps;
    o->limit_blocks = r.limitBlocks;
    o->limit_shared = r.limitShared;
    o->limit_regs = r.limitRegs;
    o->active_blocks = r.activeBlocks;
    o->active_warps = r.activeWarps;
    o->occupancy = r.occupancy;
    o->limiter_mask = 0;
    for (Limiter l : r.limiters) o->limiter_mask |= 1 << static_cast<int>(l);
}

}  // namespace

extern "C" {

const char* ssb_version(void) { return "synscale-b200 0.2 (sm_100a)"; }

double ssb_auto_dense_threshold(void) { return synscale::auto_dense_threshold(); }

int ssb_device_count(void) { return ssb::device_count(); }

int ssb_validate(const ssb_net_desc* net, char* out, size_t outlen) {
    try {
        const auto v = validate(to_spec(net));
        std::string s;
        for (const auto& x : v) s += x.field + ": " + x.message + "\n";
        put(out, outlen, s);
        return static_cast<int>(v.size());
    } catch (const std::exception& e) {
        put(out, outlen, e.what());
        return -1;
    }
}

int ssb_build_mbody(int32_t n_pn, int32_t n_lhi, int32_t n_kc, int32_t n_dn,
                    const double gscales[4], uint64_t seed, const ssb_mbody_opts* opts,
                    ssb_net_desc** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        MBodyBuildOptions o;
        if (opts) {
            o.dtMs = opts->dt_ms;
            o.durationMs = opts->duration_ms;
            o.pnRateHz = opts->pn_rate_hz;
            o.pnKcOutFraction = opts->pn_kc_out_fraction;
            o.lif.tauMMs = opts->tau_m_ms;
            o.lif.eLeakMV = opts->e_leak_mv;
            o.lif.vThreshMV = opts->v_thresh_mv;
            o.lif.vResetMV = opts->v_reset_mv;
            o.lif.eExcMV = opts->e_exc_mv;
            o.lif.eInhMV = opts->e_inh_mv;
            o.lif.tauSynMs = opts->tau_syn_ms;
            o.pnKcWeightHi = opts->pn_kc_weight_hi;
            o.pnLhiWeight = opts->pn_lhi_weight;
            o.lhiKcWeight = opts->lhi_kc_weight;
            o.kcDnWeight = opts->kc_dn_weight;
            if (opts->kc_model == SSB_MODEL_TRAUBMILES) {
                o.kcModel = ModelKind::TraubMiles;
                o.kcHH.gNa = opts->hh_gna;
                o.kcHH.ENa = opts->hh_ena;
                o.kcHH.gK = opts->hh_gk;
                o.kcHH.EK = opts->hh_ek;
                o.kcHH.gl = opts->hh_gl;
                o.kcHH.El = opts->hh_el;
                o.kcHH.C = opts->hh_c;
                o.kcHH.eExcMV = opts->e_exc_mv;
                o.kcHH.eInhMV = opts->hh_e_inh_mv;
                o.kcHH.tauSynMs = opts->kc_tau_syn_ms;
                o.kcHH.substeps = opts->hh_substeps;
            } else if (opts->kc_model != SSB_MODEL_CONDLIF) {
                throw SpecError("kc_model must be SSB_MODEL_CONDLIF or SSB_MODEL_TRAUBMILES");
            }
        }
        std::map<std::string, double> gs;
        if (gscales) {
            gs["pn_kc"] = gscales[0];
            gs["pn_lhi"] = gscales[1];
            gs["lhi_kc"] = gscales[2];
            gs["kc_dn"] = gscales[3];
        }
        *out = to_desc(build_mbody_net(n_pn, n_lhi, n_kc, n_dn, gs, seed, o));
    });
}

int ssb_build_izhikevich(int32_t n_neurons, int32_t n_conn, double exc_fraction, double g_scale,
                         uint64_t seed, const ssb_izh_opts* opts, ssb_net_desc** out, char* err,
                         size_t errlen) {
    return guarded(err, errlen, [&] {
        IzhBuildOptions o;
        if (opts) {
            o.dtMs = opts->dt_ms;
            o.durationMs = opts->duration_ms;
            o.noiseExc = opts->noise_exc;
            o.noiseInh = opts->noise_inh;
            o.excWeightHi = opts->exc_weight_hi;
            o.inhWeightHi = opts->inh_weight_hi;
            o.biasCurrent = opts->bias_current;
            o.storage = opts->storage == SSB_STORAGE_DENSE ? StorageKind::Dense : StorageKind::Sparse;
        }
        *out = to_desc(build_izhikevich_net(n_neurons, n_conn, exc_fraction, g_scale, seed, o));
    });
}

void ssb_net_desc_free(ssb_net_desc* net) { delete static_cast<OwnedDesc*>(net); }

void ssb_mbody_default_opts(ssb_mbody_opts* o) {
    const MBodyBuildOptions d;
    o->dt_ms = d.dtMs;
    o->duration_ms = d.durationMs;
    o->pn_rate_hz = d.pnRateHz;
    o->pn_kc_out_fraction = d.pnKcOutFraction;
    o->tau_m_ms = d.lif.tauMMs;
    o->e_leak_mv = d.lif.eLeakMV;
    o->v_thresh_mv = d.lif.vThreshMV;
    o->v_reset_mv = d.lif.vResetMV;
    o->e_exc_mv = d.lif.eExcMV;
    o->e_inh_mv = d.lif.eInhMV;
    o->tau_syn_ms = d.lif.tauSynMs;
    o->pn_kc_weight_hi = d.pnKcWeightHi;
    o->pn_lhi_weight = d.pnLhiWeight;
    o->lhi_kc_weight = d.lhiKcWeight;
    o->kc_dn_weight = d.kcDnWeight;
    o->kc_model = SSB_MODEL_CONDLIF;
    o->hh_gna = d.kcHH.gNa;
    o->hh_ena = d.kcHH.ENa;
    o->hh_gk = d.kcHH.gK;
    o->hh_ek = d.kcHH.EK;
    o->hh_gl = d.kcHH.gl;
    o->hh_el = d.kcHH.El;
    o->hh_c = d.kcHH.C;
    o->hh_e_inh_mv = d.kcHH.eInhMV;
    o->kc_tau_syn_ms = d.kcHH.tauSynMs;
    o->hh_substeps = d.kcHH.substeps;
}

void ssb_izh_default_opts(ssb_izh_opts* o) {
    const IzhBuildOptions d;
    o->dt_ms = d.dtMs;
    o->duration_ms = d.durationMs;
    o->noise_exc = d.noiseExc;
    o->noise_inh = d.noiseInh;
    o->exc_weight_hi = d.excWeightHi;
    o->inh_weight_hi = d.inhWeightHi;
    o->bias_current = d.biasCurrent;
    o->storage = d.storage == StorageKind::Dense ? SSB_STORAGE_DENSE : SSB_STORAGE_SPARSE;
}

void ssb_engine_default_opts(ssb_engine_opts* o) {
    std::memset(o, 0, sizeof *o);
    const ssb::EngineConfig c;
    o->window = c.window;
    o->use_graphs = 1;
    o->heavy_pre_threshold = c.heavyPreThreshold;
    o->world_size = 1;
    o->shard_min_size = c.shardMinSize;
}

uint64_t ssb_fnv1a64(const char* label) { return fnv1a64(str(label)); }
uint64_t ssb_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t ssb_derive_seed(uint64_t parent, const char* label) { return derive_seed(parent, str(label)); }

int ssb_stream_u64(uint64_t g, uint64_t e, const char* label, int64_t n, uint64_t* out) {
    return guarded(nullptr, 0, [&] {
        RandomStream s(g, e, str(label));
        for (int64_t i = 0; i < n; ++i) out[i] = s.next_u64();
    });
}

int ssb_gen_fixed_outdegree(int32_t n_pre, int32_t n_post, int32_t k, int32_t weight_kind,
                            double lo, double hi, double value, int32_t sign, uint64_t seed,
                            float* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        WeightDist w;
        w.kind = weight_kind == SSB_WEIGHT_UNIFORM ? WeightDist::Kind::Uniform : WeightDist::Kind::Constant;
        w.lo = lo;
        w.hi = hi;
        w.value = value;
        const DenseMatrix m = gen_fixed_outdegree(n_pre, n_post, k, w, sign, seed);
        std::memcpy(out, m.weights.data(), m.weights.size() * sizeof(float));
    });
}

int ssb_build_group(const ssb_net_desc* net, int32_t storage_mode, int32_t group,
                    int32_t* storage, int32_t* n_pre, int32_t* n_post, int64_t* nnz, float* values,
                    int32_t* post_ind, int64_t* row_start, int64_t cap, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const NetworkSpec spec = to_spec(net);
        require_valid(spec);
        if (group < 0 || group >= static_cast<int32_t>(spec.synapses.size()))
            throw SpecError("group index out of range");
        std::optional<DenseMatrix> d;
        std::optional<CrsMatrix> s;
        ssb::build_group_matrix(spec, to_mode(storage_mode), group, d, s);
        if (d) {
            *storage = SSB_STORAGE_DENSE;
            *n_pre = d->nPre;
            *n_post = d->nPost;
            *nnz = static_cast<int64_t>(d->weights.size());
            if (values) {
                if (cap < *nnz) throw SpecError("buffer too small");
                std::memcpy(values, d->weights.data(), d->weights.size() * sizeof(float));
            }
        } else {
            *storage = SSB_STORAGE_SPARSE;
            *n_pre = s->nPre;
            *n_post = s->nPost;
            *nnz = s->nnz();
            if (values) {
                if (cap < *nnz) throw SpecError("buffer too small");
                std::memcpy(values, s->gValues.data(), s->gValues.size() * sizeof(float));
                std::memcpy(post_ind, s->postInd.data(), s->postInd.size() * sizeof(int32_t));
                std::memcpy(row_start, s->rowStart.data(), s->rowStart.size() * sizeof(int64_t));
            }
        }
    });
}

int ssb_sweep(const ssb_net_desc* const* cells, int32_t n_cells, int32_t storage_mode,
              const char* target_population, int32_t parallelism, const ssb_engine_opts* opts,
              double* avg_spike, int64_t* sum_nans, int32_t* failed, char* errors,
              size_t err_stride, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (n_cells < 1) throw SpecError("sweep needs at least one cell");
        SweepRequest req;
        for (int32_t i = 0; i < n_cells; ++i) req.nConnValues.push_back(i);  // cell index
        req.gScaleValues = {0.0};
        req.targetPopulation = str(target_population);
        req.parallelism = parallelism;
        req.storage = to_mode(storage_mode);
        const ssb::EngineConfig c = to_config(opts);
        req.engine.device = c.device;
        req.engine.window = c.window;
        req.engine.blockSize = c.blockSize;
        req.engine.blockPolicy = c.blockPolicy;
        req.engine.useGraphs = c.useGraphs;
        req.engine.heavyPreThreshold = c.heavyPreThreshold;
        req.engine.rasterCapacity = c.rasterCapacity;
        const std::vector<SweepRow> rows =
            sweep([&](std::int32_t i, double) { return to_spec(cells[i]); }, req);
        for (int32_t i = 0; i < n_cells; ++i) {
            const SweepRow& r = rows[static_cast<std::size_t>(i)];
            avg_spike[i] = r.avgSpike;
            sum_nans[i] = r.sumNaNs;
            failed[i] = r.failed ? 1 : 0;
            if (errors && err_stride) {
                char* dst = errors + static_cast<std::size_t>(i) * err_stride;
                std::snprintf(dst, err_stride, "%s", r.error.c_str());
            }
        }
    });
}

int ssb_shard_plan(const ssb_net_desc* net, int32_t world, int32_t min_size, int64_t* bounds,
                   char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const NetworkSpec spec = to_spec(net);
        require_valid(spec);
        if (world < 1) throw SpecError("world must be >= 1");
        const ssb::ShardPlan plan =
            ssb::plan_shards(skeleton(spec), world, min_size > 0 ? min_size : 64);
        for (std::size_t p = 0; p < spec.populations.size(); ++p)
            for (int r = 0; r <= world; ++r)
                bounds[p * (world + 1) + r] = plan.split(static_cast<int>(p)) ? plan.bounds[p][r] : -1;
    });
}

int ssb_shard_group(const ssb_net_desc* net, int32_t storage_mode, int32_t group, int32_t world,
                    int32_t rank, int32_t min_size, int32_t* storage, int32_t* n_pre,
                    int32_t* n_post, int64_t* nnz, float* values, int32_t* post_ind,
                    int64_t* row_start, int64_t cap, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const NetworkSpec spec = to_spec(net);
        require_valid(spec);
        if (group < 0 || group >= static_cast<int32_t>(spec.synapses.size()))
            throw SpecError("group index out of range");
        if (world < 1) throw SpecError("world must be >= 1");
        ssb::HostNet skel = skeleton(spec, to_mode(storage_mode));
        const ssb::ShardPlan plan = ssb::plan_shards(skel, world, min_size > 0 ? min_size : 64);
        std::optional<DenseMatrix> d;
        std::optional<CrsMatrix> s;
        ssb::build_group_matrix(spec, to_mode(storage_mode), group, d, s);
        auto& g = skel.groups[group];
        g.dense = d.has_value();
        g.nPre = d ? d->nPre : s->nPre;
        g.nPost = d ? d->nPost : s->nPost;
        g.preCount = g.nPre;
        if (d) {
            g.W = d->weights.data();
        } else {
            g.g = s->gValues.data();
            g.ind = s->postInd.data();
            g.rowStart = s->rowStart.data();
            g.nnz = s->nnz();
        }
        ssb::ShardStore store;
        const ssb::HostNet local = ssb::shard_net(skel, plan, rank, store);
        const auto& L = local.groups[group];
        *storage = L.dense ? SSB_STORAGE_DENSE : SSB_STORAGE_SPARSE;
        *n_pre = L.nPre;
        *n_post = L.nPost;
        *nnz = L.dense ? static_cast<int64_t>(L.nPre) * L.nPost : L.nnz;
        if (!values) return;
        if (cap < *nnz) throw SpecError("buffer too small");
        if (L.dense) {
            std::memcpy(values, L.W, static_cast<std::size_t>(*nnz) * sizeof(float));
        } else {
            std::memcpy(values, L.g, static_cast<std::size_t>(*nnz) * sizeof(float));
            std::memcpy(post_ind, L.ind, static_cast<std::size_t>(*nnz) * sizeof(int32_t));
            std::memcpy(row_start, L.rowStart, (static_cast<std::size_t>(L.nPre) + 1) * sizeof(int64_t));
        }
    });
}

int ssb_comm_selftest(int32_t device, char* err, size_t errlen) {
    return guarded(err, errlen, [&] { ssb::comm_selftest(device); });
}

int ssb_comm_unique_id(uint8_t* out128, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const auto id = ssb::comm_unique_id();
        std::memcpy(out128, id.data(), 128);
    });
}

uint64_t ssb_mem_sparse_elements(uint64_t nnz, uint64_t n_post) { return mem_sparse_elements(nnz, n_post); }
uint64_t ssb_mem_dense_elements(uint64_t n_pre, uint64_t n_post) { return mem_dense_elements(n_pre, n_post); }

int ssb_propagate_dense(const float* w, int32_t n_pre, int32_t n_post, const int32_t* spikes,
                        int64_t n_spikes, float* acc, int64_t acc_len, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        DenseMatrix m;
        m.nPre = n_pre;
        m.nPost = n_post;
        if (n_pre < 0 || n_post < 0) throw SpecError("negative matrix dimensions");
        m.weights.assign(w, w + static_cast<std::size_t>(n_pre) * static_cast<std::size_t>(n_post));
        propagate(m, std::span<const std::int32_t>(spikes, static_cast<std::size_t>(n_spikes)),
                  std::span<scalar>(acc, static_cast<std::size_t>(acc_len)));
    });
}

int ssb_propagate_crs(const float* g, const int32_t* post_ind, const int64_t* row_start,
                      int32_t n_pre, int32_t n_post, const int32_t* spikes, int64_t n_spikes,
                      float* acc, int64_t acc_len, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (n_pre < 0 || n_post < 0) throw SpecError("negative matrix dimensions");
        CrsMatrix m;
        m.nPre = n_pre;
        m.nPost = n_post;
        m.rowStart.assign(row_start, row_start + n_pre + 1);
        m.gValues.assign(g, g + m.rowStart.back());
        m.postInd.assign(post_ind, post_ind + m.rowStart.back());
        propagate(m, std::span<const std::int32_t>(spikes, static_cast<std::size_t>(n_spikes)),
                  std::span<scalar>(acc, static_cast<std::size_t>(acc_len)));
    });
}

int ssb_propagate_dense_dev(const float* w, int32_t n_pre, int32_t n_post, const int32_t* spikes,
                            int32_t n_spikes, float* acc, void* stream) {
    return guarded(nullptr, 0, [&] {
        ssb::device_propagate_dense_dev(w, n_pre, n_post, spikes, n_spikes, acc, stream);
    });
}

int ssb_crs_segments_dev(const int32_t* post_ind, const int64_t* row_start, int32_t n_pre,
                         int32_t n_post, int32_t tile, int32_t* seg, void* stream) {
    return guarded(nullptr, 0, [&] {
        if (tile < 32 || tile > 1024 || tile % 32) throw SpecError("tile must be a warp multiple <= 1024");
        ssb::device_crs_segments_dev(post_ind, row_start, n_pre, n_post, tile, seg, stream);
    });
}

int ssb_propagate_crs_dev(const float* g, const int32_t* post_ind, const int32_t* seg, int32_t tile,
                          int32_t n_pre, int32_t n_post, const int32_t* spikes, int32_t n_spikes,
                          float* acc, void* stream) {
    return guarded(nullptr, 0, [&] {
        if (tile < 32 || tile > 1024 || tile % 32) throw SpecError("tile must be a warp multiple <= 1024");
        ssb::device_propagate_crs_dev(g, post_ind, seg, tile, n_pre, n_post, spikes, n_spikes, acc,
                                      stream);
    });
}

int ssb_crs_slices(const float* g, const int32_t* post_ind, const int64_t* row_start,
                   int32_t n_pre, int32_t n_post, int64_t* slice_off, int32_t* rows, float* vals,
                   int64_t cap, int64_t* needed, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (n_pre < 0 || n_post < 0 || !row_start || !slice_off || !needed)
            throw SpecError("bad CRS slice arguments");
        *needed = ssb::crs_slices(g, post_ind, row_start, n_pre, n_post, slice_off, rows, vals, cap);
    });
}

int ssb_propagate_crs_sliced_dev(const int32_t* rows, const float* vals, const int64_t* slice_off,
                                 int32_t n_pre, int32_t n_post, const int32_t* spikes,
                                 int32_t n_spikes, float* acc, void* stream) {
    return guarded(nullptr, 0, [&] {
        ssb::device_propagate_crs_sliced_dev(rows, vals, slice_off, n_pre, n_post, spikes, n_spikes,
                                             acc, stream);
    });
}

int ssb_detect_nans(int32_t model, const float* v, const float* u, const float* g_exc,
                    const float* g_inh, uint8_t* nan_flag, int64_t n, int64_t* flagged,
                    int64_t* newly, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (model != SSB_MODEL_IZHIKEVICH && model != SSB_MODEL_POISSON && model != SSB_MODEL_CONDLIF)
            throw SpecError("unknown model kind");
        std::int64_t c = 0;
        if (model != SSB_MODEL_POISSON)
            c = ssb::device_detect_nans(model == SSB_MODEL_IZHIKEVICH ? 0 : 2, v, u, g_exc, g_inh,
                                        nan_flag, n);
        if (flagged) *flagged += c;
        if (newly) *newly = c;
    });
}

int ssb_create(const ssb_net_desc* net, int32_t storage_mode, const ssb_engine_opts* opts,
               ssb_sim** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        auto s = std::make_unique<ssb_sim>();
        s->core = std::make_unique<ssb::SimCore>(to_spec(net), to_mode(storage_mode), to_config(opts));
        *out = s.release();
    });
}

void ssb_destroy(ssb_sim* sim) { delete sim; }

const char* ssb_last_error(const ssb_sim* sim) { return sim ? sim->lastError.c_str() : ""; }

int ssb_step(ssb_sim* sim, int64_t n) {
    return on_sim(sim, [&](ssb::SimCore& c) { c.step(n); });
}

int64_t ssb_steps_total(const ssb_sim* sim) { return sim ? sim->core->steps_total() : -1; }

int32_t ssb_world(const ssb_sim* sim) { return sim ? sim->core->engine().world() : 0; }

int ssb_shard_range(const ssb_sim* sim, int32_t pop, int64_t* lo, int64_t* n_local,
                    int64_t* n_global) {
    if (!sim) return SSB_ERR_SPEC;
    return on_sim(const_cast<ssb_sim*>(sim), [&](ssb::SimCore& c) {
        if (pop < 0 || pop >= c.n_pops()) throw SpecError("population index out of range");
        int l, n, g;
        c.engine().shard_range(pop, l, n, g);
        *lo = l;
        *n_local = n;
        *n_global = g;
    });
}
int64_t ssb_steps_done(const ssb_sim* sim) { return sim ? sim->core->steps_done() : -1; }

int ssb_sync(ssb_sim* sim) {
    return on_sim(sim, [&](ssb::SimCore& c) { c.engine().sync(); });
}

int ssb_pull_state(ssb_sim* sim, int32_t pop, int32_t field, void* dst, int64_t n) {
    return on_sim(sim, [&](ssb::SimCore& c) {
        if (pop < 0 || pop >= c.n_pops()) throw SpecError("population index out of range");
        if (field < SSB_FIELD_V || field > SSB_FIELD_N) throw SpecError("unknown state field");
        if (field >= SSB_FIELD_M && c.pop_model(pop) != ModelKind::TraubMiles)
            throw SpecError("gating variables m, h, n exist for Traub-Miles populations only");
        const int64_t want = field == SSB_FIELD_FLAGGED ? 1 : c.pop_size(pop);
        if (n != want)
            throw SpecError("state field holds " + std::to_string(want) + " elements, " +
                            std::to_string(n) + " requested");
        c.engine().pull(pop, field, dst, n);
    });
}

int ssb_push_state(ssb_sim* sim, int32_t pop, int32_t field, const void* src, int64_t n) {
    return on_sim(sim, [&](ssb::SimCore& c) {
        if (c.finished()) throw SpecError("simulation already finished");
        if (pop < 0 || pop >= c.n_pops()) throw SpecError("population index out of range");
        if (field < SSB_FIELD_V || field > SSB_FIELD_N) throw SpecError("unknown state field");
        if (field >= SSB_FIELD_M && c.pop_model(pop) != ModelKind::TraubMiles)
            throw SpecError("gating variables m, h, n exist for Traub-Miles populations only");
        const int64_t want = field == SSB_FIELD_FLAGGED ? 1 : c.pop_size(pop);
        if (n != want)
            throw SpecError("state field holds " + std::to_string(want) + " elements, " +
                            std::to_string(n) + " given");
        c.engine().push(pop, field, src, n);
    });
}

int ssb_group_info(const ssb_sim* sim, int32_t group, int32_t* storage, int32_t* n_pre,
                   int32_t* n_post, int64_t* nnz) {
    return on_sim(const_cast<ssb_sim*>(sim), [&](ssb::SimCore& c) {
        if (group < 0 || group >= c.n_groups()) throw SpecError("group index out of range");
        if (const auto* d = c.dense(group)) {
            *storage = SSB_STORAGE_DENSE;
            *n_pre = d->nPre;
            *n_post = d->nPost;
            *nnz = d->nnz();
        } else {
            const auto* s = c.sparse(group);
            *storage = SSB_STORAGE_SPARSE;
            *n_pre = s->nPre;
            *n_post = s->nPost;
            *nnz = s->nnz();
        }
    });
}

int ssb_group_dense(const ssb_sim* sim, int32_t group, float* w, int64_t n) {
    return on_sim(const_cast<ssb_sim*>(sim), [&](ssb::SimCore& c) {
        if (group < 0 || group >= c.n_groups()) throw SpecError("group index out of range");
        const auto* d = c.dense(group);
        if (!d) throw SpecError("group is stored sparse");
        if (n != static_cast<int64_t>(d->weights.size())) throw SpecError("wrong buffer size");
        std::memcpy(w, d->weights.data(), d->weights.size() * sizeof(float));
    });
}

int ssb_group_weights(ssb_sim* sim, int32_t group, float* w, int64_t n) {
    return on_sim(sim, [&](ssb::SimCore& c) {
        if (group < 0 || group >= c.n_groups()) throw SpecError("group index out of range");
        const auto* d = c.dense(group);
        if (!d) throw SpecError("group is stored sparse");
        if (n != static_cast<int64_t>(d->weights.size())) throw SpecError("wrong buffer size");
        if (!c.engine().pull_weights(group, w, n))
            std::memcpy(w, d->weights.data(), d->weights.size() * sizeof(float));
    });
}

int ssb_group_sparse(const ssb_sim* sim, int32_t group, float* g, int32_t* post_ind,
                     int64_t* row_start) {
    return on_sim(const_cast<ssb_sim*>(sim), [&](ssb::SimCore& c) {
        if (group < 0 || group >= c.n_groups()) throw SpecError("group index out of range");
        const auto* s = c.sparse(group);
        if (!s) throw SpecError("group is stored dense");
        std::memcpy(g, s->gValues.data(), s->gValues.size() * sizeof(float));
        std::memcpy(post_ind, s->postInd.data(), s->postInd.size() * sizeof(int32_t));
        std::memcpy(row_start, s->rowStart.data(), s->rowStart.size() * sizeof(int64_t));
    });
}

int ssb_finish(ssb_sim* sim, ssb_run_summary* out) {
    return on_sim(sim, [&](ssb::SimCore& c) {
        c.finish();
        if (out) {
            out->steps = c.steps_total();
            out->steps_done = c.steps_done();
            out->duration_ms = c.spec().durationMs;
            out->sum_nans = c.sum_nans();
            out->n_events = static_cast<int64_t>(c.neurons().size());
            out->wall_time_ms = c.wall_ms();
        }
    });
}

int ssb_result_rates(const ssb_sim* sim, double* rates, int32_t n_pops) {
    return on_sim(const_cast<ssb_sim*>(sim), [&](ssb::SimCore& c) {
        if (!c.finished()) throw SpecError("results are available after finish");
        if (n_pops != c.n_pops()) throw SpecError("wrong population count");
        if (static_cast<int>(c.rates().size()) != n_pops) throw SpecError("no rates recorded");
        for (int i = 0; i < n_pops; ++i) rates[i] = c.rates()[i];
    });
}

int64_t ssb_result_n_events(const ssb_sim* sim) {
    return sim && sim->core->finished() ? static_cast<int64_t>(sim->core->neurons().size()) : -1;
}

int ssb_result_raster(const ssb_sim* sim, int64_t* step, int32_t* pop, int32_t* neuron, int64_t cap) {
    return on_sim(const_cast<ssb_sim*>(sim), [&](ssb::SimCore& c) {
        if (!c.finished()) throw SpecError("results are available after finish");
        const auto& counts = c.counts();
        const auto& ids = c.neurons();
        if (cap < static_cast<int64_t>(ids.size())) throw SpecError("raster buffer too small");
        const std::size_t np = static_cast<std::size_t>(c.n_pops());
        std::size_t at = 0;
        for (std::size_t i = 0; i < counts.size(); ++i)
            for (int32_t k = 0; k < counts[i]; ++k, ++at) {
                step[at] = static_cast<int64_t>(i / np);
                pop[at] = static_cast<int32_t>(i % np);
                neuron[at] = ids[at];
            }
    });
}

int ssb_result_counts(const ssb_sim* sim, int32_t* counts, int64_t n) {
    return on_sim(const_cast<ssb_sim*>(sim), [&](ssb::SimCore& c) {
        if (!c.finished()) throw SpecError("results are available after finish");
        if (n != static_cast<int64_t>(c.counts().size())) throw SpecError("wrong counts length");
        std::memcpy(counts, c.counts().data(), c.counts().size() * sizeof(int32_t));
    });
}

int ssb_result_neurons(const ssb_sim* sim, int32_t* neuron, int64_t cap) {
    return on_sim(const_cast<ssb_sim*>(sim), [&](ssb::SimCore& c) {
        if (!c.finished()) throw SpecError("results are available after finish");
        if (cap < static_cast<int64_t>(c.neurons().size())) throw SpecError("buffer too small");
        std::memcpy(neuron, c.neurons().data(), c.neurons().size() * sizeof(int32_t));
    });
}

int ssb_spike_counts(ssb_sim* sim, int64_t* counts, int32_t n_pops) {
    return on_sim(sim, [&](ssb::SimCore& c) {
        if (n_pops != c.n_pops()) throw SpecError("wrong population count");
        std::vector<std::int64_t> v;
        c.engine().spike_totals(v);
        for (int i = 0; i < n_pops; ++i) counts[i] = v[i];
    });
}

int ssb_raster_drain(ssb_sim* sim, int64_t* n_events) {
    return on_sim(sim, [&](ssb::SimCore& c) {
        const std::int64_t n = c.engine().drain_raster();
        if (n_events) *n_events = n;
    });
}

int ssb_raster_drain_async(ssb_sim* sim) {
    return on_sim(sim, [&](ssb::SimCore& c) { c.engine().drain_raster(false); });
}

int ssb_raster_discard(ssb_sim* sim) {
    return on_sim(sim, [&](ssb::SimCore& c) { c.engine().discard_raster(); });
}

void* ssb_stream(ssb_sim* sim) { return sim ? sim->core->engine().stream() : nullptr; }
int32_t ssb_window(const ssb_sim* sim) { return sim ? sim->core->engine().window() : 0; }
int32_t ssb_block_size(const ssb_sim* sim, int32_t pop) {
    if (!sim || pop < 0 || pop >= sim->core->n_pops()) return 0;
    return sim->core->engine().block_size(pop);
}

int32_t ssb_grid_size(const ssb_sim* sim, int32_t pop) {
    if (!sim || pop < 0 || pop >= sim->core->n_pops()) return 0;
    return sim->core->engine().grid_size(pop);
}

int32_t ssb_n_kernel_stats(const ssb_sim* sim) {
    return sim ? static_cast<int32_t>(const_cast<ssb_sim*>(sim)->core->engine().kernel_stats().size()) : 0;
}

int ssb_kernel_stats(ssb_sim* sim, ssb_kernel_stat* out, int32_t n) {
    return on_sim(sim, [&](ssb::SimCore& c) {
        const auto st = c.engine().kernel_stats();
        for (int32_t i = 0; i < n && i < static_cast<int32_t>(st.size()); ++i) {
            std::memset(&out[i], 0, sizeof out[i]);
            std::strncpy(out[i].name, st[i].name.c_str(), sizeof out[i].name - 1);
            out[i].launches = st[i].launches;
            out[i].total_ms = st[i].totalMs;
            out[i].bytes = st[i].bytes;
        }
    });
}

int ssb_kernel_stats_reset(ssb_sim* sim) {
    return on_sim(sim, [&](ssb::SimCore& c) { c.engine().reset_kernel_stats(); });
}

int64_t ssb_device_bytes(const ssb_sim* sim) { return sim ? sim->core->engine().device_bytes() : 0; }

int64_t ssb_kernel_launches(const ssb_sim* sim) {
    return sim ? sim->core->engine().kernel_launches() : 0;
}

int ssb_device_preset(const char* name, ssb_device_spec* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] { to_c(device_preset(str(name)), out); });
}

const char* ssb_device_preset_names(void) {
    static const std::string names = [] {
        std::string s;
        for (const auto& n : device_preset_names()) s += (s.empty() ? "" : ",") + n;
        return s;
    }();
    return names.c_str();
}

int ssb_device_query(int32_t device, ssb_device_spec* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (ssb::device_count() == 0) throw ssb::DeviceError("no CUDA device is visible");
        const auto p = ssb::device_props(device);
        DeviceSpec s = device_preset("sm100");  // allocation units are not queryable
        s.name = p.name;
        s.warpSize = p.warpSize;
        s.maxWarpsPerSM = p.maxThreadsPerSM / p.warpSize;
        s.maxBlocksPerSM = p.maxBlocksPerSM;
        s.maxThreadsPerBlock = p.maxThreadsPerBlock;
        s.sharedMemPerSM = p.sharedPerSM;
        s.regsPerSM = p.regsPerSM;
        to_c(s, out);
    });
}

int ssb_occupancy(const ssb_device_spec* dev, int64_t threads_per_block, int64_t regs_per_thread,
                  int64_t shared_per_block, ssb_occupancy_result* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        to_c(occupancy(from_c(dev), {threads_per_block, regs_per_thread, shared_per_block}), out);
    });
}

int ssb_recommend_block_size(const ssb_device_spec* dev, int64_t regs_per_thread,
                             int64_t shared_per_block, int64_t* block_size,
                             ssb_occupancy_result* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const auto [bs, r] = recommend_block_size(from_c(dev), regs_per_thread, shared_per_block);
        *block_size = bs;
        if (out) to_c(r, out);
    });
}

int ssb_kernel_attributes(const char* kernel, int32_t* regs, int32_t* shared_bytes,
                          int32_t* max_threads) {
    return guarded(nullptr, 0, [&] {
        int r = 0, s = 0, m = 0;
        if (!ssb::kernel_attributes(str(kernel), r, s, m))
            throw SpecError("unknown kernel or no device: " + str(kernel));
        *regs = r;
        *shared_bytes = s;
        *max_threads = m;
    });
}

}  // extern "C"
