// network.cpp — spec validation and the reference network builders
// (reference network.cpp:93-362).  Validation reports every problem with a
// dotted field path; the builders reproduce the reference's population order,
// entity seeds, group order and parameter draws exactly.
#include <algorithm>
#include <cmath>
#include <set>
#include <sstream>

#include "synscale/synscale.hpp"

namespace synscale {

const NeuronPopulation* NetworkSpec::find_population(const std::string& name) const {
    for (const auto& p : populations)
        if (p.name == name) return &p;
    return nullptr;
}

std::int32_t group_pre_count(const SynapseGroupSpec& g, std::int32_t preSize) {
    return g.preCount >= 0 ? g.preCount : preSize - g.preOffset;
}

namespace {

struct Report {
    std::vector<Violation>& out;
    void add(std::string field, std::string msg) { out.push_back({std::move(field), std::move(msg)}); }
};

bool fin(double x) { return std::isfinite(x); }

void check_izh(const NeuronPopulation& p, const IzhikevichParams& z, const std::string& at,
               Report& rep) {
    const std::size_t n = static_cast<std::size_t>(p.size);
    const std::pair<const std::vector<double>*, const char*> arrays[] = {
        {&z.a, "a"}, {&z.b, "b"}, {&z.c, "c"}, {&z.d, "d"},
        {&z.noiseAmplitude, "noiseAmplitude"}, {&z.biasCurrent, "biasCurrent"}};
    for (const auto& [vec, nm] : arrays) {
        if (vec->size() != n) {
            rep.add(at + "." + nm, std::string(nm) + " holds " + std::to_string(vec->size()) +
                                       " values for a population of " + std::to_string(p.size));
            continue;
        }
        for (double x : *vec)
            if (!fin(x)) {
                rep.add(at + "." + nm, std::string(nm) + " has a non-finite entry");
                break;
            }
    }
    if (z.a.size() == n)
        for (double a : z.a)
            if (fin(a) && !(a > 0.0)) {
                rep.add(at + ".a", "every recovery rate a must be > 0");
                break;
            }
    if (z.noiseAmplitude.size() == n)
        for (double s : z.noiseAmplitude)
            if (fin(s) && s < 0.0) {
                rep.add(at + ".noiseAmplitude", "noise amplitudes must be >= 0");
                break;
            }
}

// Traub-Miles (extension, F1): finite parameters, positive capacitance and
// synaptic time constant, 1..1000 sub-steps.
void check_hh(const TraubMilesParams& h, const std::string& at, Report& rep) {
    const std::pair<double, const char*> fields[] = {
        {h.gNa, "gNa"}, {h.ENa, "ENa"}, {h.gK, "gK"}, {h.EK, "EK"}, {h.gl, "gl"},
        {h.El, "El"}, {h.C, "C"}, {h.eExcMV, "eExcMV"}, {h.eInhMV, "eInhMV"},
        {h.tauSynMs, "tauSynMs"}};
    for (const auto& [x, nm] : fields)
        if (!fin(x)) rep.add(at + "." + nm, "must be finite");
    if (fin(h.C) && !(h.C > 0.0)) rep.add(at + ".C", "membrane capacitance must be > 0");
    if (fin(h.tauSynMs) && !(h.tauSynMs > 0.0))
        rep.add(at + ".tauSynMs", "synaptic time constant must be > 0");
    if (h.substeps < 1 || h.substeps > 1000)
        rep.add(at + ".substeps", "substeps must lie in [1, 1000]");
}

void check_lif(const CondLifParams& c, const std::string& at, Report& rep) {
    const std::pair<double, const char*> fields[] = {
        {c.tauMMs, "tauMMs"}, {c.eLeakMV, "eLeakMV"}, {c.vThreshMV, "vThreshMV"},
        {c.vResetMV, "vResetMV"}, {c.eExcMV, "eExcMV"}, {c.eInhMV, "eInhMV"},
        {c.tauSynMs, "tauSynMs"}};
    for (const auto& [x, nm] : fields)
        if (!fin(x)) rep.add(at + "." + nm, "must be finite");
    if (fin(c.tauMMs) && !(c.tauMMs > 0.0)) rep.add(at + ".tauMMs", "membrane time constant must be > 0");
    if (fin(c.tauSynMs) && !(c.tauSynMs > 0.0))
        rep.add(at + ".tauSynMs", "synaptic time constant must be > 0");
    if (fin(c.vResetMV) && fin(c.vThreshMV) && !(c.vResetMV < c.vThreshMV))
        rep.add(at + ".vResetMV", "reset potential must be below threshold");
    if (fin(c.eInhMV) && fin(c.vThreshMV) && !(c.eInhMV < c.vThreshMV))
        rep.add(at + ".eInhMV", "inhibitory reversal potential must be below threshold");
    if (fin(c.eExcMV) && fin(c.vThreshMV) && !(c.eExcMV > c.vThreshMV))
        rep.add(at + ".eExcMV", "excitatory reversal potential must be above threshold");
}

std::string weight_problem(const WeightDist& w) {
    if (w.kind == WeightDist::Kind::Uniform) {
        if (!fin(w.lo) || !fin(w.hi) || w.lo < 0.0 || !(w.lo < w.hi))
            return "uniform weight range needs finite bounds with 0 <= lo < hi";
    } else if (!fin(w.value) || !(w.value > 0.0)) {
        return "constant weight must be finite and > 0";
    }
    return {};
}

}  // namespace

std::vector<Violation> validate(const NetworkSpec& spec) {
    std::vector<Violation> out;
    Report rep{out};
    if (!fin(spec.dtMs) || !(spec.dtMs > 0.0)) rep.add("dtMs", "dt must be positive and finite");
    if (!fin(spec.durationMs) || !(spec.durationMs > 0.0))
        rep.add("durationMs", "duration must be positive and finite");
    if (spec.populations.empty()) rep.add("populations", "at least one population is required");

    std::map<std::string, const NeuronPopulation*> byName;
    for (std::size_t i = 0; i < spec.populations.size(); ++i) {
        const auto& p = spec.populations[i];
        const std::string at = "populations[" + std::to_string(i) + "]";
        if (p.name.empty()) rep.add(at + ".name", "population name is empty");
        else if (!byName.emplace(p.name, &p).second)
            rep.add(at + ".name", "population name '" + p.name + "' is used twice");
        if (p.size < 1) {
            rep.add(at + ".size", "population size must be >= 1, got " + std::to_string(p.size));
            continue;
        }
        const bool ok = (p.model == ModelKind::Izhikevich &&
                         std::holds_alternative<IzhikevichParams>(p.params)) ||
                        (p.model == ModelKind::PoissonSource &&
                         std::holds_alternative<PoissonParams>(p.params)) ||
                        (p.model == ModelKind::CondLif &&
                         std::holds_alternative<CondLifParams>(p.params)) ||
                        (p.model == ModelKind::TraubMiles &&
                         std::holds_alternative<TraubMilesParams>(p.params));
        if (!ok) {
            rep.add(at + ".params", "the parameter block does not match the population model");
            continue;
        }
        if (p.model == ModelKind::Izhikevich) {
            check_izh(p, std::get<IzhikevichParams>(p.params), at, rep);
        } else if (p.model == ModelKind::PoissonSource) {
            const double r = std::get<PoissonParams>(p.params).rateHz;
            if (!fin(r) || r < 0.0) rep.add(at + ".params.rateHz", "rate must be finite and >= 0");
            else if (fin(spec.dtMs) && spec.dtMs > 0.0 && r * spec.dtMs / 1000.0 > 1.0)
                rep.add(at + ".params.rateHz",
                        "spike probability per step rate * dt is above one (p > 1)");
        } else if (p.model == ModelKind::TraubMiles) {
            check_hh(std::get<TraubMilesParams>(p.params), at + ".params", rep);
        } else {
            check_lif(std::get<CondLifParams>(p.params), at + ".params", rep);
        }
    }

    std::set<std::string> groupNames;
    for (std::size_t i = 0; i < spec.synapses.size(); ++i) {
        const auto& g = spec.synapses[i];
        const std::string at = "synapses[" + std::to_string(i) + "]";
        if (g.name.empty()) rep.add(at + ".name", "synapse group name is empty");
        else if (!groupNames.insert(g.name).second)
            rep.add(at + ".name", "synapse group name '" + g.name + "' is used twice");
        const auto pre = byName.find(g.pre), post = byName.find(g.post);
        if (pre == byName.end())
            rep.add(at + ".pre", "pre side references unknown population '" + g.pre + "'");
        if (post == byName.end())
            rep.add(at + ".post", "post side references unknown population '" + g.post + "'");
        if (pre != byName.end() && pre->second->size >= 1) {
            const std::int32_t n = pre->second->size;
            if (g.preOffset < 0 || g.preOffset >= n) {
                rep.add(at + ".preOffset",
                        "pre window offset is outside a population of " + std::to_string(n));
            } else {
                const std::int32_t cnt = group_pre_count(g, n);
                if (cnt < 1 || g.preOffset + cnt > n)
                    rep.add(at + ".preCount", "pre window [" + std::to_string(g.preOffset) + ", " +
                                                  std::to_string(g.preOffset + cnt) +
                                                  ") does not fit a population of " +
                                                  std::to_string(n));
            }
        }
        if (post != byName.end() && post->second->size >= 1) {
            const std::int32_t n = post->second->size;
            if (g.outDegree < 1 || g.outDegree > n)
                rep.add(at + ".outDegree", "out-degree " + std::to_string(g.outDegree) +
                                               " must lie in [1, " + std::to_string(n) + "]");
        }
        if (auto msg = weight_problem(g.baseWeight); !msg.empty()) rep.add(at + ".baseWeight", msg);
        if (!fin(g.gScale) || g.gScale < 0.0)
            rep.add(at + ".gScale", "gScale must be finite and >= 0, got " + std::to_string(g.gScale));
        if (g.stdp.enabled) {  // extension F2: dense all-to-all excitatory groups only
            const auto& r = g.stdp;
            if (g.storage != StorageKind::Dense)
                rep.add(at + ".stdp", "a plastic group must be stored dense");
            if (g.sign != SynapseSign::Excitatory)
                rep.add(at + ".stdp", "a plastic group must be excitatory");
            if (post != byName.end() && g.outDegree != post->second->size)
                rep.add(at + ".stdp", "a plastic group must be all-to-all (outDegree = post size)");
            if (!fin(r.aPlus) || r.aPlus < 0.0 || !fin(r.aMinus) || r.aMinus < 0.0)
                rep.add(at + ".stdp", "aPlus and aMinus must be finite and >= 0");
            if (!fin(r.tauPlusMs) || r.tauPlusMs <= 0.0 || !fin(r.tauMinusMs) || r.tauMinusMs <= 0.0)
                rep.add(at + ".stdp", "trace time constants must be finite and > 0");
            if (!fin(r.wMax) || r.wMax <= 0.0)
                rep.add(at + ".stdp", "wMax must be finite and > 0");
        }
    }
    return out;
}

void require_valid(const NetworkSpec& spec) {
    const auto v = validate(spec);
    if (v.empty()) return;
    std::ostringstream os;
    os << "invalid network spec, " << v.size() << (v.size() == 1 ? " problem:" : " problems:");
    for (const auto& x : v) os << "\n  " << x.field << ": " << x.message;
    throw SpecError(os.str());
}

// build_izhikevich_net (reference network.cpp:198-284)
NetworkSpec build_izhikevich_net(std::int32_t nNeurons, std::int32_t nConn, double excFraction,
                                 double gScale, std::uint64_t seed, const IzhBuildOptions& opt) {
    if (nNeurons < 2) throw SpecError("nNeurons must be >= 2, got " + std::to_string(nNeurons));
    if (!(excFraction > 0.0 && excFraction < 1.0))
        throw SpecError("excFraction must be inside (0, 1), got " + std::to_string(excFraction));
    if (!std::isfinite(gScale) || gScale < 0.0)
        throw SpecError("gScale must be finite and >= 0, got " + std::to_string(gScale));
    if (nConn < 1 || nConn > nNeurons)
        throw SpecError("nConn=" + std::to_string(nConn) + " must lie in [1, nNeurons=" +
                        std::to_string(nNeurons) + "]");
    const auto nExc = static_cast<std::int32_t>(std::floor(excFraction * nNeurons));
    const std::int32_t nInh = nNeurons - nExc;
    if (nExc < 1 || nInh < 1)
        throw SpecError("excFraction " + std::to_string(excFraction) + " leaves no " +
                        (nExc < 1 ? "excitatory" : "inhibitory") + " neurons out of " +
                        std::to_string(nNeurons));

    NeuronPopulation pop;
    pop.name = "neurons";
    pop.size = nNeurons;
    pop.model = ModelKind::Izhikevich;
    pop.seed = 1;
    IzhikevichParams z;
    const std::size_t n = static_cast<std::size_t>(nNeurons);
    z.a.resize(n);
    z.b.resize(n);
    z.c.resize(n);
    z.d.resize(n);
    z.noiseAmplitude.resize(n);
    z.biasCurrent.assign(n, opt.biasCurrent);
    RandomStream draw(seed, pop.seed, "neurons/params");
    for (std::int32_t i = 0; i < nNeurons; ++i) {
        const double r = draw.uniform01();
        if (i < nExc) {  // regular spiking, skewed by r^2
            z.a[i] = 0.02;
            z.b[i] = 0.2;
            z.c[i] = -65.0 + 15.0 * r * r;
            z.d[i] = 8.0 - 6.0 * r * r;
            z.noiseAmplitude[i] = opt.noiseExc;
        } else {  // fast spiking .. low-threshold spiking
            z.a[i] = 0.02 + 0.08 * r;
            z.b[i] = 0.25 - 0.05 * r;
            z.c[i] = -65.0;
            z.d[i] = 2.0;
            z.noiseAmplitude[i] = opt.noiseInh;
        }
    }
    pop.params = std::move(z);

    NetworkSpec spec;
    spec.populations.push_back(std::move(pop));
    spec.dtMs = opt.dtMs;
    spec.durationMs = opt.durationMs;
    spec.globalSeed = seed;
    auto group = [&](const char* name, SynapseSign sign, double hi, std::int32_t off,
                     std::int32_t cnt) {
        SynapseGroupSpec g;
        g.name = name;
        g.pre = g.post = "neurons";
        g.sign = sign;
        g.outDegree = nConn;
        g.baseWeight = WeightDist::uniform(0.0, hi);
        g.gScale = gScale;
        g.storage = opt.storage;
        g.preOffset = off;
        g.preCount = cnt;
        return g;
    };
    spec.synapses.push_back(group("exc", SynapseSign::Excitatory, opt.excWeightHi, 0, nExc));
    spec.synapses.push_back(group("inh", SynapseSign::Inhibitory, opt.inhWeightHi, nExc, nInh));
    return spec;
}

// build_mbody_net (reference network.cpp:286-362)
NetworkSpec build_mbody_net(std::int32_t nPN, std::int32_t nLHI, std::int32_t nKC, std::int32_t nDN,
                            const std::map<std::string, double>& gScales, std::uint64_t seed,
                            const MBodyBuildOptions& opt) {
    const std::pair<std::int32_t, const char*> sizes[] = {
        {nPN, "nPN"}, {nLHI, "nLHI"}, {nKC, "nKC"}, {nDN, "nDN"}};
    for (const auto& [n, nm] : sizes)
        if (n < 1) throw SpecError(std::string(nm) + " must be >= 1, got " + std::to_string(n));
    static const char* const kGroups[] = {"pn_kc", "pn_lhi", "lhi_kc", "kc_dn"};
    for (const auto& [name, g] : gScales) {
        (void)g;
        if (std::find(std::begin(kGroups), std::end(kGroups), name) == std::end(kGroups))
            throw SpecError("gScales names an unknown synapse group '" + name +
                            "' (expected pn_kc, pn_lhi, lhi_kc, kc_dn)");
    }
    auto scaleOf = [&](const char* name) {
        const auto it = gScales.find(name);
        if (it == gScales.end())
            throw SpecError("gScales has no entry for synapse group '" + std::string(name) +
                            "' (required: pn_kc, pn_lhi, lhi_kc, kc_dn)");
        if (!std::isfinite(it->second) || it->second < 0.0)
            throw SpecError("gScales['" + std::string(name) + "'] must be finite and >= 0");
        return it->second;
    };

    NetworkSpec spec;
    spec.dtMs = opt.dtMs;
    spec.durationMs = opt.durationMs;
    spec.globalSeed = seed;
    NeuronPopulation pn;
    pn.name = "pn";
    pn.size = nPN;
    pn.model = ModelKind::PoissonSource;
    pn.seed = 1;
    pn.params = PoissonParams{opt.pnRateHz};
    spec.populations.push_back(std::move(pn));
    const std::pair<const char*, std::int32_t> lif[] = {{"lhi", nLHI}, {"kc", nKC}, {"dn", nDN}};
    std::uint64_t entity = 2;
    for (const auto& [name, n] : lif) {
        NeuronPopulation p;
        p.name = name;
        p.size = n;
        p.model = ModelKind::CondLif;
        p.seed = entity++;
        p.params = opt.lif;
        if (std::string(name) == "kc" && opt.kcModel == ModelKind::TraubMiles) {
            p.model = ModelKind::TraubMiles;  // extension: HH KCs (F1)
            p.params = opt.kcHH;
        }
        spec.populations.push_back(std::move(p));
    }
    const auto kcFan =
        std::max<std::int32_t>(1, static_cast<std::int32_t>(std::lround(opt.pnKcOutFraction * nKC)));
    auto group = [](const char* name, const char* pre, const char* post, SynapseSign sign,
                    std::int32_t k, WeightDist w, double g, StorageKind st) {
        SynapseGroupSpec s;
        s.name = name;
        s.pre = pre;
        s.post = post;
        s.sign = sign;
        s.outDegree = k;
        s.baseWeight = w;
        s.gScale = g;
        s.storage = st;
        return s;
    };
    spec.synapses.push_back(group("pn_kc", "pn", "kc", SynapseSign::Excitatory, kcFan,
                                  WeightDist::uniform(0.0, opt.pnKcWeightHi), scaleOf("pn_kc"),
                                  StorageKind::Sparse));
    spec.synapses.push_back(group("pn_lhi", "pn", "lhi", SynapseSign::Excitatory, nLHI,
                                  WeightDist::constant(opt.pnLhiWeight), scaleOf("pn_lhi"),
                                  StorageKind::Dense));
    spec.synapses.push_back(group("lhi_kc", "lhi", "kc", SynapseSign::Inhibitory, nKC,
                                  WeightDist::constant(opt.lhiKcWeight), scaleOf("lhi_kc"),
                                  StorageKind::Dense));
    spec.synapses.push_back(group("kc_dn", "kc", "dn", SynapseSign::Excitatory, nDN,
                                  WeightDist::constant(opt.kcDnWeight), scaleOf("kc_dn"),
                                  StorageKind::Dense));
    return spec;
}

}  // namespace synscale
