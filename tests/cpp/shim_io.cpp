// shim_io.cpp — TEST INFRASTRUCTURE ONLY.  The reference's unit tests compare
// two specs with network_to_json(a) == network_to_json(b)
// (test_network.cpp:77, 147); spec JSON I/O is out of this tier's scope
// (SURVEY.md §2), so the test binaries get a canonical dump of every field
// instead, which is exactly as strict for equality.
#include <cstdio>
#include <sstream>
#include <string>

#include "synscale/synscale.hpp"

namespace synscale {

namespace {
std::string num(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}
void arr(std::ostringstream& os, const std::vector<double>& v) {
    os << '[';
    for (double x : v) os << num(x) << ',';
    os << ']';
}
}  // namespace

std::string network_to_json(const NetworkSpec& s) {
    std::ostringstream os;
    os << "dt=" << num(s.dtMs) << " dur=" << num(s.durationMs) << " seed=" << s.globalSeed << '\n';
    for (const auto& p : s.populations) {
        os << "pop " << p.name << ' ' << p.size << ' ' << static_cast<int>(p.model) << ' '
           << p.seed << ' ';
        if (const auto* q = std::get_if<PoissonParams>(&p.params)) os << num(q->rateHz);
        if (const auto* c = std::get_if<CondLifParams>(&p.params))
            os << num(c->tauMMs) << num(c->eLeakMV) << num(c->vThreshMV) << num(c->vResetMV)
               << num(c->eExcMV) << num(c->eInhMV) << num(c->tauSynMs);
        if (const auto* z = std::get_if<IzhikevichParams>(&p.params)) {
            arr(os, z->a);
            arr(os, z->b);
            arr(os, z->c);
            arr(os, z->d);
            arr(os, z->noiseAmplitude);
            arr(os, z->biasCurrent);
        }
        os << '\n';
    }
    for (const auto& g : s.synapses)
        os << "syn " << g.name << ' ' << g.pre << ' ' << g.post << ' ' << static_cast<int>(g.sign)
           << ' ' << g.outDegree << ' ' << static_cast<int>(g.baseWeight.kind) << ' '
           << num(g.baseWeight.lo) << ' ' << num(g.baseWeight.hi) << ' '
           << num(g.baseWeight.value) << ' ' << num(g.gScale) << ' '
           << static_cast<int>(g.storage) << ' ' << g.preOffset << ' ' << g.preCount << '\n';
    return os.str();
}

}  // namespace synscale
