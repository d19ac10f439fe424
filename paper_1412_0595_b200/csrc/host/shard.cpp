// shard.cpp — multi-GPU decomposition of the step path:
// which populations are split across ranks and each rank's local network.
//
// Exactness: a post population split by contiguous neuron ranges keeps every
// (post, step) fold intact -- the fold runs over the group's spiking pre rows
// in ascending order, and each rank still sees all of them (pre populations
// are either whole on every rank, replaying identical RNG streams, or their
// spike lists are all-gathered in rank order, which is ascending global
// order).  Only the post columns are divided, so results are bit-identical
// to the unsplit network.
#include <algorithm>
#include <numeric>
#include <string>

#include "../engine.hpp"
#include "synscale/synscale.hpp"

namespace ssb {

namespace {
int round_up(int v, int u) { return (v + u - 1) / u * u; }
}  // namespace

ShardPlan plan_shards(const HostNet& net, int world, int minSize, bool force, int heavyThreshold,
                      bool pipeline) {
    ShardPlan plan;
    plan.world = std::max(1, world);
    const int np = static_cast<int>(net.pops.size());
    plan.bounds.assign(np, {});
    plan.chunk.assign(np, 0);
    plan.pipeSink.assign(np, 0);
    plan.rowSplit.assign(net.groups.size(), 0);
    if (plan.world == 1 && !force) return plan;
    // feed-forward check (the windowed schedule exchanges once per window)
    std::vector<std::vector<int>> succ(np);
    std::vector<int> indeg(np, 0);
    for (const auto& g : net.groups) {
        if (net.pops[g.post].kind == kPoisson) continue;
        if (g.pre == g.post)
            throw synscale::SpecError("multi-GPU runs need a feed-forward population graph ('" +
                                      g.name + "' is recurrent)");
        succ[g.pre].push_back(g.post);
        ++indeg[g.post];
    }
    std::vector<int> q;
    for (int i = 0; i < np; ++i)
        if (indeg[i] == 0) q.push_back(i);
    for (std::size_t h = 0; h < q.size(); ++h)
        for (int s : succ[q[h]])
            if (--indeg[s] == 0) q.push_back(s);
    if (static_cast<int>(q.size()) != np)
        throw synscale::SpecError("multi-GPU runs need a feed-forward population graph");
    const int R = plan.world;
    for (int p = 0; p < np; ++p) {
        const auto& P = net.pops[p];
        if ((P.kind != kCondLif && P.kind != kTraubMiles) || P.n < std::max(minSize, R)) continue;
        int chunk = (P.n + R - 1) / R;
        chunk = round_up(chunk, P.n >= 1024 * R ? 32 : 4);
        plan.chunk[p] = chunk;
        auto& b = plan.bounds[p];
        b.resize(R + 1);
        for (int r = 0; r <= R; ++r)
            b[r] = static_cast<int>(std::min<std::int64_t>(static_cast<std::int64_t>(r) * chunk, P.n));
    }
    // rank pipeline (ShardPlan::pipeSink): a split sink whose every input is
    // one heavy dense group per sign from a split pre population, whole pre
    // range, at most kChainMaxPost (128) columns in 16-byte rows
    if (R > 1 && pipeline) {
        for (int p = 0; p < np; ++p) {
            if (!plan.split(p)) continue;
            bool ok = true, any = false;
            int perSign[2] = {0, 0};
            for (std::size_t gi = 0; gi < net.groups.size() && ok; ++gi) {
                const auto& g = net.groups[gi];
                if (g.pre == p) ok = false;  // not a sink
                if (g.post != p) continue;
                any = true;
                const auto& pre = net.pops[g.pre];
                ok = ok && g.dense && !g.plastic && plan.split(g.pre) && g.pre != p &&
                     g.preOffset == 0 && g.preCount == pre.n && pre.n >= heavyThreshold &&
                     g.nPost % 4 == 0 && g.nPost <= 128 && ++perSign[g.inhibitory ? 1 : 0] == 1;
            }
            if (!ok || !any) continue;
            plan.pipeSink[p] = 1;
            plan.chunk[p] = net.pops[p].n;  // rank 0 owns the whole population
            auto& b = plan.bounds[p];
            b.assign(R + 1, net.pops[p].n);
            b[0] = 0;
            for (std::size_t gi = 0; gi < net.groups.size(); ++gi)
                if (net.groups[gi].post == p) plan.rowSplit[gi] = 1;
        }
    }
    return plan;
}

HostNet shard_net(const HostNet& net, const ShardPlan& plan, int rank, ShardStore& store) {
    HostNet out = net;
    bool any = false;
    for (const auto& b : plan.bounds) any = any || !b.empty();
    if (!any) return out;
    if (rank < 0 || rank >= plan.world)
        throw synscale::SpecError("rank " + std::to_string(rank) + " outside a world of " +
                                  std::to_string(plan.world));
    for (std::size_t p = 0; p < net.pops.size(); ++p) {
        if (!plan.split(static_cast<int>(p))) continue;
        auto& P = out.pops[p];
        P.nGlobal = net.pops[p].n;
        P.chunk = plan.chunk[p];
        P.lo = plan.bounds[p][rank];
        P.n = plan.bounds[p][rank + 1] - P.lo;
    }
    for (std::size_t gi = 0; gi < net.groups.size(); ++gi) {
        const auto& g = net.groups[gi];
        // (a skeleton's groups without matrices -- ssb_shard_group builds one)
        if (g.dense ? !g.W : !g.rowStart) continue;
        if (!plan.rowSplit.empty() && plan.rowSplit[gi]) {
            // this rank's own pre rows, every post column (dense, whole pre range)
            auto& G = out.groups[gi];
            const int lo = plan.bounds[g.pre][rank], hi = plan.bounds[g.pre][rank + 1];
            G.rowSplit = true;
            G.preLo = lo;
            G.nPre = G.preCount = hi - lo;
            G.preOffset = 0;
            auto& w = store.f.emplace_back(g.W + static_cast<std::size_t>(lo) * g.nPost,
                                           g.W + static_cast<std::size_t>(hi) * g.nPost);
            G.W = w.data();
            continue;
        }
        if (!plan.split(g.post)) continue;
        auto& G = out.groups[gi];
        const int lo = plan.bounds[g.post][rank], hi = plan.bounds[g.post][rank + 1];
        const int nl = hi - lo;
        G.nPost = nl;
        if (g.dense) {
            auto& w = store.f.emplace_back(static_cast<std::size_t>(g.nPre) * nl);
            for (int r = 0; r < g.nPre; ++r)
                std::copy(g.W + static_cast<std::size_t>(r) * g.nPost + lo,
                          g.W + static_cast<std::size_t>(r) * g.nPost + hi,
                          w.begin() + static_cast<std::size_t>(r) * nl);
            G.W = w.data();
        } else {
            auto& rs = store.i64.emplace_back(static_cast<std::size_t>(g.nPre) + 1, 0);
            auto& ind = store.i32.emplace_back();
            auto& val = store.f.emplace_back();
            for (int r = 0; r < g.nPre; ++r) {
                const std::int32_t* b = g.ind + g.rowStart[r];
                const std::int32_t* e = g.ind + g.rowStart[r + 1];
                const std::int32_t* a0 = std::lower_bound(b, e, lo);  // rows are sorted
                const std::int32_t* a1 = std::lower_bound(a0, e, hi);
                for (const std::int32_t* q = a0; q < a1; ++q) {
                    ind.push_back(*q - lo);
                    val.push_back(g.g[q - g.ind]);
                }
                rs[r + 1] = static_cast<std::int64_t>(ind.size());
            }
            G.ind = ind.data();
            G.g = val.data();
            G.rowStart = rs.data();
            G.nnz = static_cast<std::int64_t>(ind.size());
        }
    }
    return out;
}

}  // namespace ssb
