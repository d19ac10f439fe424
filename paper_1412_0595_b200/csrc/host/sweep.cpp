// sweep.cpp — the calibration sweep (reference calibration.cpp:16-86): every
// (nConn, gScale) grid cell built by the caller's template and run to its
// end; the hot path's direct caller.  Each cell is an
// independent device simulation with its own streams, so `parallelism` host
// threads keep that many networks in flight on the GPU at once.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <limits>
#include <mutex>
#include <thread>

#include "synscale/synscale.hpp"

namespace synscale {

std::vector<SweepRow> sweep(const TemplateBuilder& builder, const SweepRequest& req) {
    if (!builder) throw SpecError("sweep needs a network builder");
    if (req.nConnValues.empty()) throw SpecError("sweep needs at least one nConn value");
    if (req.gScaleValues.empty()) throw SpecError("sweep needs at least one gScale value");
    if (req.targetPopulation.empty()) throw SpecError("sweep needs a target population name");
    for (double g : req.gScaleValues)
        if (!std::isfinite(g)) throw SpecError("sweep gScale values must be finite");

    // the grid: duplicates collapsed, (nConn, gScale) ascending
    std::vector<std::int32_t> ns(req.nConnValues);
    std::sort(ns.begin(), ns.end());
    ns.erase(std::unique(ns.begin(), ns.end()), ns.end());
    std::vector<double> gs(req.gScaleValues);
    std::sort(gs.begin(), gs.end());
    gs.erase(std::unique(gs.begin(), gs.end()), gs.end());

    std::vector<SweepRow> rows;
    rows.reserve(ns.size() * gs.size());
    for (std::int32_t n : ns)
        for (double g : gs) {
            SweepRow r;
            r.nConn = n;
            r.gScale = g;
            rows.push_back(r);
        }

    std::atomic<std::size_t> next{0}, done{0};
    std::mutex hook;
    auto cell = [&](SweepRow& row) {
        try {
            const NetworkSpec spec = builder(row.nConn, row.gScale);
            const RunResult res = run(spec, req.storage, req.engine);
            const auto it = res.avgSpike.find(req.targetPopulation);
            if (it == res.avgSpike.end())
                throw SpecError("network has no population named '" + req.targetPopulation + "'");
            row.avgSpike = it->second;
            row.sumNaNs = res.sumNaNs;
        } catch (const std::exception& e) {  // recorded, the sweep goes on
            row.failed = true;
            row.error = e.what();
            row.avgSpike = std::numeric_limits<double>::quiet_NaN();
            row.sumNaNs = -1;
        }
    };
    auto worker = [&] {
        for (std::size_t i; (i = next.fetch_add(1)) < rows.size();) {
            cell(rows[i]);
            const std::size_t d = done.fetch_add(1) + 1;
            if (req.onCell) {
                std::lock_guard<std::mutex> lock(hook);
                req.onCell(rows[i], d, rows.size());
            }
        }
    };
    const int workers = std::max(1, req.parallelism);
    if (workers == 1) {
        worker();
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < workers; ++t) pool.emplace_back(worker);
        for (auto& t : pool) t.join();
    }
    return rows;
}

}  // namespace synscale
