// sweep.cpp — the calibration sweep, the hot path's direct caller (SURVEY.md
// §8(f) F3).  Contract of reference calibration.hpp:12-42 / calibration.cpp:16-86:
// the grid is the sorted, de-duplicated nConn x gScale product; one row per
// cell in (nConn, gScale) order; a cell that fails to build or run is recorded
// in its row (NaN rate, sumNaNs -1) and the sweep goes on; onCell runs after
// every finished cell, serialised.
//
// B200 design: cells are device simulations driven round-robin from ONE host
// thread instead of one thread per cell.  Up to `parallelism` cells are in
// flight; each pass of the driver advances every in-flight cell by a slice of
// steps (the engine enqueues its window graphs on the cell's own streams and
// returns), so the in-flight cells' kernels share the SMs while the next
// cells' specs are built on host threads ahead of time.
#include <cmath>
#include <deque>
#include <future>
#include <limits>
#include <mutex>
#include <set>

#include "synscale/synscale.hpp"

namespace synscale {

namespace {

constexpr std::int64_t kSliceSteps = 4096;  // steps per cell per driver pass

struct LiveCell {
    std::size_t row;
    std::unique_ptr<Simulation> sim;
    std::int64_t stepsLeft;
};

void check_request(const TemplateBuilder& builder, const SweepRequest& req) {
    if (!builder) throw SpecError("sweep needs a network builder");
    if (req.nConnValues.empty()) throw SpecError("sweep needs at least one nConn value");
    if (req.gScaleValues.empty()) throw SpecError("sweep needs at least one gScale value");
    if (req.targetPopulation.empty()) throw SpecError("sweep needs a target population name");
    for (double g : req.gScaleValues)
        if (!std::isfinite(g)) throw SpecError("sweep gScale values must be finite");
}

}  // namespace

std::vector<SweepRow> sweep(const TemplateBuilder& builder, const SweepRequest& req) {
    check_request(builder, req);
    const std::set<std::int32_t> nGrid(req.nConnValues.begin(), req.nConnValues.end());
    const std::set<double> gGrid(req.gScaleValues.begin(), req.gScaleValues.end());
    std::vector<SweepRow> rows;
    for (std::int32_t n : nGrid)
        for (double g : gGrid) rows.push_back(SweepRow{n, g, 0.0, 0, false, {}});
    const std::size_t total = rows.size();
    const std::size_t width = static_cast<std::size_t>(std::max(1, req.parallelism));

    // host-side spec construction runs `2 * width` cells ahead of the driver
    std::vector<std::future<NetworkSpec>> specs(total);
    std::size_t specsIssued = 0;
    auto issue_specs = [&](std::size_t upTo) {
        for (; specsIssued < std::min(upTo, total); ++specsIssued) {
            const SweepRow& r = rows[specsIssued];
            specs[specsIssued] = std::async(std::launch::async,
                                            [&builder, n = r.nConn, g = r.gScale] {
                                                return builder(n, g);
                                            });
        }
    };

    std::size_t finished = 0;
    std::mutex hookLock;
    auto complete = [&](std::size_t i) {
        ++finished;
        if (req.onCell) {
            std::lock_guard<std::mutex> lk(hookLock);
            req.onCell(rows[i], finished, total);
        }
    };
    auto fail = [&](std::size_t i, const std::exception& e) {
        rows[i].failed = true;
        rows[i].error = e.what();
        rows[i].avgSpike = std::numeric_limits<double>::quiet_NaN();
        rows[i].sumNaNs = -1;
        complete(i);
    };

    std::deque<LiveCell> live;
    std::size_t nextRow = 0;
    auto admit = [&] {
        while (live.size() < width && nextRow < total) {
            const std::size_t i = nextRow++;
            issue_specs(i + 2 * width);
            try {
                NetworkSpec spec = specs[i].get();
                if (!spec.find_population(req.targetPopulation))
                    throw SpecError("network has no population named '" + req.targetPopulation +
                                    "'");
                auto sim = std::make_unique<Simulation>(spec, req.storage, req.engine);
                const std::int64_t n = sim->steps_total();
                live.push_back(LiveCell{i, std::move(sim), n});
            } catch (const std::exception& e) {
                fail(i, e);
            }
        }
    };

    admit();
    while (!live.empty()) {
        for (auto it = live.begin(); it != live.end();) {
            SweepRow& row = rows[it->row];
            try {
                const std::int64_t k = std::min(kSliceSteps, it->stepsLeft);
                if (k > 0) it->sim->step(k);
                it->stepsLeft -= k;
                if (it->stepsLeft > 0) {
                    ++it;
                    continue;
                }
                const RunResult res = it->sim->finish();
                row.avgSpike = res.avgSpike.at(req.targetPopulation);
                row.sumNaNs = res.sumNaNs;
                complete(it->row);
            } catch (const std::exception& e) {
                fail(it->row, e);
            }
            it = live.erase(it);
        }
        admit();
    }
    return rows;
}

}  // namespace synscale
