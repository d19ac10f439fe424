// connect_detail.hpp — row-at-a-time fixed-out-degree generator shared by
// gen_fixed_outdegree() and the engine's connectivity build.
#pragma once

#include <optional>
#include <vector>

#include "synscale/synscale.hpp"

namespace synscale::detail {

void check_outdegree_args(std::int32_t nPre, std::int32_t nPost, std::int32_t k,
                          const WeightDist& dist, int sign);

// Produces the rows of gen_fixed_outdegree in order: after each next(),
// cols[0..k) holds the ascending targets and vals[0..k) their weights.
struct OutdegreeRows {
    std::int32_t nPre = 0, nPost = 0, k = 0, row = 0;
    int sign = 1;
    bool full = false;
    WeightDist dist;
    std::optional<RandomStream> targets, weights;
    std::vector<std::int32_t> cols, pool, swaps;
    std::vector<scalar> vals;

    void begin(std::int32_t nPre, std::int32_t nPost, std::int32_t k, const WeightDist& dist,
               int sign, std::uint64_t seed);
    bool next();
};

}  // namespace synscale::detail
