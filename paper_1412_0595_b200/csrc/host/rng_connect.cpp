// rng_connect.cpp — random streams and connectivity generation.
//
// Both are inputs of the parity contract: the matrices built here must be
// byte-identical to the reference's (matrix.cpp:91-162, random.hpp:40-83),
// so every draw is consumed in the reference's order.  The row generator
// additionally emits rows directly (no dense nPre x nPost scratch), which is
// what the engine uses to build CRS groups of the 1M-neuron configs.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>

#include "connect_detail.hpp"
#include "synscale/synscale.hpp"

namespace synscale {

// ---- MT19937-64 -------------------------------------------------------------

void Mt19937_64::reseed(std::uint64_t seed) {
    s_[0] = seed;
    for (int i = 1; i < kN; ++i) {
        const std::uint64_t prev = s_[i - 1];
        s_[i] = 6364136223846793005ull * (prev ^ (prev >> 62)) + static_cast<std::uint64_t>(i);
    }
    pos_ = kN;
}

void Mt19937_64::regenerate() {
    constexpr int kM = 156;
    constexpr std::uint64_t kMatrix = 0xb5026f5aa96619e9ull;
    constexpr std::uint64_t kHi = ~std::uint64_t(0) << 31, kLo = ~kHi;
    auto mix = [&](std::uint64_t a, std::uint64_t b) {
        const std::uint64_t y = (a & kHi) | (b & kLo);
        return (y >> 1) ^ ((y & 1u) ? kMatrix : 0u);
    };
    int i = 0;
    for (; i < kN - kM; ++i) s_[i] = s_[i + kM] ^ mix(s_[i], s_[i + 1]);
    for (; i < kN - 1; ++i) s_[i] = s_[i + kM - kN] ^ mix(s_[i], s_[i + 1]);
    s_[kN - 1] = s_[kM - 1] ^ mix(s_[kN - 1], s_[0]);
    pos_ = 0;
}

std::uint64_t Mt19937_64::operator()() {
    if (pos_ >= kN) regenerate();
    std::uint64_t z = s_[pos_++];
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71d67fffeda60000ull;
    z ^= (z << 37) & 0xfff7eee000000000ull;
    return z ^ (z >> 43);
}

double RandomStream::gaussian() {
    if (cached_) {
        cached_ = false;
        return cache_;
    }
    double u1 = uniform01();
    while (u1 <= 0.0) u1 = uniform01();
    const double u2 = uniform01();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 6.283185307179586476925286766559 * u2;
    cache_ = radius * std::sin(angle);
    cached_ = true;
    return radius * std::cos(angle);
}

// ---- weights and matrices -----------------------------------------------------

WeightDist WeightDist::uniform(double lo, double hi) {
    if (!(std::isfinite(lo) && std::isfinite(hi)) || lo < 0.0 || !(lo < hi))
        throw SpecError("uniform weight range [" + std::to_string(lo) + ", " + std::to_string(hi) +
                        ") is invalid: need finite bounds with 0 <= lo < hi");
    WeightDist d;
    d.kind = Kind::Uniform;
    d.lo = lo;
    d.hi = hi;
    return d;
}

WeightDist WeightDist::constant(double value) {
    if (!std::isfinite(value) || !(value > 0.0))
        throw SpecError("constant weight " + std::to_string(value) + " is invalid: need a finite value > 0");
    WeightDist d;
    d.kind = Kind::Constant;
    d.value = value;
    return d;
}

std::int64_t DenseMatrix::nnz() const {
    return std::count_if(weights.begin(), weights.end(), [](scalar w) { return w != scalar(0); });
}

bool operator==(const DenseMatrix& a, const DenseMatrix& b) {
    return a.nPre == b.nPre && a.nPost == b.nPost && a.weights == b.weights;
}

bool operator==(const CrsMatrix& a, const CrsMatrix& b) {
    return a.nPre == b.nPre && a.nPost == b.nPost && a.rowStart == b.rowStart &&
           a.postInd == b.postInd && a.gValues == b.gValues;
}

void check_dense(const DenseMatrix& m) {
    if (m.nPre < 1 || m.nPost < 1)
        throw SpecError("dense matrix must be at least 1 x 1, got " + std::to_string(m.nPre) + " x " +
                        std::to_string(m.nPost));
    const std::size_t want = static_cast<std::size_t>(m.nPre) * static_cast<std::size_t>(m.nPost);
    if (m.weights.size() != want)
        throw SpecError("dense matrix holds " + std::to_string(m.weights.size()) +
                        " weights, nPre*nPost is " + std::to_string(want));
    for (std::size_t k = 0; k < m.weights.size(); ++k)
        if (!std::isfinite(m.weights[k]))
            throw SpecError("dense matrix weight " + std::to_string(k) + " is not finite");
}

void check_crs(const CrsMatrix& m) {
    if (m.nPre < 1 || m.nPost < 1)
        throw SpecError("sparse matrix must be at least 1 x 1, got " + std::to_string(m.nPre) + " x " +
                        std::to_string(m.nPost));
    if (m.rowStart.size() != static_cast<std::size_t>(m.nPre) + 1)
        throw SpecError("rowStart needs nPre+1 = " + std::to_string(m.nPre + 1) + " entries, has " +
                        std::to_string(m.rowStart.size()));
    if (m.rowStart.front() != 0)
        throw SpecError("rowStart must begin at 0, begins at " + std::to_string(m.rowStart.front()));
    if (m.postInd.size() != m.gValues.size())
        throw SpecError("postInd has " + std::to_string(m.postInd.size()) + " entries but gValues " +
                        std::to_string(m.gValues.size()));
    if (m.rowStart.back() != static_cast<std::int64_t>(m.gValues.size()))
        throw SpecError("rowStart ends at " + std::to_string(m.rowStart.back()) +
                        ", the nonzero count is " + std::to_string(m.gValues.size()));
    for (std::int32_t r = 0; r < m.nPre; ++r) {
        const std::int64_t b = m.rowStart[r], e = m.rowStart[r + 1];
        if (b > e) throw SpecError("rowStart decreases at row " + std::to_string(r));
        for (std::int64_t k = b; k < e; ++k) {
            const std::int32_t c = m.postInd[k];
            if (c < 0 || c >= m.nPost)
                throw SpecError("row " + std::to_string(r) + " has postInd " + std::to_string(c) +
                                " outside [0, " + std::to_string(m.nPost) + ")");
            if (k > b && c <= m.postInd[k - 1])
                throw SpecError("row " + std::to_string(r) + " postInd is not strictly increasing");
            if (m.gValues[k] == scalar(0) || !std::isfinite(m.gValues[k]))
                throw SpecError("row " + std::to_string(r) + " stores a zero or non-finite gValue");
        }
    }
}

namespace detail {

void check_outdegree_args(std::int32_t nPre, std::int32_t nPost, std::int32_t k,
                          const WeightDist& dist, int sign) {
    if (nPre < 1 || nPost < 1)
        throw SpecError("connectivity needs nPre, nPost >= 1, got " + std::to_string(nPre) + " x " +
                        std::to_string(nPost));
    if (k < 1 || k > nPost)
        throw SpecError("out-degree k=" + std::to_string(k) + " must lie in [1, nPost=" +
                        std::to_string(nPost) + "]");
    if (sign != 1 && sign != -1) throw SpecError("sign must be +1 or -1, got " + std::to_string(sign));
    if (dist.kind == WeightDist::Kind::Uniform) (void)WeightDist::uniform(dist.lo, dist.hi);
    else (void)WeightDist::constant(dist.value);
}

void OutdegreeRows::begin(std::int32_t nPre_, std::int32_t nPost_, std::int32_t k_,
                          const WeightDist& dist_, int sign_, std::uint64_t seed) {
    check_outdegree_args(nPre_, nPost_, k_, dist_, sign_);
    nPre = nPre_;
    nPost = nPost_;
    k = k_;
    dist = dist_;
    sign = sign_;
    row = 0;
    targets.emplace(seed, 0, "gen/targets");
    weights.emplace(seed, 0, "gen/weights");
    cols.resize(static_cast<std::size_t>(k));
    vals.resize(static_cast<std::size_t>(k));
    full = k == nPost;
    if (full) {
        // every target is chosen whatever the draws are; the target stream is
        // private to this generator, so skipping its draws is unobservable
        std::iota(cols.begin(), cols.end(), 0);
    } else {
        pool.resize(static_cast<std::size_t>(nPost));
        std::iota(pool.begin(), pool.end(), 0);
        swaps.resize(static_cast<std::size_t>(k));
    }
}

bool OutdegreeRows::next() {
    if (row >= nPre) return false;
    if (!full) {
        // partial Fisher-Yates over an identity pool (matrix.cpp:117-124); the
        // swaps are undone afterwards so the pool is identity for the next row
        for (std::int32_t j = 0; j < k; ++j) {
            const std::uint32_t r = targets->below(static_cast<std::uint32_t>(nPost - j));
            swaps[j] = j + static_cast<std::int32_t>(r);
            std::swap(pool[j], pool[swaps[j]]);
            cols[j] = pool[j];
        }
        for (std::int32_t j = k - 1; j >= 0; --j) std::swap(pool[j], pool[swaps[j]]);
        std::sort(cols.begin(), cols.end());
    }
    for (std::int32_t j = 0; j < k; ++j) {  // matrix.cpp:128-139, ascending post order
        scalar w;
        do {
            const double raw = dist.kind == WeightDist::Kind::Uniform
                                   ? weights->uniform(dist.lo, dist.hi)
                                   : dist.value;
            w = static_cast<scalar>(raw * sign);
            if (dist.kind == WeightDist::Kind::Constant && w == scalar(0))
                throw SpecError("constant weight " + std::to_string(dist.value) +
                                " underflows to zero in fp32");
        } while (w == scalar(0));
        vals[j] = w;
    }
    ++row;
    return true;
}

}  // namespace detail

DenseMatrix gen_fixed_outdegree(std::int32_t nPre, std::int32_t nPost, std::int32_t k,
                                const WeightDist& dist, int sign, std::uint64_t seed) {
    detail::OutdegreeRows gen;
    gen.begin(nPre, nPost, k, dist, sign, seed);
    DenseMatrix m;
    m.nPre = nPre;
    m.nPost = nPost;
    m.weights.assign(static_cast<std::size_t>(nPre) * static_cast<std::size_t>(nPost), scalar(0));
    for (std::int32_t i = 0; gen.next(); ++i) {
        scalar* dst = m.weights.data() + static_cast<std::size_t>(i) * static_cast<std::size_t>(nPost);
        for (std::int32_t j = 0; j < k; ++j) dst[gen.cols[j]] = gen.vals[j];
    }
    return m;
}

CrsMatrix to_sparse(const DenseMatrix& d) {
    check_dense(d);
    CrsMatrix s;
    s.nPre = d.nPre;
    s.nPost = d.nPost;
    s.rowStart.reserve(static_cast<std::size_t>(d.nPre) + 1);
    s.rowStart.push_back(0);
    for (std::int32_t r = 0; r < d.nPre; ++r) {
        const scalar* src = d.weights.data() + static_cast<std::size_t>(r) * static_cast<std::size_t>(d.nPost);
        for (std::int32_t c = 0; c < d.nPost; ++c)
            if (src[c] != scalar(0)) {
                s.postInd.push_back(c);
                s.gValues.push_back(src[c]);
            }
        s.rowStart.push_back(static_cast<std::int64_t>(s.gValues.size()));
    }
    return s;
}

DenseMatrix to_dense(const CrsMatrix& s) {
    check_crs(s);
    DenseMatrix d;
    d.nPre = s.nPre;
    d.nPost = s.nPost;
    d.weights.assign(static_cast<std::size_t>(s.nPre) * static_cast<std::size_t>(s.nPost), scalar(0));
    for (std::int32_t r = 0; r < s.nPre; ++r)
        for (std::int64_t k = s.rowStart[r]; k < s.rowStart[r + 1]; ++k)
            d.weights[static_cast<std::size_t>(r) * static_cast<std::size_t>(s.nPost) + s.postInd[k]] =
                s.gValues[k];
    return d;
}

std::uint64_t mem_sparse_elements(std::uint64_t nNZ, std::uint64_t nPostSynN) {
    return nNZ * 2 + nPostSynN;
}

std::uint64_t mem_dense_elements(std::uint64_t nPreSynN, std::uint64_t nPostSynN) {
    return nPreSynN * nPostSynN;
}

namespace {

void require_positive_scale(double gScale) {
    if (!(std::isfinite(gScale) && gScale > 0.0))
        throw SpecError("gScale must be finite and > 0, got " + std::to_string(gScale));
}

scalar scaled(scalar w, double gScale) {
    const scalar out = static_cast<scalar>(static_cast<double>(w) * gScale);
    if (!std::isfinite(out)) throw SpecError("gScale overflows a weight to a non-finite value");
    if (out == scalar(0))
        throw SpecError("gScale underflows a weight to zero (the sparsity pattern would change)");
    return out;
}

}  // namespace

DenseMatrix scale(const DenseMatrix& m, double gScale) {
    require_positive_scale(gScale);
    check_dense(m);
    DenseMatrix out = m;
    for (scalar& w : out.weights)
        if (w != scalar(0)) w = scaled(w, gScale);
    return out;
}

CrsMatrix scale(const CrsMatrix& m, double gScale) {
    require_positive_scale(gScale);
    check_crs(m);
    CrsMatrix out = m;
    for (scalar& w : out.gValues) w = scaled(w, gScale);
    return out;
}

}  // namespace synscale
