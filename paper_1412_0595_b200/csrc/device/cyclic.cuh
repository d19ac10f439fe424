// cyclic.cuh — windowed path for small recurrent networks (included inside
// namespace ssbk::<unnamed> by kernels.cuh).
//
// A population graph with a cycle (build_izhikevich_net's neurons -> neurons,
// reference network.cpp:198-284) has no lag to pipeline over: step t + 1's
// input needs step t's spikes of the same population.  The general engine runs
// such networks in step mode (a few dependent kernels per step).  When every
// population fits one block (<= kCycMaxN neurons, padded to whole spike
// words), one block runs a whole window instead, step by step, with only
// block barriers (reference engine.cpp:316-356 per step):
//   advance + NaN flag + threshold of every population (a neuron per thread
//     slot, state in registers; Izhikevich noise and Poisson spikes are drawn
//     for the window beforehand by gaussian_window_kernel /
//     poisson_window_kernel, in the reference's stream order);
//   the step's spike bits (shared memory and the window's bitmask rows);
//   the inputs of step t + 1: every group (spec order), every spiking pre row
//     (ascending), every entry of the row -- the contributions in exactly the
//     reference's scatter order (their enumeration index e) -- bucketed by
//     accumulator element (post neuron x sign) with a counting sort, each
//     bucket put back in e order, and folded from +0 in that order.
// Bit-identical to the reference's scatter: every accumulator element sees
// the same fp32 additions in the same order.
constexpr int kCycIzh = 0, kCycPoisson = 1, kCycLif = 2;  // PopDev::kind (engine.hpp PopKind)
constexpr int kCycThreads = 1024;
constexpr int kCycMaxN = 2048;       // padded neurons (a neuron per thread slot, two slots)
constexpr int kCycMaxAcc = 4096;     // accumulator elements (post neuron x sign)
constexpr int kCycMaxRows = 4096;    // spiking pre rows of one step over all groups
constexpr int kCycChunk = 4096;      // contributions bucketed per round
constexpr int kCycMaxPops = 6;
constexpr int kCycMaxGroups = 12;
constexpr int kCycSmem = (3 * kCycMaxAcc + 1) * 4 + (2 * kCycMaxRows + 1) * 4 + 4 * kCycChunk * 4 +
                         kCycMaxN / 8;

struct CycPop {
    PopDev P;     // state and this buffer set's bits / noise
    int base;     // first slot (a multiple of 32)
    int acc[2];   // offset of (population, sign) in the accumulator array, -1: no input
};

struct CycGroup {
    int pre, post, preOffset, preCount, dense, nPost, accBase;
    const float* W;           // dense [preCount][nPost]
    const float* g;           // CRS values
    const int* ind;           // CRS post indices
    const long long* rowPtr;  // CRS [nPre + 1]
};

struct CycDev {
    int nPops, nGroups, nPad, nAcc;
    CycPop pops[kCycMaxPops];
    CycGroup groups[kCycMaxGroups];
};

// first index q in [0, n) with off[q + 1] > e (off ascending, off[0] = 0)
__device__ __forceinline__ int cyc_row_of(const int* off, int n, int e) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= e) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__global__ void __launch_bounds__(kCycThreads, 1) cyclic_block_kernel(const CycDev* __restrict__ Dg,
                                                                      int W) {
    __shared__ CycDev D;
    __shared__ int s_scan[33];
    extern __shared__ __align__(16) int s_cyc[];
    float* s_acc = reinterpret_cast<float*>(s_cyc);           // [kCycMaxAcc]
    int* s_cnt = s_cyc + kCycMaxAcc;                          // [kCycMaxAcc]
    int* s_off = s_cnt + kCycMaxAcc;                          // [kCycMaxAcc + 1]
    int* s_rows = s_off + kCycMaxAcc + 1;                     // [kCycMaxRows]: row | group << 24
    int* s_rowOff = s_rows + kCycMaxRows;                     // [kCycMaxRows + 1]
    int* s_ea = s_rowOff + kCycMaxRows + 1;                   // [kCycChunk]: accumulator element
    float* s_ev = reinterpret_cast<float*>(s_ea + kCycChunk);  // [kCycChunk]: value
    int* s_pk = s_ea + 2 * kCycChunk;                         // [kCycChunk]: placed e
    float* s_pv = reinterpret_cast<float*>(s_ea + 3 * kCycChunk);  // [kCycChunk]: placed value
    uint32_t* s_bits = reinterpret_cast<uint32_t*>(s_ea + 4 * kCycChunk);  // [kCycMaxN / 32]
    const int t = threadIdx.x, lane = t & 31;
    {
        const int* src = reinterpret_cast<const int*>(Dg);
        int* dst = reinterpret_cast<int*>(&D);
        for (int i = t; i < static_cast<int>(sizeof(CycDev) / 4); i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const int nAcc = D.nAcc;
    // accumulators from the last window's end (the inputs of this window's first step)
    for (int p = 0; p < D.nPops; ++p)
        for (int s = 0; s < 2; ++s) {
            if (D.pops[p].acc[s] < 0) continue;
            const float* src = s ? D.pops[p].P.inhIn : D.pops[p].P.excIn;
            for (int j = t; j < D.pops[p].P.n; j += blockDim.x) s_acc[D.pops[p].acc[s] + j] = src[j];
        }
    for (int i = t; i < kCycMaxAcc; i += blockDim.x) s_cnt[i] = 0;
    // this thread's two neuron slots: population, index, state in registers
    int sp[2], sj[2];
    float v[2] = {0.f, 0.f}, u[2] = {0.f, 0.f}, gi[2] = {0.f, 0.f};
    uint32_t flag[2] = {1u, 1u}, expMax[2] = {0u, 0u}, bad = 0;
    IzhNeuron z[2] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int i = t + k * kCycThreads;
        sp[k] = -1;
        sj[k] = 0;
        for (int p = 0; p < D.nPops; ++p)
            if (i >= D.pops[p].base && i - D.pops[p].base < D.pops[p].P.n) {
                sp[k] = p;
                sj[k] = i - D.pops[p].base;
            }
        if (sp[k] < 0) continue;
        const PopDev& P = D.pops[sp[k]].P;
        const int j = sj[k];
        if (P.kind == kCycIzh) {
            v[k] = P.v[j];
            u[k] = P.u[j];
            z[k] = IzhNeuron{P.ia[j], P.ib[j], P.ic[j], P.id[j]};
            flag[k] = P.nanFlag[j] ? 1u : 0u;
        } else if (P.kind == kCycLif) {
            v[k] = P.v[j];
            u[k] = P.gExc[j];  // CondLif: u holds gExc
            gi[k] = P.gInh[j];
            flag[k] = P.nanFlag[j] ? 1u : 0u;
        }
    }
    __syncthreads();
    for (int w = 0; w < W; ++w) {
        // ---- advance, NaN flag, threshold (engine.cpp:320-326)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int i = t + k * kCycThreads;
            bool spike = false;
            if (sp[k] >= 0) {
                const CycPop& C = D.pops[sp[k]];
                const PopDev& P = C.P;
                const int j = sj[k];
                const float ex = C.acc[0] >= 0 ? s_acc[C.acc[0] + j] : 0.f;
                const float ih = C.acc[1] >= 0 ? s_acc[C.acc[1] + j] : 0.f;
                if (P.kind == kCycIzh) {
                    spike = izh_step(z[k], P.dt, P.noiseIn[(size_t)w * P.n + j], ex, ih, v[k], u[k],
                                     expMax[k]);
                } else if (P.kind == kCycLif) {
                    const LifConst lc = lif_const(P);
                    spike = lif_step<true>(lc, ex, ih, v[k], u[k], gi[k], expMax[k], bad);
                } else {  // Poisson: drawn for the window beforehand
                    spike = (P.bits[(size_t)w * P.nwords + (j >> 5)] >> (j & 31)) & 1u;
                }
            }
            const uint32_t m = __ballot_sync(kFull, spike);
            if (lane == 0 && i < D.nPad) {
                s_bits[i >> 5] = m;
                if (sp[k] >= 0) {
                    const PopDev& P = D.pops[sp[k]].P;
                    if (P.kind != kCycPoisson) P.bits[(size_t)w * P.nwords + (sj[k] >> 5)] = m;
                }
            }
        }
        __syncthreads();
        // ---- zero the accumulators; the step's spiking rows, group by group
        for (int i = t; i < nAcc; i += blockDim.x) s_acc[i] = 0.f;
        int nRows = 0;
        for (int gq = 0; gq < D.nGroups; ++gq) {
            const CycGroup& G = D.groups[gq];
            const int base = D.pops[G.pre].base + G.preOffset;
            for (int r0 = 0; r0 < G.preCount; r0 += blockDim.x) {
                const int r = r0 + t;
                const int x = base + r;
                const bool on = r < G.preCount && ((s_bits[x >> 5] >> (x & 31)) & 1u);
                int total;
                const int pos = block_exclusive_scan(on ? 1 : 0, total, s_scan);
                if (on && nRows + pos < kCycMaxRows) s_rows[nRows + pos] = r | (gq << 24);
                nRows += total;
            }
        }
        nRows = min(nRows, kCycMaxRows);  // (checked on the host: sum of preCount <= kCycMaxRows)
        // row lengths, then their prefix: the enumeration of every contribution
        for (int q = t; q < nRows; q += blockDim.x) {
            const int gq = s_rows[q] >> 24, r = s_rows[q] & 0xffffff;
            const CycGroup& G = D.groups[gq];
            s_rowOff[q] = G.dense ? G.nPost
                                  : static_cast<int>(G.rowPtr[r + 1] - G.rowPtr[r]);
        }
        __syncthreads();
        block_scan_inplace(s_rowOff, nRows, s_scan);
        const int E = s_rowOff[nRows];
        // ---- contributions, kCycChunk per round, folded in enumeration order
        for (int c0 = 0; c0 < E; c0 += kCycChunk) {
            const int cn = min(kCycChunk, E - c0);
            for (int e = t; e < cn; e += blockDim.x) {
                const int q = cyc_row_of(s_rowOff, nRows, c0 + e);
                const int gq = s_rows[q] >> 24, r = s_rows[q] & 0xffffff;
                const int m = c0 + e - s_rowOff[q];
                const CycGroup& G = D.groups[gq];
                int j;
                float val;
                if (G.dense) {
                    j = m;
                    val = __ldg(G.W + (size_t)r * G.nPost + m);
                } else {
                    const long long k = G.rowPtr[r] + m;
                    j = __ldg(G.ind + k);
                    val = __ldg(G.g + k);
                }
                const int a = G.accBase + j;
                s_ea[e] = a;
                s_ev[e] = val;
                atomicAdd(&s_cnt[a], 1);
            }
            __syncthreads();
            for (int i = t; i < nAcc; i += blockDim.x) s_off[i] = s_cnt[i];
            __syncthreads();
            block_scan_inplace(s_off, nAcc, s_scan);
            for (int i = t; i < nAcc; i += blockDim.x) s_cnt[i] = 0;  // now the placement cursor
            __syncthreads();
            for (int e = t; e < cn; e += blockDim.x) {
                const int a = s_ea[e];
                const int pos = s_off[a] + atomicAdd(&s_cnt[a], 1);
                s_pk[pos] = e;
                s_pv[pos] = s_ev[e];
            }
            __syncthreads();
            for (int a = t; a < nAcc; a += blockDim.x) {
                const int lo = s_off[a], hi = s_off[a + 1];
                if (lo == hi) continue;
                // the bucket back in enumeration order (insertion sort: buckets are small)
                for (int x = lo + 1; x < hi; ++x) {
                    const int key = s_pk[x];
                    const float val = s_pv[x];
                    int y = x - 1;
                    while (y >= lo && s_pk[y] > key) {
                        s_pk[y + 1] = s_pk[y];
                        s_pv[y + 1] = s_pv[y];
                        --y;
                    }
                    s_pk[y + 1] = key;
                    s_pv[y + 1] = val;
                }
                float acc = s_acc[a];
                for (int x = lo; x < hi; ++x) acc = __fadd_rn(acc, s_pv[x]);
                s_acc[a] = acc;
                s_cnt[a] = 0;
            }
            __syncthreads();
        }
    }
    // ---- end of window: state, the next window's first inputs, NaN flags
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        if (sp[k] < 0) continue;
        const PopDev& P = D.pops[sp[k]].P;
        const int j = sj[k];
        if (P.kind == kCycIzh) {
            P.v[j] = v[k];
            P.u[j] = u[k];
        } else if (P.kind == kCycLif) {
            P.v[j] = v[k];
            P.gExc[j] = u[k];
            P.gInh[j] = gi[k];
        } else {
            continue;
        }
        P.nanFlag[j] = static_cast<uint8_t>(flag[k] | (expMax[k] == 0x7f800000u));
        if (!flag[k] && expMax[k] == 0x7f800000u) atomicAdd(P.flagged, 1ull);
    }
    for (int p = 0; p < D.nPops; ++p)
        for (int s = 0; s < 2; ++s) {
            float* dst = s ? D.pops[p].P.inhIn : D.pops[p].P.excIn;
            for (int j = t; j < D.pops[p].P.n; j += blockDim.x)
                dst[j] = D.pops[p].acc[s] >= 0 ? s_acc[D.pops[p].acc[s] + j] : 0.f;
        }
    (void)bad;
}
