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
//     for the window beforehand by gaussian_draw/transform_kernel and
//     poisson_window_kernel, in the reference's stream order);
//   the step's spike bits (shared memory and the window's bitmask rows);
//   the inputs of step t + 1, group by group in spec order: every post folds
//     the group's spiking rows in ascending order (the reference's scatter
//     order per post); CRS groups are expanded to dense rows on the host
//     (absent entries +0.0f; the block's populations bound them to
//     kCycMaxN^2 weights), so a post reads one coalesced word per row.
// Bit-identical to the reference's scatter: every accumulator element sees
// the same fp32 additions in the same order (an added +0.0f leaves a fold
// that started at +0.0f unchanged: it never holds -0.0f).
constexpr int kCycIzh = 0, kCycPoisson = 1, kCycLif = 2;  // PopDev::kind (engine.hpp PopKind)
constexpr int kCycThreads = 1024;
constexpr int kCycMaxN = 2048;       // padded neurons (a neuron per thread slot, two slots)
constexpr int kCycMaxAcc = 4096;     // accumulator elements (post neuron x sign)
constexpr int kCycMaxRows = kCycMaxN;  // spiking pre rows of one group and step
constexpr int kCycMaxPops = 6;
constexpr int kCycMaxGroups = 12;
constexpr int kCycSmem = kCycMaxAcc * 4 + kCycMaxRows * 4 + kCycMaxN / 8;

struct CycPop {
    PopDev P;     // state and this buffer set's bits / noise
    int base;     // first slot (a multiple of 32)
    int acc[2];   // offset of (population, sign) in the accumulator array, -1: no input
};

struct CycGroup {
    int pre, post, preOffset, preCount, nPost, accBase;
    const float* W;  // dense rows [preCount][nPost] (CRS groups expanded, absent entries +0.0f)
};

struct CycDev {
    int nPops, nGroups, nPad, nAcc;
    CycPop pops[kCycMaxPops];
    CycGroup groups[kCycMaxGroups];
};

__global__ void __launch_bounds__(kCycThreads, 1) cyclic_block_kernel(const CycDev* __restrict__ Dg,
                                                                      int W) {
    __shared__ CycDev D;
    __shared__ int s_scan[33];
    __shared__ int s_gStart[kCycMaxGroups + 1];  // a wave's groups: first row of each in s_rows
    extern __shared__ __align__(16) int s_cyc[];
    float* s_acc = reinterpret_cast<float*>(s_cyc);                      // [kCycMaxAcc]
    int* s_rows = s_cyc + kCycMaxAcc;                                    // [kCycMaxRows]
    uint32_t* s_bits = reinterpret_cast<uint32_t*>(s_rows + kCycMaxRows);  // [kCycMaxN / 32]
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
    // this thread's two neuron slots: population, index, state in registers
    int sp[2], sj[2];
    float v[2] = {0.f, 0.f}, u[2] = {0.f, 0.f}, gi[2] = {0.f, 0.f};
    uint32_t flag[2] = {1u, 1u}, expMax[2] = {0u, 0u}, bad = 0;
    IzhNeuron z[2] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    float nzNext[2] = {0.f, 0.f};
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
            if (W > 0) nzNext[k] = __ldg(P.noiseIn + j);
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
                    const float nz = nzNext[k];  // loaded a step ahead
                    if (w + 1 < W) nzNext[k] = __ldg(P.noiseIn + (size_t)(w + 1) * P.n + j);
                    spike = izh_step(z[k], P.dt, nz, ex, ih, v[k], u[k], expMax[k]);
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
        // ---- zero the accumulators, then every group's contributions in spec
        //      order (engine.cpp:341-355), each folded into its accumulators
        for (int i = t; i < nAcc; i += blockDim.x) s_acc[i] = 0.f;
        // groups in waves: consecutive groups (spec order) into distinct
        // accumulators fold at once (a group into the same accumulator as an
        // earlier one waits for the next wave); one ordered compaction of all
        // the wave's candidate rows
        for (int g0 = 0; g0 < D.nGroups;) {
            int g1 = g0, cand = 0;
            while (g1 < D.nGroups) {
                const CycGroup& G = D.groups[g1];
                bool clash = cand + G.preCount > kCycMaxRows && g1 > g0;
                for (int h = g0; h < g1 && !clash; ++h)
                    clash = D.groups[h].accBase >= 0 && D.groups[h].accBase == G.accBase;
                if (clash) break;
                cand += G.preCount;
                ++g1;
            }
            // the wave's spiking rows: group by group, rows ascending
            int nRows = 0;
            for (int c0 = 0; c0 < cand; c0 += blockDim.x) {
                const int cidx = c0 + t;
                bool on = false;
                int r = 0, gl = 0;
                if (cidx < cand) {
                    int off = cidx;
                    gl = g0;
                    while (off >= D.groups[gl].preCount) off -= D.groups[gl++].preCount;
                    r = off;
                    const CycGroup& G = D.groups[gl];
                    const int x = D.pops[G.pre].base + G.preOffset + r;
                    on = G.accBase >= 0 && ((s_bits[x >> 5] >> (x & 31)) & 1u);
                }
                int total;
                const int pos = block_exclusive_scan(on ? 1 : 0, total, s_scan);
                if (on) s_rows[nRows + pos] = r | ((gl - g0) << 24);
                if (cidx < cand && r == 0) s_gStart[gl - g0] = nRows + pos;  // first row of the group
                nRows += total;
            }
            if (t == 0) s_gStart[g1 - g0] = nRows;
            __syncthreads();
            if (nRows > 0) {
                // post-centric folds: each post folds its group's rows in order;
                // four posts per item (16-byte row loads) where the rows allow
                int items = 0;
                for (int h = g0; h < g1; ++h)
                    items += D.groups[h].accBase < 0 ? 0 : ((D.groups[h].nPost & 3) == 0 ? D.groups[h].nPost >> 2
                                                                                        : D.groups[h].nPost);
                for (int it = t; it < items; it += blockDim.x) {
                    int h = g0, off = it;
                    for (;;) {
                        const CycGroup& G = D.groups[h];
                        const int ni = G.accBase < 0 ? 0 : ((G.nPost & 3) == 0 ? G.nPost >> 2 : G.nPost);
                        if (off < ni) break;
                        off -= ni;
                        ++h;
                    }
                    const CycGroup& G = D.groups[h];
                    const int q0 = s_gStart[h - g0], q1 = s_gStart[h - g0 + 1];
                    if ((G.nPost & 3) == 0) {
                        const int j = off << 2;
                        float a0 = s_acc[G.accBase + j], a1 = s_acc[G.accBase + j + 1];
                        float a2 = s_acc[G.accBase + j + 2], a3 = s_acc[G.accBase + j + 3];
                        for (int q = q0; q < q1; q += 4) {
                            float4 x[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                x[u] = q + u < q1 ? __ldg(reinterpret_cast<const float4*>(
                                                        G.W + (size_t)(s_rows[q + u] & 0xffffff) * G.nPost + j))
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                if (q + u < q1) {
                                    a0 = __fadd_rn(a0, x[u].x);
                                    a1 = __fadd_rn(a1, x[u].y);
                                    a2 = __fadd_rn(a2, x[u].z);
                                    a3 = __fadd_rn(a3, x[u].w);
                                }
                        }
                        s_acc[G.accBase + j] = a0;
                        s_acc[G.accBase + j + 1] = a1;
                        s_acc[G.accBase + j + 2] = a2;
                        s_acc[G.accBase + j + 3] = a3;
                    } else {
                        const int j = off;
                        float acc = s_acc[G.accBase + j];
                        for (int q = q0; q < q1; q += 8) {
                            float x[8];
#pragma unroll
                            for (int u = 0; u < 8; ++u)
                                x[u] = q + u < q1 ? __ldg(G.W + (size_t)(s_rows[q + u] & 0xffffff) * G.nPost + j) : 0.f;
#pragma unroll
                            for (int u = 0; u < 8; ++u)
                                if (q + u < q1) acc = __fadd_rn(acc, x[u]);
                        }
                        s_acc[G.accBase + j] = acc;
                    }
                }
            }
            __syncthreads();
            g0 = g1;
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
