// plastic.cuh — the window pipeline for a plastic group into a sink (extension
// F2: KC -> DN with pair STDP; included inside namespace ssbk::<unnamed> by
// kernels.cuh).
//
// A plastic group's weights change after every step, which used to force the
// whole network into step mode (one launch per population per step, ~80 us
// per step at config 3).  But when the plastic group's post population is a
// sink fed by that group alone (the mushroom body's DN), nothing upstream
// depends on the weights: the pre population (KC) keeps its window pipeline
// and two kernels per window run the rest step by step.
//
// The rule (DESIGN.md §1 row A22, kernels.cuh stdp_update_kernel) touches a
// weight w[r][j] at step t in two ways only: row r spiked (w -= aMinus·yd_j,
// += aPlus·xd_r if j spiked too, clip) or, r silent, column j spiked
// (w += aPlus·xd_r, clip).  Post column j's input at t + 1 is the fold of
// the rows spiking at t over column j, in row order, of the weights as they
// are before step t's learning.  One cooperative kernel per window, one grid
// barrier per step; phase t:
//   sink blocks (kSinkCols post columns each, the weights transposed
//     [nPost][nPre] so a column is contiguous): the post update at t (input:
//     the block's own fold of t - 1); then for every row spiking at t, the
//     potentiation still owed from t - 1 (row silent at t - 1, column spiked),
//     the staged value for the fold, and the row's learning at t; warp 0's
//     lanes run the column chains over the staged chunks, rows ascending;
//   background blocks: the potentiation of t - 1 for the rows silent at both
//     t - 1 and t (contiguous, coalesced along the columns that spiked).
// The two touch disjoint rows; every weight sees the same operations in the
// same order as in step mode (potentiation of t - 1 before the row's next
// learning), so weights and spikes are bit-identical.  After the last step
// the background blocks apply its potentiation to every silent row.  The pre
// traces' decayed values xd[t][r] come from a table the prepass writes
// (sink_trace_kernel, [W][nPre]).
constexpr int kSinkThreads = 512;
constexpr int kSinkCols = 2;                      // post columns per sink block
constexpr int kSinkRows = kSinkThreads - 32;      // rows per staged chunk (a producer thread each)
constexpr int kTailMaxPost = 128;

struct TailDev {
    PopDev P;                   // the post population (state, spike bits of the set)
    const int* preList;         // pre spikes of window step w: preList[w * preN + k]
    const int* preCnt;          // [W]
    const uint32_t* preBits;    // [W][preWords]
    int preN, preWords, preOffset;
    float* WT;                  // transposed weights [nPost][nPre]
    float* x;                   // pre traces [nPre] (end of the last window)
    float* y;                   // post traces [nPost]
    float* xd;                  // [Wmax][nPre]: the pre traces' decayed values of each window step
    int nPre, nPost, nSink;
    float aPlus, aMinus, decPlus, decMinus, wMax;
};

// xd[t][r] = x_r(t-1)·decPlus for the window's steps, and x moved on
// (x = xd + 1 where r spiked) -- the pre trace update of stdp_update_kernel,
// a thread per row.
__global__ void __launch_bounds__(256) sink_trace_kernel(TailDev T, int W) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= T.nPre) return;
    const int i = r + T.preOffset;
    float x = T.x[r];
    const uint32_t* pb = T.preBits + (i >> 5);
    float* out = T.xd + r;
#pragma unroll 8
    for (int t = 0; t < W; ++t) {
        const uint32_t word = __ldg(pb + (size_t)t * T.preWords);
        const float xd = __fmul_rn(x, T.decPlus);
        out[(size_t)t * T.nPre] = xd;
        x = (word >> (i & 31)) & 1u ? __fadd_rn(xd, 1.0f) : xd;
    }
    T.x[r] = x;
}

__device__ __forceinline__ float stdp_pot(float w, float xd, float aPlus, float wMax) {
    return stdp_clip(__fadd_rn(w, __fmul_rn(aPlus, xd)), wMax);
}

__device__ __forceinline__ bool pre_bit(const TailDev& T, int step, int r) {
    const int i = r + T.preOffset;
    return (__ldg(T.preBits + (size_t)step * T.preWords + (i >> 5)) >> (i & 31)) & 1u;
}

// Potentiation of step s for the rows silent at s (and, ex >= 0, at ex) at
// the post columns that spiked at s; rows over the background blocks' threads.
__device__ __forceinline__ void sink_background(const TailDev& T, int s, int ex, int* s_q,
                                                int* s_nq) {
    const int nwp = (T.nPost + 31) >> 5;
    __syncthreads();
    if (threadIdx.x == 0) {
        int c = 0;
        for (int i = 0; i < nwp; ++i)
            for (uint32_t m = __ldcg(T.P.bits + (size_t)s * T.P.nwords + i); m; m &= m - 1)
                s_q[c++] = i * 32 + __ffs(m) - 1;
        *s_nq = c;
    }
    __syncthreads();
    const int nq = *s_nq;
    if (nq == 0) return;
    const int nBg = gridDim.x - T.nSink;
    for (int r = (blockIdx.x - T.nSink) * blockDim.x + threadIdx.x; r < T.nPre;
         r += nBg * blockDim.x) {
        if (pre_bit(T, s, r) || (ex >= 0 && pre_bit(T, ex, r))) continue;
        const float dw = __fmul_rn(T.aPlus, __ldg(T.xd + (size_t)s * T.nPre + r));
        for (int k0 = 0; k0 < nq; k0 += 8) {  // eight loads in flight
            float vals[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (k0 + u < nq) vals[u] = __ldcg(T.WT + (size_t)s_q[k0 + u] * T.nPre + r);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (k0 + u < nq)
                    T.WT[(size_t)s_q[k0 + u] * T.nPre + r] = stdp_clip(__fadd_rn(vals[u], dw), T.wMax);
        }
    }
}

__global__ void __launch_bounds__(kSinkThreads, 1) sink_step_kernel(TailDev T, int W) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ float s_stage[2][kSinkRows][kSinkCols];
    __shared__ float s_yd[kSinkCols];
    __shared__ uint32_t s_spk;
    __shared__ int s_q[kTailMaxPost];
    __shared__ int s_nq;
    __shared__ long long s_red[32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const PopDev& P = T.P;
    const int nPre = T.nPre;
    // the window's post spike bits are OR-ed in by the sink blocks
    if (blockIdx.x == 0)
        for (int i = t; i < W * P.nwords; i += blockDim.x) P.bits[i] = 0u;
    const bool sink = static_cast<int>(blockIdx.x) < T.nSink;
    const int c0 = blockIdx.x * kSinkCols;
    const int nc = sink ? min(kSinkCols, T.nPost - c0) : 0;
    const bool col = warp == 0 && lane < nc;
    const LifConst lc = lif_const(P);
    float v = 0.f, ge = 0.f, gi = 0.f, y = 0.f, a = 0.f;
    uint32_t flag = 1, expMax = 0, bad = 0;
    if (col) {
        v = P.v[c0 + lane];
        ge = P.gExc[c0 + lane];
        gi = P.gInh[c0 + lane];
        flag = P.nanFlag[c0 + lane] ? 1u : 0u;
        y = T.y[c0 + lane];
    }
    uint32_t prev = 0;  // the block's columns that spiked at w - 1
    grid.sync();
    for (int w = 0; w < W; ++w) {
        if (sink) {
            if (warp == 0) {
                const float ex = w == 0 ? (col ? P.excIn[c0 + lane] : 0.f) : a;
                const float ih = w == 0 ? (col ? P.inhIn[c0 + lane] : 0.f) : 0.f;
                bool spike = false;
                if (col) spike = lif_step<true>(lc, ex, ih, v, ge, gi, expMax, bad);
                const uint32_t m = __ballot_sync(kFull, spike);
                if (spike) atomicOr(P.bits + (size_t)w * P.nwords + ((c0 + lane) >> 5), 1u << ((c0 + lane) & 31));
                if (lane == 0) s_spk = m;
                const float yd = __fmul_rn(y, T.decMinus);
                if (lane < kSinkCols) s_yd[lane] = yd;
                y = spike ? __fadd_rn(yd, 1.0f) : yd;
                a = 0.f;
            }
            __syncthreads();
            const uint32_t spk = s_spk;
            const int cnt = T.preCnt[w];
            const int* L = T.preList + (size_t)w * T.preN;
            const int nChunks = (cnt + kSinkRows - 1) / kSinkRows;
            for (int k = 0; k <= nChunks; ++k) {
                if (warp == 0) {
                    if (k > 0 && lane < kSinkCols) {  // the column chains of chunk k - 1
                        const int n = min(kSinkRows, cnt - (k - 1) * kSinkRows);
                        const float* sb = &s_stage[(k - 1) & 1][0][lane];
#pragma unroll 8
                        for (int i = 0; i < n; ++i) a = __fadd_rn(a, sb[i * kSinkCols]);
                    }
                } else if (k < nChunks) {
                    const int i = t - 32;
                    const int e = k * kSinkRows + i;
                    if (e < cnt) {
                        const int r = __ldg(L + e) - T.preOffset;
                        const bool live = (unsigned)r < (unsigned)nPre;
                        const bool pend = live && w > 0 && prev != 0 && !pre_bit(T, w - 1, r);
                        const float xdp = pend ? __ldg(T.xd + (size_t)(w - 1) * nPre + r) : 0.f;
                        const float xdw = live && spk ? __ldg(T.xd + (size_t)w * nPre + r) : 0.f;
                        float vals[kSinkCols];
#pragma unroll
                        for (int j = 0; j < kSinkCols; ++j)
                            vals[j] = live && j < nc ? __ldcg(T.WT + (size_t)(c0 + j) * nPre + r) : 0.f;
#pragma unroll
                        for (int j = 0; j < kSinkCols; ++j) {
                            float val = vals[j];
                            if (pend && ((prev >> j) & 1u)) val = stdp_pot(val, xdp, T.aPlus, T.wMax);
                            s_stage[k & 1][i][j] = val;
                            if (!live || j >= nc) continue;
                            float nv = __fsub_rn(val, __fmul_rn(T.aMinus, s_yd[j]));
                            if ((spk >> j) & 1u) nv = __fadd_rn(nv, __fmul_rn(T.aPlus, xdw));
                            T.WT[(size_t)(c0 + j) * nPre + r] = stdp_clip(nv, T.wMax);
                        }
                    }
                }
                __syncthreads();
            }
            prev = spk;
        } else if (w > 0) {
            sink_background(T, w - 1, w, s_q, &s_nq);
        }
        grid.sync();
    }
    if (!sink && W > 0) sink_background(T, W - 1, -1, s_q, &s_nq);
    // ---- end of window: post state, next window's first input, traces
    if (col) {
        const int j = c0 + lane;
        P.v[j] = v;
        P.gExc[j] = ge;
        P.gInh[j] = gi;
        P.excIn[j] = a;
        P.inhIn[j] = 0.f;
        P.nanFlag[j] = static_cast<uint8_t>(flag | (expMax == 0x7f800000u));
        T.y[j] = y;
    }
    const int newly = col && !flag && expMax == 0x7f800000u ? 1 : 0;
    const long long tot = block_sum(static_cast<long long>(newly), s_red);
    if (t == 0 && tot) atomicAdd(P.flagged, (unsigned long long)tot);
}
