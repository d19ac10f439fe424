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
// traces move one step behind, in the background blocks (phase t: x(t-1) from
// x(t-2), two buffers), so a sink block derives xd(t-1) and xd(t) of its rows
// from x(t-2) and the row's spike bit at t - 1 with the same operations.
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
    float* x;                   // pre traces [nPre]: x(t) for odd t (x(-1): the last window's end)
    float* x2;                  // pre traces [nPre]: x(t) for even t
    float* y;                   // post traces [nPost]
    int nPre, nPost, nSink;
    int skip;  // diagnostic (SSB_TAIL_SKIP, timing only): 1 no sink rows, 2 no background
    float aPlus, aMinus, decPlus, decMinus, wMax;
};

__device__ __forceinline__ float* sink_x(const TailDev& T, int step) {
    return step & 1 ? T.x : T.x2;
}

__device__ __forceinline__ float stdp_pot(float w, float xd, float aPlus, float wMax) {
    return stdp_clip(__fadd_rn(w, __fmul_rn(aPlus, xd)), wMax);
}

__device__ __forceinline__ bool pre_bit(const TailDev& T, int step, int r) {
    const int i = r + T.preOffset;
    return (__ldg(T.preBits + (size_t)step * T.preWords + (i >> 5)) >> (i & 31)) & 1u;
}

// Phase s + 1 of the background blocks: the pre traces of step s (x(s) from
// x(s - 1); dst: where x(s) goes) and the potentiation of step s for the rows
// silent at s (and, ex >= 0, at ex) at the post columns that spiked at s;
// rows over the background blocks' threads.
__device__ __forceinline__ void sink_background(const TailDev& T, int s, int ex, float* dst,
                                                int* s_q, int* s_nq) {
    const int nwp = (T.nPost + 31) >> 5;
    __syncthreads();
    if (threadIdx.x < nwp) s_q[kTailMaxPost + threadIdx.x] = __ldcg(T.P.bits + (size_t)s * T.P.nwords + threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0) {
        int c = 0;
        for (int i = 0; i < nwp; ++i)
            for (uint32_t m = s_q[kTailMaxPost + i]; m; m &= m - 1) s_q[c++] = i * 32 + __ffs(m) - 1;
        *s_nq = c;
    }
    __syncthreads();
    const int nq = *s_nq;
    const float* src = sink_x(T, s - 1);
    const int nBg = gridDim.x - T.nSink;
    const int tid = (blockIdx.x - T.nSink) * blockDim.x + threadIdx.x, nth = nBg * blockDim.x;
    const uint32_t* bs = T.preBits + (size_t)s * T.preWords;
    const uint32_t* be = ex >= 0 ? T.preBits + (size_t)ex * T.preWords : nullptr;
    if ((T.nPre & 3) == 0 && (T.preOffset & 3) == 0) {
        // four rows per thread (16-byte accesses): a volley step (most post
        // neurons spiking together) rewrites the whole matrix
        // work items (quad, block of eight spiking columns), quads fastest
        const int nQuad = T.nPre >> 2;
        const int nKb = max(1, (nq + 7) >> 3);
        for (int it = tid; it < nQuad * nKb; it += nth) {
            const int qd = it % nQuad, k0 = (it / nQuad) * 8;
            const int r = qd << 2, i = r + T.preOffset;
            const uint32_t spk = (__ldg(bs + (i >> 5)) >> (i & 31)) & 0xfu;
            uint32_t busy = spk;
            if (be) busy |= (__ldg(be + (i >> 5)) >> (i & 31)) & 0xfu;
            const float4 x = __ldcg(reinterpret_cast<const float4*>(src + r));
            const float xd[4] = {__fmul_rn(x.x, T.decPlus), __fmul_rn(x.y, T.decPlus),
                                 __fmul_rn(x.z, T.decPlus), __fmul_rn(x.w, T.decPlus)};
            if (k0 == 0) {
                float4 xn;
                xn.x = spk & 1u ? __fadd_rn(xd[0], 1.0f) : xd[0];
                xn.y = spk & 2u ? __fadd_rn(xd[1], 1.0f) : xd[1];
                xn.z = spk & 4u ? __fadd_rn(xd[2], 1.0f) : xd[2];
                xn.w = spk & 8u ? __fadd_rn(xd[3], 1.0f) : xd[3];
                *reinterpret_cast<float4*>(dst + r) = xn;
            }
            if (busy == 0xfu || nq == 0) continue;
            const float dw[4] = {__fmul_rn(T.aPlus, xd[0]), __fmul_rn(T.aPlus, xd[1]),
                                 __fmul_rn(T.aPlus, xd[2]), __fmul_rn(T.aPlus, xd[3])};
            float4 vals[8];  // eight 16-byte loads in flight
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (k0 + u < nq)
                    vals[u] = __ldcg(reinterpret_cast<const float4*>(T.WT + (size_t)s_q[k0 + u] * T.nPre + r));
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (k0 + u >= nq) continue;
                float4 o = vals[u];
                o.x = stdp_clip(__fadd_rn(o.x, dw[0]), T.wMax);
                o.y = stdp_clip(__fadd_rn(o.y, dw[1]), T.wMax);
                o.z = stdp_clip(__fadd_rn(o.z, dw[2]), T.wMax);
                o.w = stdp_clip(__fadd_rn(o.w, dw[3]), T.wMax);
                float* wp = T.WT + (size_t)s_q[k0 + u] * T.nPre + r;
                if (busy == 0) {
                    *reinterpret_cast<float4*>(wp) = o;
                } else {  // a spiking row belongs to the sink blocks this step
                    if (!(busy & 1u)) wp[0] = o.x;
                    if (!(busy & 2u)) wp[1] = o.y;
                    if (!(busy & 4u)) wp[2] = o.z;
                    if (!(busy & 8u)) wp[3] = o.w;
                }
            }
        }
        return;
    }
    for (int r = tid; r < T.nPre; r += nth) {
        const bool spk = pre_bit(T, s, r);
        const float xd = __fmul_rn(__ldcg(src + r), T.decPlus);
        dst[r] = spk ? __fadd_rn(xd, 1.0f) : xd;
        if (spk || nq == 0 || (ex >= 0 && pre_bit(T, ex, r))) continue;
        const float dw = __fmul_rn(T.aPlus, xd);
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

// A producer thread's spiking row of a step: its index and whether it was
// silent at the step before (owed that step's potentiation where a column
// spiked).  Read-only data, so the next step's rows are fetched while the
// current step's chains finish; the row's trace x(w-2) and weights load at
// the step's start.
struct SinkRow {
    int r = -1;  // row (local), -1: none
    bool silentPrev = false;
};

// xd(w - 1) and xd(w) of a spiking row from x(w - 2) (w = 0: xd(0) from x(-1))
__device__ __forceinline__ void sink_xd(const TailDev& T, int w, const SinkRow& q, float xs,
                                        float& xdp, float& xdw) {
    if (w == 0) {
        xdp = 0.f;
        xdw = __fmul_rn(xs, T.decPlus);
        return;
    }
    xdp = __fmul_rn(xs, T.decPlus);
    xdw = __fmul_rn(q.silentPrev ? xdp : __fadd_rn(xdp, 1.0f), T.decPlus);
}

__device__ __forceinline__ SinkRow sink_fetch(const TailDev& T, int w, int e, int cnt) {
    SinkRow q;
    if (e >= cnt) return q;
    const int r = __ldg(T.preList + (size_t)w * T.preN + e) - T.preOffset;
    if ((unsigned)r >= (unsigned)T.nPre) return q;
    q.r = r;
    q.silentPrev = w > 0 && !pre_bit(T, w - 1, r);
    return q;
}

// Stage a spiking row's values for the fold (after the potentiation owed from
// w - 1) and store its learning at w (depression, + potentiation where the
// column spiked at w).
__device__ __forceinline__ void sink_row(const TailDev& T, int w, const SinkRow& q, float xs,
                                         const float* vals, int c0, int nc, uint32_t prev,
                                         uint32_t spk, const float* s_yd, float* stage) {
    float xdp, xdw;
    sink_xd(T, w, q, xs, xdp, xdw);
#pragma unroll
    for (int j = 0; j < kSinkCols; ++j) {
        float val = vals[j];
        if (q.silentPrev && ((prev >> j) & 1u)) val = stdp_pot(val, xdp, T.aPlus, T.wMax);
        stage[j] = val;
        if (q.r < 0 || j >= nc) continue;
        float nv = __fsub_rn(val, __fmul_rn(T.aMinus, s_yd[j]));
        if ((spk >> j) & 1u) nv = __fadd_rn(nv, __fmul_rn(T.aPlus, xdw));
        T.WT[(size_t)(c0 + j) * T.nPre + q.r] = stdp_clip(nv, T.wMax);
    }
}

constexpr int kSinkPre = 3;  // chunks of a step whose rows are fetched ahead

__global__ void __launch_bounds__(kSinkThreads, 1) sink_step_kernel(TailDev T, int W) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ float s_stage[2][kSinkRows][kSinkCols];
    __shared__ float s_yd[kSinkCols];
    __shared__ uint32_t s_spk;
    __shared__ int s_cnt;
    __shared__ int s_q[kTailMaxPost + kTailMaxPost / 32];
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
    uint32_t prev = 0;     // the block's columns that spiked at w - 1
    const int i = t - 32;  // producers (warps 1..): chunk row i
    SinkRow rec[kSinkPre];
    if (sink && warp > 0 && W > 0) {
        const int cn = T.skip & 1 ? 0 : T.preCnt[0];
#pragma unroll
        for (int kk = 0; kk < kSinkPre; ++kk) rec[kk] = sink_fetch(T, 0, kk * kSinkRows + i, cn);
    }
    // SSB_TRACE: block 0 (sink) and block nSink (background) record each step:
    // {tag | count << 32, post update end | rows end << 32 (ns from the step's
    // start), barrier end, chain cycles}
    const bool tr = g_trace != nullptr && t == 0 &&
                    (blockIdx.x == 0 || static_cast<int>(blockIdx.x) == T.nSink);
    unsigned trBase = 0;
    if (tr) trBase = atomicAdd(&g_traceN, static_cast<unsigned>(W));
    grid.sync();
    for (int w = 0; w < W; ++w) {
        unsigned long long t0 = 0, tA = 0, tB = 0;
        long long chainCy = 0;
        int cnt = 0;
        if (tr) t0 = global_ns();
        if (sink) {
            float wv[kSinkPre][kSinkCols];
            float xs[kSinkPre];
            if (warp == 0) {
                const float ex = w == 0 ? (col ? P.excIn[c0 + lane] : 0.f) : a;
                const float ih = w == 0 ? (col ? P.inhIn[c0 + lane] : 0.f) : 0.f;
                bool spike = false;
                if (col) spike = lif_step<true>(lc, ex, ih, v, ge, gi, expMax, bad);
                const uint32_t m = __ballot_sync(kFull, spike);
                if (spike) atomicOr(P.bits + (size_t)w * P.nwords + ((c0 + lane) >> 5), 1u << ((c0 + lane) & 31));
                if (lane == 0) {
                    s_spk = m;
                    s_cnt = T.skip & 1 ? 0 : T.preCnt[w];
                }
                const float yd = __fmul_rn(y, T.decMinus);
                if (lane < kSinkCols) s_yd[lane] = yd;
                y = spike ? __fadd_rn(yd, 1.0f) : yd;
                a = 0.f;
            } else {  // meanwhile: the fetched rows' weights (final for this step) and traces
                const float* xsrc = sink_x(T, w == 0 ? -1 : w - 2);
#pragma unroll
                for (int kk = 0; kk < kSinkPre; ++kk) {
                    xs[kk] = rec[kk].r >= 0 ? __ldcg(xsrc + rec[kk].r) : 0.f;
#pragma unroll
                    for (int j = 0; j < kSinkCols; ++j)
                        wv[kk][j] = rec[kk].r >= 0 && j < nc
                                        ? __ldcg(T.WT + (size_t)(c0 + j) * nPre + rec[kk].r) : 0.f;
                }
            }
            __syncthreads();
            if (tr) tA = global_ns();
            const uint32_t spk = s_spk;
            cnt = s_cnt;
            const int nChunks = (cnt + kSinkRows - 1) / kSinkRows;
            for (int k = 0; k <= nChunks; ++k) {
                if (warp == 0) {
                    if (k > 0 && lane < kSinkCols) {  // the column chains of chunk k - 1
                        const long long cy0 = tr ? clock64() : 0;
                        const int n = min(kSinkRows, cnt - (k - 1) * kSinkRows);
                        const float* sb = &s_stage[(k - 1) & 1][0][lane];
                        // software-pipelined: the next eight staged values load
                        // while the current eight add (the chain is the step's floor)
                        const int n8 = n & ~7;
                        if (n8 > 0) {
                            float c[8];
#pragma unroll
                            for (int u = 0; u < 8; ++u) c[u] = sb[u * kSinkCols];
                            for (int q = 8; q < n8; q += 8) {
                                float d[8];
#pragma unroll
                                for (int u = 0; u < 8; ++u) d[u] = sb[(q + u) * kSinkCols];
#pragma unroll
                                for (int u = 0; u < 8; ++u) a = __fadd_rn(a, c[u]);
#pragma unroll
                                for (int u = 0; u < 8; ++u) c[u] = d[u];
                            }
#pragma unroll
                            for (int u = 0; u < 8; ++u) a = __fadd_rn(a, c[u]);
                        }
                        for (int q = n8; q < n; ++q) a = __fadd_rn(a, sb[q * kSinkCols]);
                        if (tr) {
                            const float aa = a;
                            asm volatile("" ::"f"(aa));
                            chainCy += clock64() - cy0;
                        }
                    }
                } else {
                    if (k < nChunks) {
                        const int e = k * kSinkRows + i;
                        float* stage = &s_stage[k & 1][i][0];
                        if (k < kSinkPre) {
#pragma unroll
                            for (int kk = 0; kk < kSinkPre; ++kk)
                                if (kk == k && e < cnt)
                                    sink_row(T, w, rec[kk], xs[kk], wv[kk], c0, nc, prev, spk, s_yd, stage);
                        } else if (e < cnt) {  // beyond the fetched chunks: on demand
                            const SinkRow q = sink_fetch(T, w, e, cnt);
                            float vals[kSinkCols];
#pragma unroll
                            for (int j = 0; j < kSinkCols; ++j)
                                vals[j] = q.r >= 0 && j < nc ? __ldcg(T.WT + (size_t)(c0 + j) * nPre + q.r) : 0.f;
                            const float x0 = q.r >= 0 ? __ldcg(sink_x(T, w == 0 ? -1 : w - 2) + q.r) : 0.f;
                            sink_row(T, w, q, x0, vals, c0, nc, prev, spk, s_yd, stage);
                        }
                    }
                    // after the last chunk: the next step's rows (read-only data)
                    if (k == max(nChunks - 1, 0) && w + 1 < W) {
                        const int cn = T.skip & 1 ? 0 : __ldg(T.preCnt + w + 1);
#pragma unroll
                        for (int kk = 0; kk < kSinkPre; ++kk)
                            rec[kk] = sink_fetch(T, w + 1, kk * kSinkRows + i, cn);
                    }
                }
                __syncthreads();
            }
            prev = spk;
            if (tr) tB = global_ns();
        } else if (w > 0) {
            if (!(T.skip & 2)) sink_background(T, w - 1, w, sink_x(T, w - 1), s_q, &s_nq);
            if (tr) {
                tA = tB = global_ns();
                cnt = s_nq;
            }
        } else if (tr) {
            tA = tB = global_ns();
        }
        grid.sync();
        if (tr) {
            unsigned long long* e = g_trace + 4ull * (trBase + w);
            if (trBase + w < g_traceCap) {
                e[0] = (sink ? 0x5100ull : 0x5110ull) | (static_cast<unsigned long long>(cnt) << 32);
                e[1] = (tA - t0) | ((tB - t0) << 32);
                e[2] = global_ns() - t0;
                e[3] = static_cast<unsigned long long>(chainCy);
            }
        }
    }
    // the last step's potentiation and traces (x(W-1) where the next window expects x(-1))
    if (!sink && W > 0 && !(T.skip & 2)) sink_background(T, W - 1, -1, T.x, s_q, &s_nq);
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
