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
// += aPlus·xd_r(t) if j spiked too, clip) or, r silent, column j spiked
// (potentiation: w += aPlus·xd_r(t), clip).  Post column j's input at t + 1
// is the fold of the rows spiking at t over column j, in row order, of the
// weights as they are before step t's learning.  The weights are kept
// transposed [nPost][nPre] (a column contiguous).  One cooperative kernel per
// window, two roles, no grid-wide barrier:
//   sink blocks (kSinkCols post columns each), warps in four parts:
//     two chain warps (warp 0: even steps, warp 4: odd steps) fold the staged
//     chunks of their steps, rows ascending, and the warp that finishes
//     fold(t) runs the post update of t + 1 (fold(t + 1) needs the post spikes
//     of t, not fold(t), so consecutive steps' chains overlap; the post state
//     passes between them in shared memory);
//     fifteen producer warps stage every row spiking at t -- its weights after
//     the potentiations it still owes from steps t - L .. t - 1 (silent since,
//     a column spiked) -- into a per-parity ring of chunk buffers
//     (full/empty mbarriers), then, once t's post spikes are out, store the
//     row's learning at t; a step's rows and weights load during the step
//     before (rows that spiked then take their learned values from shared
//     memory);
//     a notifier warp tells the background blocks when t's post spikes are out;
//   background blocks: the potentiation of step s for the rows silent through
//     s .. s + L (a volley step rewrites the whole matrix), up to L steps behind
//     the sink blocks -- so a volley's matrix pass overlaps the next steps.
// Every potentiation of a weight is applied once, by exactly one of the two
// (the background iff the row stays silent L more steps), and every weight
// sees the same operations in the same step order as in step mode: weights
// and spikes are bit-identical.  Ordering: per-step counters (the sink blocks'
// post updates of step s before the background's step s; the background's step
// t - L - 1 before a sink block reads rows at t).  At the window's end the
// background applies the last steps' potentiations to every silent row.  The
// pre traces' decayed values xd[t][r] come from a table the prepass writes
// (sink_trace_kernel, [W][nPre]).
constexpr int kSinkThreads = 640;
constexpr int kSinkCols = 2;                      // post columns per sink block
// producers: the warps off scheduler 0 (15 of 20), where the chain warps (the step's
// critical path) issue; a staged chunk is a row per producer
constexpr int kSinkRows = kSinkThreads / 4 * 3;   // 480
constexpr int kSinkLag = 4;                       // L: the background's lag in steps
constexpr int kTailMaxPost = 128;
constexpr int kSinkMaxW = 256;                    // window steps (the sink blocks' spike history)

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
    int* sinkDone;              // [Wmax]: sink blocks past their post update of step s
    int* bgDone;                // [Wmax]: background blocks done with step s
    int nPre, nPost, nSink;
    int skip;  // diagnostic (SSB_TAIL_SKIP, timing only): 1 no sink rows, 2 no background
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

__device__ __forceinline__ uint32_t pre_word(const TailDev& T, int step, int i) {
    return __ldg(T.preBits + (size_t)step * T.preWords + (i >> 5));
}

__device__ int* g_watch = nullptr;  // diagnostic (SSB_SINK_WATCH): progress of each role

__device__ __forceinline__ void spin_until(const int* ctr, int target) {
    while (*reinterpret_cast<const volatile int*>(ctr) < target) __nanosleep(32);
    __threadfence();
}

// ---- background blocks -------------------------------------------------------
// Step s: for post column j that spiked at s, w[r][j] += aPlus·xd_r(s) (clip)
// for every row r silent at s .. min(s + L, W - 1).  A thread owns fixed work
// items (four rows x a group of eight post columns) for the whole window, so
// a weight's potentiations of consecutive steps come from one thread in order.
__device__ void sink_background(const TailDev& T, int W, uint32_t* s_m) {
    const int nwp = (T.nPost + 31) >> 5;
    const int nBg = gridDim.x - T.nSink;
    const int tid = (blockIdx.x - T.nSink) * blockDim.x + threadIdx.x, nth = nBg * blockDim.x;
    const bool quads = (T.nPre & 3) == 0 && (T.preOffset & 3) == 0;
    const int nRowIt = quads ? T.nPre >> 2 : T.nPre;
    const int nGrp = (T.nPost + 7) >> 3;
    for (int s = 0; s < W; ++s) {
        if (threadIdx.x == 0) spin_until(T.sinkDone + s, T.nSink);
        __syncthreads();
        if (threadIdx.x < nwp) s_m[threadIdx.x] = __ldcg(T.P.bits + (size_t)s * T.P.nwords + threadIdx.x);
        __syncthreads();
        uint32_t any = 0;
        for (int k = 0; k < nwp; ++k) any |= s_m[k];
        const int hi = min(s + kSinkLag, W - 1);
        if (any && !(T.skip & 2)) {
            for (int it = tid; it < nRowIt * nGrp; it += nth) {
                const int g = it / nRowIt, ri = it - g * nRowIt;
                const uint32_t cols = (s_m[g >> 2] >> ((g & 3) * 8)) & 0xffu;
                if (!cols) continue;
                if (quads) {
                    const int r = ri << 2, i = r + T.preOffset;
                    uint32_t busy = 0;
                    for (int u = s; u <= hi; ++u) busy |= (pre_word(T, u, i) >> (i & 31)) & 0xfu;
                    if (busy == 0xfu) continue;
                    const float4 xd = __ldg(reinterpret_cast<const float4*>(T.xd + (size_t)s * T.nPre + r));
                    const float dw0 = __fmul_rn(T.aPlus, xd.x), dw1 = __fmul_rn(T.aPlus, xd.y);
                    const float dw2 = __fmul_rn(T.aPlus, xd.z), dw3 = __fmul_rn(T.aPlus, xd.w);
                    float4 vals[8];  // the group's spiking columns: every load in flight
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if ((cols >> u) & 1u)
                            vals[u] = __ldcg(reinterpret_cast<const float4*>(T.WT + (size_t)(g * 8 + u) * T.nPre + r));
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        if (!((cols >> u) & 1u)) continue;
                        float4 o = vals[u];
                        o.x = stdp_clip(__fadd_rn(o.x, dw0), T.wMax);
                        o.y = stdp_clip(__fadd_rn(o.y, dw1), T.wMax);
                        o.z = stdp_clip(__fadd_rn(o.z, dw2), T.wMax);
                        o.w = stdp_clip(__fadd_rn(o.w, dw3), T.wMax);
                        float* wp = T.WT + (size_t)(g * 8 + u) * T.nPre + r;
                        if (busy == 0) {
                            *reinterpret_cast<float4*>(wp) = o;
                        } else {  // a row spiking by s + L belongs to the sink blocks
                            if (!(busy & 1u)) wp[0] = o.x;
                            if (!(busy & 2u)) wp[1] = o.y;
                            if (!(busy & 4u)) wp[2] = o.z;
                            if (!(busy & 8u)) wp[3] = o.w;
                        }
                    }
                } else {
                    const int r = ri, i = r + T.preOffset;
                    bool busy = false;
                    for (int u = s; u <= hi; ++u) busy = busy || ((pre_word(T, u, i) >> (i & 31)) & 1u);
                    if (busy) continue;
                    const float dw = __fmul_rn(T.aPlus, __ldg(T.xd + (size_t)s * T.nPre + r));
                    float vals[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if ((cols >> u) & 1u) vals[u] = __ldcg(T.WT + (size_t)(g * 8 + u) * T.nPre + r);
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if ((cols >> u) & 1u)
                            T.WT[(size_t)(g * 8 + u) * T.nPre + r] = stdp_clip(__fadd_rn(vals[u], dw), T.wMax);
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(T.bgDone + s, 1);
            if (g_watch && static_cast<int>(blockIdx.x) == T.nSink) g_watch[3 * T.nSink] = s;
        }
    }
}

// ---- sink blocks -------------------------------------------------------------
// The pre spike bits of steps w - L .. w + 1 stay in a shared-memory ring
// (dynamic shared memory, [L + 2][preWords]).
constexpr int kSinkRing = kSinkLag + 2;  // steps w - L .. w + 1

__device__ __forceinline__ bool ring_bit(const uint32_t* ring, int preWords, int step, int i) {
    return (ring[(step % kSinkRing) * preWords + (i >> 5)] >> (i & 31)) & 1u;
}

// words [lo, hi) of a step's pre spike bits into the ring, threads i0 + n·k
__device__ __forceinline__ void ring_load(const TailDev& T, uint32_t* ring, int step, int i0, int n,
                                          int lo = 0, int hi = 1 << 30) {
    const uint32_t* pb = T.preBits + (size_t)step * T.preWords;
    uint32_t* dst = ring + (step % kSinkRing) * T.preWords;
    hi = min(hi, T.preWords);
    for (int k0 = lo + i0; k0 < hi; k0 += 8 * n) {  // eight loads in flight
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (k0 + u * n < hi) v[u] = __ldg(pb + k0 + u * n);
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (k0 + u * n < hi) dst[k0 + u * n] = v[u];
    }
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src)
                 : "memory");
}

// A producer thread's spiking row of a step: its index, its spike bits over
// the L steps before (bit d - 1: spiked at w - d), and xd at the first step
// it owes a potentiation for (w - run; xd(w) when it spiked at w - 1).
// Read-only data, so the next step's rows are fetched while the current
// step's chains finish; the weights load at the step's start.
struct SinkRow {
    int r = -1;  // row (local), -1: none
    uint32_t hist = 0;
    float xs = 0.f;
};

// steps since the row's last spike, at most L and not before the window
__device__ __forceinline__ int sink_run(uint32_t hist, int w) {
    return min(hist ? __ffs(hist) - 1 : kSinkLag, w);
}

// the ring must hold steps w - L .. w - 1
__device__ __forceinline__ SinkRow sink_fetch_row(const TailDev& T, int w, int rg,
                                                  const uint32_t* ring) {
    SinkRow q;
    const int r = rg - T.preOffset;
    if ((unsigned)r >= (unsigned)T.nPre) return q;
    q.r = r;
    uint32_t h = 0;
#pragma unroll
    for (int d = 1; d <= kSinkLag; ++d)
        if (w - d >= 0) h |= static_cast<uint32_t>(ring_bit(ring, T.preWords, w - d, rg)) << (d - 1);
    q.hist = h;
    q.xs = __ldg(T.xd + (size_t)(w - sink_run(h, w)) * T.nPre + r);
    return q;
}

__device__ __forceinline__ SinkRow sink_fetch(const TailDev& T, int w, int e, int cnt,
                                              const uint32_t* ring) {
    if (e >= cnt) return SinkRow{};
    return sink_fetch_row(T, w, __ldg(T.preList + (size_t)w * T.preN + e), ring);
}

// the rows of chunks 0 .. kSinkPre - 1 (slot e0 + k·rows): every index load first
template <int N>
__device__ __forceinline__ void sink_fetch_all(const TailDev& T, int w, int e0, int rows, int cnt,
                                               const uint32_t* ring, SinkRow* out) {
    int rg[N];
#pragma unroll
    for (int k = 0; k < N; ++k)
        rg[k] = e0 + k * rows < cnt ? __ldg(T.preList + (size_t)w * T.preN + e0 + k * rows) : -1;
#pragma unroll
    for (int k = 0; k < N; ++k)
        out[k] = e0 + k * rows < cnt ? sink_fetch_row(T, w, rg[k], ring) : SinkRow{};
}

// A spiking row's values for the fold: its weights after the potentiations
// it owes (steps w - run .. w - 1, silent, where a column spiked: s_hist[s],
// oldest first; xd(s + 1) = xd(s)·decPlus along a silent run, as the prepass
// computes it); xdw = xd(w).
__device__ __forceinline__ void sink_stage(const TailDev& T, int w, const SinkRow& q, float* v,
                                           const uint32_t* s_hist, float& xdw) {
    float xd = q.xs;
    for (int s = w - sink_run(q.hist, w); s < w; ++s) {
        const uint32_t m = s_hist[s];
#pragma unroll
        for (int j = 0; j < kSinkCols; ++j)
            if ((m >> j) & 1u) v[j] = stdp_pot(v[j], xd, T.aPlus, T.wMax);
        xd = __fmul_rn(xd, T.decPlus);
    }
    xdw = xd;
}

// The row's learning at w: depression, + potentiation where the column spiked.
__device__ __forceinline__ void sink_learn(const TailDev& T, const SinkRow& q, const float* v,
                                           float xdw, int c0, int nc, uint32_t spk, const float* yd,
                                           float* out) {
#pragma unroll
    for (int j = 0; j < kSinkCols; ++j) {
        out[j] = 0.f;
        if (j >= nc) continue;
        float nv = __fsub_rn(v[j], __fmul_rn(T.aMinus, yd[j]));
        if ((spk >> j) & 1u) nv = __fadd_rn(nv, __fmul_rn(T.aPlus, xdw));
        out[j] = stdp_clip(nv, T.wMax);
        T.WT[(size_t)(c0 + j) * T.nPre + q.r] = out[j];
    }
}

struct SinkState {
    float v, ge, gi, y;
    uint32_t flag, expMax;
};

constexpr int kSinkPre = 4;    // chunks of a step whose rows are fetched ahead
constexpr int kSinkBufs = 4;   // staged chunk buffers per ring (one ring per step parity:
                               // each chain warp consumes its own ring in order)
constexpr int kSinkProdWarps = kSinkRows / 32;
constexpr int kSinkLearnBytes = 2 * kSinkCols * kSinkPre * kSinkRows * 4;
constexpr int kSinkIdxBytes = 3 * kSinkPre * kSinkRows * 4;  // + the rows of three steps

__global__ void __launch_bounds__(kSinkThreads, 1) sink_step_kernel(TailDev T, int W) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ __align__(16) float s_stage[2][kSinkBufs][kSinkCols][kSinkRows];  // a column's rows contiguous
    __shared__ __align__(8) uint64_t s_full[2][kSinkBufs], s_empty[2][kSinkBufs], s_dn[2], s_pdone[2];
    __shared__ float s_yd[2][kSinkCols];
    __shared__ uint32_t s_hist[kSinkMaxW];  // sink: the block's column spikes of each step
    __shared__ long long s_red[32];
    __shared__ SinkState s_state[kSinkCols];  // the post neurons' state after the last post update
    extern __shared__ __align__(16) uint32_t s_bitRing[];  // sink: pre spike bits [L + 2][preWords],
    // then the rows' learned weights [2][kSinkCols][kSinkPre * kSinkRows] (producers)
    using LearnBuf = float[kSinkCols][kSinkPre * kSinkRows];
    LearnBuf* s_learn = reinterpret_cast<LearnBuf*>(s_bitRing + ((kSinkRing * T.preWords + 3) & ~3));
    // producers: step w's rows at w % 3 (global index), ascending
    using IdxBuf = int[kSinkPre][kSinkRows];
    IdxBuf* s_idx = reinterpret_cast<IdxBuf*>(reinterpret_cast<char*>(s_learn) + kSinkLearnBytes);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const PopDev& P = T.P;
    const int nPre = T.nPre;
    // the window's post spike bits are OR-ed in by the sink blocks; counters
    if (blockIdx.x == 0) {
        for (int i = t; i < W * P.nwords; i += blockDim.x) P.bits[i] = 0u;
        for (int i = t; i < W; i += blockDim.x) T.sinkDone[i] = T.bgDone[i] = 0;
    }
    const bool sink = static_cast<int>(blockIdx.x) < T.nSink;
    if (sink && t == 0) {
        for (int r = 0; r < 2; ++r)
            for (int b = 0; b < kSinkBufs; ++b) {
                mbar_init(&s_full[r][b], kSinkProdWarps);
                mbar_init(&s_empty[r][b], 1);
            }
        mbar_init(&s_dn[0], 1);
        mbar_init(&s_dn[1], 1);
        mbar_init(&s_pdone[0], kSinkProdWarps + 1);  // + the notifier warp
        mbar_init(&s_pdone[1], kSinkProdWarps + 1);
        mbar_fence_init();
    }
    grid.sync();
    if (!sink) {
        sink_background(T, W, reinterpret_cast<uint32_t*>(s_hist));
        return;
    }
    const int c0 = blockIdx.x * kSinkCols;
    const int nc = min(kSinkCols, T.nPost - c0);
    // producers: the warps off scheduler 0, where warp 0 (post update + the
    // column chains, the step's critical path) issues alone
    const bool producer = (warp & 3) != 0;
    const int i = ((warp >> 2) * 3 + (warp & 3) - 1) * 32 + lane;  // producers: chunk row i
    // SSB_TRACE: warp 0 of block 0 records each step: {tag | count << 32,
    // post update end (ns from the step's start) | chains end << 32, 0, chain cycles}
    const bool tr = g_trace != nullptr && t == 32 && blockIdx.x == 0;  // producer thread 32
    unsigned trBase = 0;
    if (tr) trBase = atomicAdd(&g_traceN, static_cast<unsigned>(W));
    if (warp == 0 || warp == 4) {
        // ---- two chain warps (warp 0: the even steps' folds, warp 4: the odd
        //      ones; both on scheduler 0, each latency-bound): fold(t + 1)
        //      needs the post spikes of t (through the learning of t), not
        //      fold(t), so consecutive steps' chains run at once.  The warp
        //      that finishes fold(t) runs the post update of t + 1; the
        //      post neurons' state passes between the two through s_state.
        const int c = warp >> 2;
        const bool colc = lane < nc;
        const LifConst lc = lif_const(P);
        float a = 0.f;
        uint32_t bad = 0;
        const auto post_update = [&](int s, float ex, float ih, float& v, float& ge, float& gi,
                                     float& y, uint32_t flag, uint32_t& expMax) {
            // the producers have read step s - 2's post spikes and traces
            // (their slots are rewritten now)
            if (s >= 2) mbar_wait(&s_pdone[s & 1], ((s - 2) >> 1) & 1);
            bool spike = false;
            if (colc) spike = lif_step<true>(lc, ex, ih, v, ge, gi, expMax, bad);
            const uint32_t m = __ballot_sync(kFull, spike);
            if (spike) atomicOr(P.bits + (size_t)s * P.nwords + ((c0 + lane) >> 5), 1u << ((c0 + lane) & 31));
            const float yd = __fmul_rn(y, T.decMinus);
            if (lane < kSinkCols) s_yd[s & 1][lane] = yd;
            if (lane == 0) s_hist[s] = m;
            y = spike ? __fadd_rn(yd, 1.0f) : yd;
            if (colc) s_state[lane] = SinkState{v, ge, gi, y, flag, expMax};
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_dn[s & 1]);
        };
        float v = 0.f, ge = 0.f, gi = 0.f, y = 0.f;
        uint32_t flag = 1, expMax = 0;
        int last = -1;  // the last post update this warp ran
        if (c == 1 && W > 0) {  // step 0's post update (input: the last window's last fold)
            if (colc) {
                v = P.v[c0 + lane];
                ge = P.gExc[c0 + lane];
                gi = P.gInh[c0 + lane];
                flag = P.nanFlag[c0 + lane] ? 1u : 0u;
                y = T.y[c0 + lane];
            }
            post_update(0, colc ? P.excIn[c0 + lane] : 0.f, colc ? P.inhIn[c0 + lane] : 0.f, v, ge,
                        gi, y, flag, expMax);
            last = 0;
        }
        int g = 0;  // chunk sequence number in this warp's ring (the producers count the same way)
        for (int w = c; w < W; w += 2) {
            const int cnt = T.skip & 1 ? 0 : __ldg(T.preCnt + w);
            const int nCh = (cnt + kSinkRows - 1) / kSinkRows;
            // the fold of step w: the staged chunks in order, rows ascending
            a = 0.f;
            for (int k = 0; k < nCh; ++k, ++g) {
                const int b = g % kSinkBufs;
                mbar_wait(&s_full[c][b], (g / kSinkBufs) & 1);
                if (lane < kSinkCols) {
                    const int n = min(kSinkRows, cnt - k * kSinkRows);
                    const float* sb = &s_stage[c][b][lane][0];
                    const int n4 = n & ~3;
                    if (n4 > 0) {
                        float4 cc = *reinterpret_cast<const float4*>(sb);
                        for (int q = 4; q < n4; q += 4) {
                            const float4 d = *reinterpret_cast<const float4*>(sb + q);
                            a = __fadd_rn(a, cc.x);
                            a = __fadd_rn(a, cc.y);
                            a = __fadd_rn(a, cc.z);
                            a = __fadd_rn(a, cc.w);
                            cc = d;
                        }
                        a = __fadd_rn(a, cc.x);
                        a = __fadd_rn(a, cc.y);
                        a = __fadd_rn(a, cc.z);
                        a = __fadd_rn(a, cc.w);
                    }
                    for (int q = n4; q < n; ++q) a = __fadd_rn(a, sb[q]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_empty[c][b]);
            }
            if (g_watch && lane == 0) g_watch[blockIdx.x * 2 + c] = w;
            if (w + 1 < W) {  // the post update of w + 1: the state of w from the other warp
                mbar_wait(&s_dn[w & 1], (w >> 1) & 1);
                if (colc) {
                    const SinkState st = s_state[lane];
                    v = st.v;
                    ge = st.ge;
                    gi = st.gi;
                    y = st.y;
                    flag = st.flag;
                    expMax = st.expMax;
                }
                post_update(w + 1, a, 0.f, v, ge, gi, y, flag, expMax);
                last = w + 1;
            } else if (colc) {  // the window's last fold: the next window's first input
                P.excIn[c0 + lane] = a;
                P.inhIn[c0 + lane] = 0.f;
            }
        }
        if (last == W - 1 && colc) {
            const int j = c0 + lane;
            P.v[j] = v;
            P.gExc[j] = ge;
            P.gInh[j] = gi;
            P.nanFlag[j] = static_cast<uint8_t>(flag | (expMax == 0x7f800000u));
            T.y[j] = y;
            if (!flag && expMax == 0x7f800000u) atomicAdd(P.flagged, 1ull);
        }
        (void)s_red;
        (void)bad;
        (void)tr;
        (void)trBase;
        return;
    }
    if (warp == 8) {
        // the notifier: once a step's post spikes are out, tell the background
        // blocks (its fence stays off the chains' and the producers' paths)
        for (int w = 0; w < W; ++w) {
            mbar_wait(&s_dn[w & 1], (w >> 1) & 1);
            __syncwarp();
            if (lane == 0) {
                __threadfence();
                atomicAdd(T.sinkDone + w, 1);
                mbar_arrive(&s_pdone[w & 1]);
            }
            __syncwarp();
        }
        return;
    }
    if (!producer) return;
    // ---- producers: stage each step's rows (a step ahead of the chains),
    //      then, once the step's post spikes are out, its learning.  A step's
    //      weights load during the step before (only rows that spiked at that
    //      step change in between: their learned values come from s_learn).
    SinkRow rec[kSinkPre], recN[kSinkPre];
    float v[kSinkPre][kSinkCols], vN[kSinkPre][kSinkCols];
    int cntCur = W > 0 && !(T.skip & 1) ? T.preCnt[0] : 0;
    if (W > 0) {
        sink_fetch_all<kSinkPre>(T, 0, i, kSinkRows, cntCur, s_bitRing, rec);
#pragma unroll
        for (int kk = 0; kk < kSinkPre; ++kk) {
            s_idx[0][kk][i] = rec[kk].r >= 0 ? rec[kk].r + T.preOffset : INT_MAX;
#pragma unroll
            for (int j = 0; j < kSinkCols; ++j)
                v[kk][j] = rec[kk].r >= 0 && j < nc ? __ldcg(T.WT + (size_t)(c0 + j) * nPre + rec[kk].r) : 0.f;
        }
        ring_load(T, s_bitRing, 0, i, kSinkRows);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kSinkRows));
    int gr0 = 0, gr1 = 0, cntPrev = 0;  // chunk sequence numbers of the two rings
    for (int w = 0; w < W; ++w) {
        const int cnt = cntCur;
        const int nCh = (cnt + kSinkRows - 1) / kSinkRows;
        const int nextCnt = w + 1 < W && !(T.skip & 1) ? __ldg(T.preCnt + w + 1) : 0;
        // the background's step w - L (the next step's weights wait for it),
        // read early; the next step's row indices and pre spike bits, copied
        // asynchronously (read-only; indices past the count are never read)
        const int bgEarly = w + 1 > kSinkLag && w + 1 < W
                                ? *reinterpret_cast<const volatile int*>(T.bgDone + (w - kSinkLag)) : 0;
        if (w + 1 < W) {
            const int* Ln = T.preList + (size_t)(w + 1) * T.preN;
#pragma unroll
            for (int kk = 0; kk < kSinkPre; ++kk)
                if (kk * kSinkRows + i < T.preN) cp_async4(&s_idx[(w + 1) % 3][kk][i], Ln + kk * kSinkRows + i);
            const uint32_t* pb = T.preBits + (size_t)(w + 1) * T.preWords;
            uint32_t* dst = s_bitRing + ((w + 1) % kSinkRing) * T.preWords;
            for (int k = i; k < T.preWords; k += kSinkRows) cp_async4(dst + k, pb + k);
            cp_async_commit();
        }
        // rows that spiked at w - 1 too: their weights after that step's learning
        if (w > 0) {
            const int* prevIdx = &s_idx[(w - 1) % 3][0][0];  // step w - 1's rows, ascending
            const int nPrev = min(cntPrev, kSinkPre * kSinkRows);
#pragma unroll
            for (int kk = 0; kk < kSinkPre; ++kk) {
                if (rec[kk].r < 0 || !(rec[kk].hist & 1u)) continue;
                const int key = rec[kk].r + T.preOffset;
                int lo = 0, hi = nPrev;  // first position with prevIdx >= key
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (prevIdx[mid] < key) lo = mid + 1;
                    else hi = mid;
                }
#pragma unroll
                for (int j = 0; j < kSinkCols; ++j)
                    v[kk][j] = j >= nc ? 0.f
                               : lo < nPrev && prevIdx[lo] == key
                                   ? s_learn[(w - 1) & 1][j][lo]
                                   : __ldcg(T.WT + (size_t)(c0 + j) * nPre + rec[kk].r);  // on-demand row
            }
        }
        // stage the fetched chunks (s_hist of the steps before w is final: the
        // producers waited for the post update of w - 1)
        float xdw[kSinkPre];
#pragma unroll
        unsigned long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (tr) tp[0] = global_ns();
        const int ring = w & 1;
        const int g = ring ? gr1 : gr0;
        for (int kk = 0; kk < kSinkPre; ++kk) {
            if (kk >= nCh) break;
            const int gg = g + kk, b = gg % kSinkBufs;
            xdw[kk] = 0.f;
            if (rec[kk].r >= 0) sink_stage(T, w, rec[kk], v[kk], s_hist, xdw[kk]);
            if (gg >= kSinkBufs) mbar_wait(&s_empty[ring][b], ((gg / kSinkBufs) - 1) & 1);
            const bool live = kk * kSinkRows + i < cnt;
#pragma unroll
            for (int j = 0; j < kSinkCols; ++j)
                s_stage[ring][b][j][i] = live && rec[kk].r >= 0 ? v[kk][j] : 0.f;
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_full[ring][b]);
        }
        if (tr) tp[1] = global_ns();  // staged
        // the step's post spikes, then its learning
        mbar_wait(&s_dn[w & 1], (w >> 1) & 1);
        if (tr) tp[2] = global_ns();  // post spikes out
        const uint32_t spk = s_hist[w];
        const float yd[kSinkCols] = {s_yd[w & 1][0], s_yd[w & 1][1]};
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_pdone[w & 1]);
#pragma unroll
        for (int kk = 0; kk < kSinkPre; ++kk) {
            if (kk >= nCh || kk * kSinkRows + i >= cnt || rec[kk].r < 0) continue;
            float lw[kSinkCols];
            sink_learn(T, rec[kk], v[kk], xdw[kk], c0, nc, spk, yd, lw);
#pragma unroll
            for (int j = 0; j < kSinkCols; ++j) s_learn[w & 1][j][kk * kSinkRows + i] = lw[j];
        }
        if (tr) tp[3] = global_ns();  // learned
        for (int k = kSinkPre; k < nCh; ++k) {  // beyond the fetched chunks: on demand
            const int gg = g + k, b = gg % kSinkBufs;
            const int e = k * kSinkRows + i;
            const SinkRow q = sink_fetch(T, w, e, cnt, s_bitRing);
            float vv[kSinkCols] = {0.f, 0.f};
            float xw = 0.f;
            if (q.r >= 0) {
#pragma unroll
                for (int j = 0; j < kSinkCols; ++j)
                    vv[j] = j < nc ? __ldcg(T.WT + (size_t)(c0 + j) * nPre + q.r) : 0.f;
                sink_stage(T, w, q, vv, s_hist, xw);
            }
            if (gg >= kSinkBufs) mbar_wait(&s_empty[ring][b], ((gg / kSinkBufs) - 1) & 1);
#pragma unroll
            for (int j = 0; j < kSinkCols; ++j) s_stage[ring][b][j][i] = q.r >= 0 ? vv[j] : 0.f;
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_full[ring][b]);
            float lw[kSinkCols];
            if (q.r >= 0) sink_learn(T, q, vv, xw, c0, nc, spk, yd, lw);
        }
        if (ring) gr1 += nCh;
        else gr0 += nCh;
        if (w + 1 < W) {
            // the next step's rows from the copies issued above, and their
            // weights: final except for the rows spiking now (fixed up above
            // from s_learn) once the background's step w - L is in
            cp_async_wait<0>();
#pragma unroll
            for (int kk = 0; kk < kSinkPre; ++kk) {
                const int e = kk * kSinkRows + i;
                recN[kk] = e < nextCnt ? sink_fetch_row(T, w + 1, s_idx[(w + 1) % 3][kk][i], s_bitRing)
                                       : SinkRow{};
            }
            if (tr) tp[4] = global_ns();  // fetched
            if (w + 1 > kSinkLag && bgEarly < static_cast<int>(gridDim.x) - T.nSink)
                spin_until(T.bgDone + (w - kSinkLag), gridDim.x - T.nSink);
            if (tr) tp[5] = global_ns();  // background in
#pragma unroll
            for (int kk = 0; kk < kSinkPre; ++kk)
#pragma unroll
                for (int j = 0; j < kSinkCols; ++j)
                    vN[kk][j] = recN[kk].r >= 0 && j < nc
                                    ? __ldcg(T.WT + (size_t)(c0 + j) * nPre + recN[kk].r) : 0.f;
        }
        cntPrev = cnt;
        cntCur = nextCnt;
#pragma unroll
        for (int kk = 0; kk < kSinkPre; ++kk) {
            rec[kk] = recN[kk];
#pragma unroll
            for (int j = 0; j < kSinkCols; ++j) v[kk][j] = vN[kk][j];
        }
        // every producer's learning of w (s_learn, the weights) and ring slot
        // w + 1 in before step w + 1 is staged
        asm volatile("bar.sync 1, %0;" ::"r"(kSinkRows));
        if (g_watch && t == 32) g_watch[2 * T.nSink + blockIdx.x] = w;
        if (tr && trBase + w < g_traceCap) {
            tp[6] = global_ns();  // barrier passed
            unsigned long long* e = g_trace + 4ull * (trBase + w);
            e[0] = 0x5200ull | (static_cast<unsigned long long>(cnt) << 32);
            e[1] = tp[0];
            e[2] = (tp[1] - tp[0]) | ((tp[2] - tp[0]) << 16) | ((tp[3] - tp[0]) << 32) | ((tp[4] - tp[0]) << 48);
            e[3] = (tp[5] - tp[0]) | ((tp[6] - tp[0]) << 16);
        }
    }
}
