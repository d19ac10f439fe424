// gather_tma.cuh — heavy dense group inputs (kc_dn: 100k KC rows x 100 DN
// columns) with TMA row gathers (included inside namespace ssbk::<unnamed> by
// kernels.cuh; reference propagate(Dense), engine.cpp:53-67, in the order of
// engine.cpp:343-353).
//
// One warp folds one window step: post column j's input is the left fold,
// from +0, of W[r][j] over the step's spiking pre rows r in ascending order
// (one dependent add chain per column, as long as the step's spike count).
// The rows reach shared memory through cp.async.bulk.tensor ... tile::gather4:
// one instruction brings four whole rows (4 x nPost floats) named by their row
// indices into a stage of the warp's ring, completing on the stage's
// mbarrier; lane 0 issues, lanes fold columns 4l..4l+3 with 16-byte loads.
// No copier threads: a block of 8 warps (8 steps in flight) takes ~77 KB of
// shared memory and 256 threads, so it fits on an SM beside a KC update block
// instead of holding SMs the next window's update waits for.  Rows outside
// the group's pre window get the out-of-range row index preCount, which the
// TMA unit fills with +0 (exact: the folds start at +0 and never hold -0).
constexpr int kTmaWarps = 8;   // steps in flight per block
constexpr int kTmaStages = 6;  // four-row stages per warp

// floats per stage (four rows, padded to 128 bytes) and the kernel's shared bytes
__host__ __device__ __forceinline__ int tma_stage_floats(int np) { return (4 * np + 31) / 32 * 32; }
__host__ __device__ __forceinline__ int tma_smem_bytes(int np) {
    return kTmaWarps * kTmaStages * tma_stage_floats(np) * 4 + 128;
}

__device__ __forceinline__ void tma_gather4(void* dst, const void* tmap, int col, int r0, int r1,
                                            int r2, int r3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_addr(dst)),
        "l"(tmap), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}

// nPost = NP: a multiple of 4, <= 128 (lane l folds columns 4l..4l+3)
__global__ void __launch_bounds__(32 * kTmaWarps) dense_window_tma_kernel(
    const __grid_constant__ CUtensorMap tmap, GroupDev G, float* __restrict__ out,
    long long outStride, int wLo, int nW, int first) {
    const int NP = G.nPost;
    extern __shared__ __align__(128) float s_ring[];  // [warp][stage][4][NP]
    __shared__ __align__(8) uint64_t full[kTmaWarps][kTmaStages];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned long long tStart = g_trace ? global_ns() : 0ull;
    const uint32_t kStageBytes = 4u * NP * 4u;
    // stages start on 128-byte boundaries (tensor TMA destinations)
    const int stageF = tma_stage_floats(NP);
    float* aligned = reinterpret_cast<float*>(
        (reinterpret_cast<uintptr_t>(s_ring) + 127) & ~static_cast<uintptr_t>(127));
    float* ring = aligned + (size_t)warp * kTmaStages * stageF;
    if (lane == 0) {
        for (int i = 0; i < kTmaStages; ++i) mbar_init(&full[warp][i], 1);
        mbar_fence_init();
    }
    __syncwarp();
    const bool act = 4 * lane < NP;
    uint32_t phases = 0;  // parity of each stage's next completion
    for (int s = blockIdx.x * kTmaWarps + warp; s < nW; s += gridDim.x * kTmaWarps) {
        const int w = wLo + s;
        const int cnt = G.preCnt[w - 1];
        const int* __restrict__ L = G.preList + (size_t)(w - 1) * G.preN;
        const int ng = (cnt + 3) >> 2;
        // row indices, 32 at a time (lane i holds entry 32 b + i), one block ahead
        auto rows_of = [&](int b) {
            const int q = 32 * b + lane;
            int r = q < cnt ? L[q] - G.preOffset : -1;
            return (unsigned)r < (unsigned)G.preCount ? r : G.preCount;  // OOB row -> zeros
        };
        int blk = 0, cur = rows_of(0), nxt = rows_of(1);
        auto issue = [&](int g) {  // all lanes (shuffles), lane 0 issues
            const int b = g >> 3;
            while (blk < b) {
                cur = nxt;
                ++blk;
                nxt = rows_of(blk + 1);
            }
            const int o = (g & 7) * 4;
            const int r0 = __shfl_sync(kFull, cur, o), r1 = __shfl_sync(kFull, cur, o + 1);
            const int r2 = __shfl_sync(kFull, cur, o + 2), r3 = __shfl_sync(kFull, cur, o + 3);
            if (lane == 0) {
                const int slot = g % kTmaStages;
                uint64_t* bar = &full[warp][slot];
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                                 smem_addr(bar)),
                             "r"(kStageBytes)
                             : "memory");
                tma_gather4(ring + (size_t)slot * stageF, &tmap, 0, r0, r1, r2, r3, bar);
            }
        };
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        float* o = out + (size_t)s * outStride;
        if (!first && act) a = *reinterpret_cast<const float4*>(o + 4 * lane);
        const int pre = min(ng, kTmaStages);
        for (int g = 0; g < pre; ++g) issue(g);
        for (int g = 0; g < ng; ++g) {
            const int slot = g % kTmaStages;
            const uint32_t ph = (phases >> slot) & 1u;
            while (!mbar_try(&full[warp][slot], ph)) {
            }
            phases ^= 1u << slot;
            if (act) {
                const float* st = ring + (size_t)slot * stageF + 4 * lane;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float4 x = *reinterpret_cast<const float4*>(st + k * NP);
                    a.x = __fadd_rn(a.x, x.x);
                    a.y = __fadd_rn(a.y, x.y);
                    a.z = __fadd_rn(a.z, x.z);
                    a.w = __fadd_rn(a.w, x.w);
                }
            }
            __syncwarp();  // the stage is consumed before it is refilled
            if (g + kTmaStages < ng) issue(g + kTmaStages);
        }
        if (act) *reinterpret_cast<float4*>(o + 4 * lane) = a;
    }
    if (threadIdx.x == 0) trace_block(0xfffffffcull, tStart);
}

// The same fold with the rows streamed through registers: lane l loads its
// 16 bytes of each row (one coalesced 400-byte row per warp instruction),
// eight rows per batch and the next batch in flight while this one is
// folded.  No shared memory: a block of 8 warps fits beside a KC block.
__global__ void __launch_bounds__(256) dense_window_ldg_kernel(GroupDev G, float* __restrict__ out,
                                                               long long outStride, int wLo,
                                                               int nW, int first) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned long long tStart = g_trace ? global_ns() : 0ull;
    const int NP = G.nPost;
    const bool act = 4 * lane < NP;
    const float* __restrict__ Wb = G.W + 4 * (act ? lane : 0);
    for (int s = blockIdx.x * 8 + warp; s < nW; s += gridDim.x * 8) {
        const int w = wLo + s;
        const int cnt = G.preCnt[w - 1];
        const int* __restrict__ L = G.preList + (size_t)(w - 1) * G.preN;
        auto rows_of = [&](int blk) {  // lane i: entry 32 blk + i (-1: contributes +0)
            const int q = 32 * blk + lane;
            const int r = q < cnt ? L[q] - G.preOffset : -1;
            return (unsigned)r < (unsigned)G.preCount ? r : -1;
        };
        int blk = 0, cur = rows_of(0), nxt = rows_of(1);
        auto load = [&](int b, float4 (&x)[8]) {  // rows 8b .. 8b+7 (all lanes)
            while (blk < (b >> 2)) {
                cur = nxt;
                ++blk;
                nxt = rows_of(blk + 1);
            }
            const int o = (b & 3) * 8;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int r = __shfl_sync(kFull, cur, o + k);
                x[k] = (r >= 0 && act) ? __ldg(reinterpret_cast<const float4*>(Wb + (size_t)r * NP))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        };
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        float* o = out + (size_t)s * outStride;
        if (!first && act) a = *reinterpret_cast<const float4*>(o + 4 * lane);
        const int nb = (cnt + 7) >> 3;
        float4 xa[8], xb[8];
        if (nb > 0) load(0, xa);
        for (int b = 0; b < nb; b += 2) {
            if (b + 1 < nb) load(b + 1, xb);
#pragma unroll
            for (int k = 0; k < 8; ++k) {  // rows past the count are +0 (exact)
                a.x = __fadd_rn(a.x, xa[k].x);
                a.y = __fadd_rn(a.y, xa[k].y);
                a.z = __fadd_rn(a.z, xa[k].z);
                a.w = __fadd_rn(a.w, xa[k].w);
            }
            if (b + 1 >= nb) break;
            if (b + 2 < nb) load(b + 2, xa);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                a.x = __fadd_rn(a.x, xb[k].x);
                a.y = __fadd_rn(a.y, xb[k].y);
                a.z = __fadd_rn(a.z, xb[k].z);
                a.w = __fadd_rn(a.w, xb[k].w);
            }
        }
        if (act) *reinterpret_cast<float4*>(o + 4 * lane) = a;
    }
    if (threadIdx.x == 0) trace_block(0xfffffffcull, tStart);
}

// ---- row streaming (heavy dense groups into few post columns: kc_dn) --------
// The fold of column j at window step s walks the step's spiking pre rows in
// ascending order.  Instead of gathering each step's rows (every spiking row
// re-read at each of its ~3.6 spikes per 256-step window, 140 MB per window
// at config 3), stream the weight matrix once per window in ascending row
// order and let every step take the rows it spiked on as they pass: for any
// (step, column) the adds still arrive in ascending row order, so the folds
// are bit-identical, and the matrix is read once (~40 MB) by TMA tile loads
// (2D boxes of 256 rows x 8 columns) instead of 350k random row gathers.
// Block = 8 post columns x (up to) 256 window steps, thread = one step (its 8
// accumulators in registers); the rows pass through a double-buffered stage
// of kRsRows rows; a thread walks its step's spike list (ascending) along.
constexpr int kRsCols = 8;        // post columns per block (TMA box width: 32 bytes)
constexpr int kRsBox = 256;       // rows per TMA box (the box-size limit)
constexpr int kRsRows = 1024;     // rows per stage (4 boxes, 32 KB)
constexpr int kRsStages = 2;
constexpr int kRsThreads = 256;   // window steps per block
constexpr int kRsSmem = kRsStages * kRsRows * kRsCols * 4 + 128;

__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int r0,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_addr(dst)),
        "l"(tmap), "r"(c0), "r"(r0), "r"(smem_addr(bar))
        : "memory");
}

__global__ void __launch_bounds__(kRsThreads) dense_window_rowstream_kernel(
    const __grid_constant__ CUtensorMap tmap, GroupDev G, float* __restrict__ out,
    long long outStride, int wLo, int nW, int first) {
    extern __shared__ __align__(128) float s_rs[];
    __shared__ __align__(8) uint64_t full[kRsStages];
    float* stage0 = reinterpret_cast<float*>(
        (reinterpret_cast<uintptr_t>(s_rs) + 127) & ~static_cast<uintptr_t>(127));
    const int t = threadIdx.x;
    const unsigned long long tStart = g_trace ? global_ns() : 0ull;
    const int c0 = blockIdx.x * kRsCols;
    const int s = blockIdx.y * kRsThreads + t;  // this thread's window step
    const bool live = s < nW;
    const int nRows = G.preCount;
    const int nStages = (nRows + kRsRows - 1) / kRsRows;
    constexpr uint32_t kStageBytes = kRsRows * kRsCols * 4;
    if (t == 0) {
        for (int i = 0; i < kRsStages; ++i) mbar_init(&full[i], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int k) {  // thread 0: stage k's rows into buffer k % kRsStages
        float* dst = stage0 + (size_t)(k % kRsStages) * kRsRows * kRsCols;
        uint64_t* bar = &full[k % kRsStages];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                     "r"(kStageBytes)
                     : "memory");
        for (int b = 0; b < kRsRows / kRsBox; ++b)
            tma_load_2d(dst + b * kRsBox * kRsCols, &tmap, c0, k * kRsRows + b * kRsBox, bar);
    };
    if (t == 0)
        for (int k = 0; k < min(kRsStages, nStages); ++k) issue(k);

    // this step's spike list, four entries per load, three loads ahead
    const int cnt = live ? G.preCnt[wLo + s - 1] : 0;
    const int* __restrict__ L = G.preList + (size_t)(wLo + s - 1) * G.preN;
    auto fetch = [&](int e4) {  // entries 4 e4 .. 4 e4 + 3 (rows; INT_MAX past the end)
        int4 q = make_int4(INT_MAX, INT_MAX, INT_MAX, INT_MAX);
        if (4 * e4 < cnt) {
            if (4 * e4 + 3 < cnt) {
                q = __ldg(reinterpret_cast<const int4*>(L) + e4);
            } else {
                q.x = L[4 * e4];
                if (4 * e4 + 1 < cnt) q.y = L[4 * e4 + 1];
                if (4 * e4 + 2 < cnt) q.z = L[4 * e4 + 2];
            }
        }
        return q;
    };
    int4 qa = fetch(0), qb = fetch(1), qc = fetch(2), qd = fetch(3);
    int e = 0;  // next entry
    auto entry = [&](int i) {
        const int k = i & 3;
        return k == 0 ? qa.x : k == 1 ? qa.y : k == 2 ? qa.z : qa.w;
    };
    float acc[kRsCols];
    {
        const float* o = out + (size_t)s * outStride + c0;
#pragma unroll
        for (int j = 0; j < kRsCols; ++j)
            acc[j] = (!first && live && c0 + j < G.nPost) ? o[j] : 0.f;
    }
    int r = cnt > 0 ? entry(0) - G.preOffset : INT_MAX;
    for (int k = 0; k < nStages; ++k) {
        mbar_wait(&full[k % kRsStages], (k / kRsStages) & 1);
        const float* st = stage0 + (size_t)(k % kRsStages) * kRsRows * kRsCols;
        const int lo = k * kRsRows, hi = lo + kRsRows;
        while (r < hi) {
            if (r >= 0 && r < nRows) {  // rows outside the pre window add nothing
                const float4 x0 = *reinterpret_cast<const float4*>(st + (r - lo) * kRsCols);
                const float4 x1 = *reinterpret_cast<const float4*>(st + (r - lo) * kRsCols + 4);
                acc[0] = __fadd_rn(acc[0], x0.x);
                acc[1] = __fadd_rn(acc[1], x0.y);
                acc[2] = __fadd_rn(acc[2], x0.z);
                acc[3] = __fadd_rn(acc[3], x0.w);
                acc[4] = __fadd_rn(acc[4], x1.x);
                acc[5] = __fadd_rn(acc[5], x1.y);
                acc[6] = __fadd_rn(acc[6], x1.z);
                acc[7] = __fadd_rn(acc[7], x1.w);
            }
            ++e;
            if ((e & 3) == 0) {  // next four entries; fetch four ahead
                qa = qb;
                qb = qc;
                qc = qd;
                qd = fetch((e >> 2) + 3);
            }
            r = e < cnt ? entry(e) - G.preOffset : INT_MAX;
        }
        __syncthreads();  // everyone is past this buffer
        if (t == 0 && k + kRsStages < nStages) issue(k + kRsStages);
    }
    if (live) {
        float* o = out + (size_t)s * outStride + c0;
#pragma unroll
        for (int j = 0; j < kRsCols; ++j)
            if (c0 + j < G.nPost) o[j] = acc[j];
    }
    if (t == 0) trace_block(0xfffffffcull, tStart);
}

// ---- CRS propagate over column slices (reference propagate(Crs),
//      engine.cpp:69-80) --------------------------------------------------------
// The matrix re-laid once (host, ssb_crs_slices) as slices of 32 post columns:
// slice s holds, for k = 0 .. len_s - 1 and lane l, the k-th entry of column
// 32 s + l (its pre row and value; row -1 pads a shorter column), rows
// ascending within a column.  Lane l folds column 32 s + l over its entries
// whose row is spiking (a bitmask in shared memory), so every load of the
// kernel is a coalesced 128-byte line and every column's adds arrive in
// ascending row order: bit-identical to the reference's row-by-row scatter
// for a spike list in ascending order without repeats (the engine's lists).
__global__ void __launch_bounds__(256) propagate_crs_sliced_kernel(
    const int* __restrict__ rows, const float* __restrict__ vals,
    const long long* __restrict__ sliceOff, int nPre, int nPost, const int* __restrict__ spikes,
    int nSpikes, float* __restrict__ acc) {
    extern __shared__ uint32_t s_spk[];  // [(nPre + 31) / 32]
    const int nw = (nPre + 31) >> 5;
    for (int i = threadIdx.x; i < nw; i += blockDim.x) s_spk[i] = 0u;
    __syncthreads();
    for (int k = threadIdx.x; k < nSpikes; k += blockDim.x) {
        const int r = spikes[k];
        if ((unsigned)r < (unsigned)nPre) atomicOr(&s_spk[r >> 5], 1u << (r & 31));
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int nSlices = (nPost + 31) >> 5;
    for (int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < nSlices;
         s += gridDim.x * (blockDim.x >> 5)) {
        const int j = s * 32 + lane;
        const long long base = sliceOff[s];
        const int len = static_cast<int>((sliceOff[s + 1] - base) >> 5);
        const int* __restrict__ R = rows + base + lane;
        const float* __restrict__ V = vals + base + lane;
        float a = j < nPost ? acc[j] : 0.f;
        int k = 0;
        constexpr int U = 16;  // loads in flight per lane (DRAM latency x bandwidth)
        for (; k < len; k += U) {  // the last round predicated (no load-by-load tail)
            int r[U];
            float v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool in = k + u < len;
                r[u] = in ? __ldg(R + (k + u) * 32) : -1;
                v[u] = in ? __ldg(V + (k + u) * 32) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (r[u] >= 0 && ((s_spk[r[u] >> 5] >> (r[u] & 31)) & 1u)) a = __fadd_rn(a, v[u]);
        }
        if (j < nPost) acc[j] = a;
    }
}
