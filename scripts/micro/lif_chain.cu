// Microbenchmark (diagnostic): cycles per step of the conductance-LIF
// recurrence of one warp (lif_step of kernels.cuh), inputs in shared memory;
// the latency chain that bounds the single-block populations (LHI, DN).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1412_0595_b200/csrc/device/kernels.cuh"
using namespace ssbk;

template <bool kExact>
__global__ void chain(const float* g, float* out, int steps, long long* cyc, PopDev P) {
    __shared__ float s_in[2][256];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) (&s_in[0][0])[i] = g[i];
    __syncthreads();
    const LifConst lc = lif_const(P);
    float v = -60.f, ge = 0.f, gi = 0.f;
    uint32_t em = 0, mine = 0, bad = 0;
    const int lane = threadIdx.x & 31;
    long long t0 = clock64();
    for (int r = 0; r < steps; r += 256) {
#pragma unroll 4
        for (int wl = 0; wl < 256; ++wl) {
            const bool spike = lif_step<kExact>(lc, s_in[0][wl], s_in[1][wl], v, ge, gi, em, bad);
            const unsigned b = __ballot_sync(0xffffffffu, spike);
            mine = lane == (wl & 31) ? b : mine;
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = v + ge + gi + (float)em + (float)mine + (float)bad;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    float *g, *o; long long* c;
    cudaMalloc(&g, 512 * 4); cudaMalloc(&o, 1024 * 4); cudaMalloc(&c, 8);
    float h[512];
    for (int i = 0; i < 512; ++i) h[i] = (i % 7) * 0.01f;
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    PopDev P{};
    P.synDecay = 0.98f; P.eLeak = -60.f; P.tauM = 10.f; P.eExc = 0.f; P.eInh = -80.f;
    P.dt = 0.1f; P.vThresh = -45.f; P.vReset = -60.f;
    const int steps = 256 * 64;
    long long cy;
    chain<true><<<1, 32>>>(g, o, steps, c, P);
    chain<true><<<1, 32>>>(g, o, steps, c, P);
    cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    printf("one warp, exact division (branch per step): %.1f cycles per LIF step\n", (double)cy / steps);
    chain<false><<<1, 32>>>(g, o, steps, c, P);
    chain<false><<<1, 32>>>(g, o, steps, c, P);
    cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    printf("one warp, branch-free division + range flag: %.1f cycles per LIF step\n", (double)cy / steps);
    return 0;
}
