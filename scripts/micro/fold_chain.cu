// Microbenchmark (diagnostic): cycles per row of a dependent fp32 add chain
// over rows staged in shared memory, one folding warp per block; variants of
// the fold loop's load scheduling.
#include <cstdio>
#include <cuda_runtime.h>
template <int NP, int V>
__global__ void fold(const float* __restrict__ g, float* out, int rows, long long* cyc) {
    __shared__ float ring[256 * NP];
    for (int i = threadIdx.x; i < 256 * NP; i += blockDim.x) ring[i] = g[i];
    __syncthreads();
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    float a = 0.f;
    long long t0 = clock64();
    if (lane < NP) {
        const float* src = ring + lane;
        for (int base = 0; base < rows; base += 256) {
            if (V == 0) {
#pragma unroll 8
                for (int u = 0; u < 256; ++u) a = __fadd_rn(a, src[u * NP]);
            } else if (V == 1) {  // groups of 16, next group's loads interleaved
                float x[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) x[k] = src[k * NP];
#pragma unroll 1
                for (int g0 = 0; g0 < 256; g0 += 16) {
                    float y[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        y[k] = src[((g0 + 16 + k) & 255) * NP];
                        a = __fadd_rn(a, x[k]);
                    }
#pragma unroll
                    for (int k = 0; k < 16; ++k) x[k] = y[k];
                }
            } else if (V == 2) {  // fully unrolled stage
#pragma unroll
                for (int u = 0; u < 256; ++u) a = __fadd_rn(a, src[u * NP]);
            } else {  // float4 loads of 4 rows' worth? (two chains per lane impossible) -- group 32
                float x[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) x[k] = src[k * NP];
#pragma unroll 1
                for (int g0 = 0; g0 < 256; g0 += 32) {
                    float y[32];
#pragma unroll
                    for (int k = 0; k < 32; ++k) {
                        y[k] = src[((g0 + 32 + k) & 255) * NP];
                        a = __fadd_rn(a, x[k]);
                    }
#pragma unroll
                    for (int k = 0; k < 32; ++k) x[k] = y[k];
                }
            }
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * 32 + lane] = a;
    if (lane == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int V>
void run(float* g, float* o, long long* c) {
    const int rows = 12800, blocks = 256;
    fold<16, V><<<blocks, 128>>>(g, o, rows, c);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    fold<16, V><<<blocks, 128>>>(g, o, rows, c);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h[1024]; cudaMemcpy(h, c, blocks * 8, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < blocks; ++i) avg += h[i]; avg /= blocks;
    printf("variant %d: %.1f us, %.2f cycles/row\n", V, ms * 1e3, avg / rows);
}
int main() {
    float *g, *o; long long* c;
    cudaMalloc(&g, 256 * 32 * 4); cudaMemset(g, 0, 256 * 32 * 4);
    cudaMalloc(&o, 1024 * 32 * 4); cudaMalloc(&c, 1024 * 8);
    run<0>(g, o, c); run<1>(g, o, c); run<2>(g, o, c); run<3>(g, o, c);
    return 0;
}
