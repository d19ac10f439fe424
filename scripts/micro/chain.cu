// Floor of a dependent fp32 add chain fed from shared memory (the sink
// kernel's column fold): cycles per element, one warp, two active lanes.
#include <cstdio>
constexpr int C = 2;
__global__ void chain(int n, float* out, long long* cyc) {
    __shared__ float s[2048][C];
    for (int i = threadIdx.x; i < 2048 * C; i += blockDim.x) (&s[0][0])[i] = 1e-3f * (i % 97);
    __syncthreads();
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    float a = 0.f;
    long long t0 = clock64();
    if (lane < C) {
        const float* sb = &s[0][lane];
        const int n8 = n & ~7;
        float c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = sb[u * C];
        for (int q = 8; q < n8; q += 8) {
            float d[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) d[u] = sb[(q + u) * C];
#pragma unroll
            for (int u = 0; u < 8; ++u) a = __fadd_rn(a, c[u]);
#pragma unroll
            for (int u = 0; u < 8; ++u) c[u] = d[u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) a = __fadd_rn(a, c[u]);
    }
    __syncwarp();
    long long t1 = clock64();
    if (lane == 0) { out[0] = a; cyc[0] = t1 - t0; }
}
__global__ void chain_reg(int n, float* out, long long* cyc) {
    float a = 0.f, b = threadIdx.x * 1e-3f;
    long long t0 = clock64();
    for (int q = 0; q < n; q += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) a = __fadd_rn(a, b);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = a; cyc[0] = t1 - t0; }
}
int main() {
    float* out; long long* cyc; cudaMalloc(&out, 4); cudaMalloc(&cyc, 8);
    for (int n : {480, 1440}) {
        long long h;
        chain<<<1, 512>>>(n, out, cyc); cudaDeviceSynchronize();
        chain<<<1, 512>>>(n, out, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("smem chain n %d: %.2f cycles/elem\n", n, (double)h / n);
        chain_reg<<<1, 32>>>(n, out, cyc); cudaDeviceSynchronize();
        chain_reg<<<1, 32>>>(n, out, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("reg chain n %d: %.2f cycles/elem\n", n, (double)h / n);
    }
    return 0;
}
