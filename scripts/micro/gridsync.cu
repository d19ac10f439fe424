// Grid barrier cost on B200: cooperative_groups grid.sync vs a hand-rolled
// sense-reversal barrier (one arriving thread per block), 148 x 512 threads.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void cg_sync(int n, int* out) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < n; ++i) g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = n;
}

__device__ __forceinline__ void bar(unsigned* count, volatile unsigned* gen, unsigned nb, unsigned& my) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned target = my + 1;
        __threadfence();
        if (atomicAdd(count, 1u) == nb - 1) {
            *count = 0;
            __threadfence();
            atomicExch(const_cast<unsigned*>(gen), target);
        } else {
            while (*gen != target) {}
        }
        __threadfence();
    }
    ++my;
    __syncthreads();
}

__global__ void own_sync(int n, unsigned* count, unsigned* gen) {
    unsigned my = *(volatile unsigned*)gen;
    for (int i = 0; i < n; ++i) bar(count, gen, gridDim.x, my);
}

int main() {
    int* out; unsigned* cnt; unsigned* gen;
    cudaMalloc(&out, 4); cudaMalloc(&cnt, 4); cudaMalloc(&gen, 4);
    cudaMemset(cnt, 0, 4); cudaMemset(gen, 0, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int grid : {50, 100, 148}) {
        int n = 2560;
        void* args[] = {&n, &out};
        cudaLaunchCooperativeKernel((void*)cg_sync, grid, 512, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)cg_sync, grid, 512, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        void* args2[] = {&n, &cnt, &gen};
        cudaLaunchCooperativeKernel((void*)own_sync, grid, 512, args2, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)own_sync, grid, 512, args2, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms2; cudaEventElapsedTime(&ms2, a, b);
        printf("grid %d: cg %.3f us/sync, own %.3f us/sync (%s)\n", grid, ms * 1e3 / n, ms2 * 1e3 / n,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
