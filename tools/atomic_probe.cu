// atomic_probe.cu — same-address atomicAdd throughput on the B200, the
// pattern of the stage-1 queue counter (one u64 atomic per warp step,
// ~780 K per config-B frame).  Experiment for DESIGN.md §7; not shipped.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomic_probe atomic_probe.cu
// Prints the time of 780 K warp-aggregated atomics spread over 1, 2, 8 or 32
// counters (each on its own 256-byte line), with a little work between them.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void __launch_bounds__(256, 4) k_atom(unsigned long long *ctr, int lines, int64_t total, float *sink) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float acc = 0.0f;
    unsigned long long *c = ctr + 32 * (warp % lines);
    for (int64_t s = warp; s < total; s += nw) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(c, 13ull);
        base = __shfl_sync(0xffffffffu, base, 0);
        acc += (float)(base & 7);
#pragma unroll 8
        for (int k = 0; k < 64; ++k) acc = __fmaf_rn(acc, 0.999f, 1.0f);   // ~0.7 us of filter-like ALU work per step
    }
    if (acc == 123.456f) sink[0] = acc;
}

int main() {
    unsigned long long *ctr;
    float *sink;
    cudaMalloc(&ctr, 32 * 64 * 8);
    cudaMalloc(&sink, 16);
    cudaMemset(ctr, 0, 32 * 64 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int64_t total = 780000;
    const int lines_list[4] = {1, 2, 8, 32};
    for (int rep = 0; rep < 3; ++rep) {
        for (int li = 0; li < 4; ++li) {
            const int lines = lines_list[li];
            k_atom<<<148 * 4, 256>>>(ctr, lines, total, sink);
            cudaEventRecord(e0);
            for (int it = 0; it < 10; ++it) k_atom<<<148 * 4, 256>>>(ctr, lines, total, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("lines %2d  %.4f ms per 780K atomics\n", lines, ms / 10);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
