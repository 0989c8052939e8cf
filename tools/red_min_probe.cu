// red_min_probe.cu — peak L2 throughput of 64-bit unsigned atomicMin with
// an unused result (REDG.E.MIN.64.STRONG.GPU, the visibility-buffer merge
// of kernels.py:40-46) on the B200, as the denominator for the stage
// kernels' measured L2 reduction rate (ncu lts__t_requests_op_red).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_min_probe red_min_probe.cu
// Patterns over a 3840x2160 uint64 buffer (66 MB, L2-resident):
//   scattered  each thread merges into pseudo-random pixels
//   rows       a warp merges 32 consecutive pixels (coalesced, 2 lines)
//   tile       a warp merges an 8x4 pixel block (stage-3-like)
// Prints merges/s and the per-kernel time.  Experiment tool; not shipped.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_red(unsigned long long *fb, int W, int H, int64_t per_thread,
                                             uint32_t salt) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int64_t warp = tid >> 5;
    const int64_t npix = (int64_t)W * H;
    for (int64_t k = 0; k < per_thread; ++k) {
        int64_t pix;
        if (MODE == 0) {
            pix = hash32((uint32_t)(tid * 977 + k * 7919) ^ salt) % (uint32_t)npix;
        } else if (MODE == 1) {
            const int64_t b = hash32((uint32_t)(warp * 131 + k) ^ salt) % (uint32_t)(npix / 32);
            pix = b * 32 + lane;
        } else {
            const uint32_t h = hash32((uint32_t)(warp * 131 + k) ^ salt);
            const int bx = (int)(h % (uint32_t)(W / 8)), by = (int)((h >> 12) % (uint32_t)(H / 4));
            pix = (int64_t)(by * 4 + (lane >> 3)) * W + bx * 8 + (lane & 7);
        }
        const unsigned long long word =
            ((unsigned long long)hash32((uint32_t)(tid + k * 31) ^ 0x55u) << 32) | (uint32_t)tid;
        atomicMin(fb + pix, word);
    }
}

int main() {
    const int W = 3840, H = 2160;
    unsigned long long *fb;
    cudaMalloc(&fb, (size_t)W * H * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = 148 * 8, threads = 256;
    const int64_t per = 64;
    const double merges = (double)blocks * threads * per;
    const char *names[3] = {"scattered", "rows", "tile8x4"};
    for (int mode = 0; mode < 3; ++mode) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemset(fb, 0xff, (size_t)W * H * 8);
            cudaEventRecord(e0);
            if (mode == 0) k_red<0><<<blocks, threads>>>(fb, W, H, per, rep);
            else if (mode == 1) k_red<1><<<blocks, threads>>>(fb, W, H, per, rep);
            else k_red<2><<<blocks, threads>>>(fb, W, H, per, rep);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("{\"pattern\": \"%s\", \"merges\": %.0f, \"ms\": %.4f, \"merges_per_s\": %.4e}\n",
               names[mode], merges, best, merges / (best * 1e-3));
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
